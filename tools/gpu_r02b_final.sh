# round-2 (session 2) evidence at the final build: full GPU suite (incl. full-size parity and the checked
# build), smoke, ncu of the C3 eval, bench lines for every config, launch list, reference arm
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id_r02b.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r02b_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02b_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02b_smoke.log
bash tools/gpu_ncu_src.sh r02b C3
for c in C3 C4 C4n4 C5 C2 X1 X1L X2; do
  timeout 900 python bench.py --config $c > gpurun_out/r02b_bench_$c.json 2> gpurun_out/r02b_bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02b_bench_$c.json')); r=d['roofline']; print('  ', d['value'], d['ms_per_step'], round(r['frac'],4), round(r['frac_of_measured'] or 0,4), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b_bench_ref_C3.json 2> gpurun_out/r02b_bench_ref.err; echo "ref rc=$?"
tail -1 gpurun_out/r02b_bench_ref_C3.json | cut -c1-300
