# round-2 (session 3) evidence at the final build (modified-weights pipeline): full GPU suite (incl.
# full-size parity and the checked build), smoke, ncu of the C3 eval (traffic record re-tied to this build)
# and of the C5 modified weights, bench lines for every config, launch list, reference arm
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id_r02f.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r02f_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02f_smoke.log
bash tools/gpu_ncu_src.sh r02f C3
python tools/ncu_summary.py gpurun_out/prof_r02f.ncu-rep > gpurun_out/r02f_ncu_eval_C3.txt 2>&1
python tools/ncu_traffic.py C3 gpurun_out/prof_r02f.ncu-rep $(cat gpurun_out/build_id_r02f.txt) profiles/r02f_ncu_eval_C3.txt
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_r02f.json
bash tools/gpu_ncu_weights.sh r02f C5
python tools/ncu_summary.py gpurun_out/prof_w_r02f.ncu-rep > gpurun_out/r02f_ncu_weights_C5.txt 2>&1
for c in C3 C5 C4 C4n4 C2 X1 X1L X2; do
  timeout 900 python bench.py --config $c > gpurun_out/r02f_bench_$c.json 2> gpurun_out/r02f_bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02f_bench_$c.json')); r=d['roofline']; print('  ', d['value'], d['ms_per_step'], round(r['frac'],4), round(r['frac_of_measured'] or 0,4), r.get('traffic_same_build'), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_ref_C3.json 2> gpurun_out/r02f_bench_ref.err; echo "ref rc=$?"
tail -1 gpurun_out/r02f_bench_ref_C3.json | cut -c1-300
