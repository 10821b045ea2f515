# round-2 evidence: full GPU suite, smoke, bench lines for every config, reference arm, launch list, ncu of the eval
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02_smoke.log
for c in ${CFGS:-C3 C4 C4n4 C5 C2 X1 X1L X2}; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02_bench_$c.json')); r=d['roofline']; print('  ', d['value'], d['ms_per_step'], round(r['frac'],4), round(r['frac_of_measured'] or 0,4), r['peak_measured'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d.get('check'))"
done
timeout 900 python bench.py --impl reference --config C3 --steps 2 --warmup 1 > gpurun_out/r02_bench_ref_C3.json 2> gpurun_out/r02_bench_ref_C3.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/r02_plain_launches.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/r02_ncu_launches.log 2>&1; echo "launches rc=$?"
bash tools/gpu_ncu_src.sh r02final C3
