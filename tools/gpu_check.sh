mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/tb_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tb_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in X1 X1L C3; do timeout 600 python bench.py --config $c > gpurun_out/tb_bench_$c.json 2> gpurun_out/tb_bench_$c.err; echo "$c rc=$?"; python -c "import json; d=json.load(open('gpurun_out/tb_bench_$c.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'], d.get('check'))"; done
FUZZ_OFFSET=500 timeout 900 python tools/fuzz_medium.py 40 > gpurun_out/tb_fuzz.log 2>&1; echo fuzz rc=$?; tail -2 gpurun_out/tb_fuzz.log
