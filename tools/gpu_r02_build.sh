# device-build check: GPU tests (non-slow), phase times C3/C5, C3 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider -x -rf > gpurun_out/tb_gpu_fast.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/tb_gpu_fast.log
for c in C3 C5 C2; do timeout 300 python tools/phase_times.py $c 10 2>&1 | tail -1; done
timeout 600 python bench.py --config C3 --no-cpu-baseline > gpurun_out/tb_bench_C3.json 2> gpurun_out/tb_bench_C3.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/tb_bench_C3.json')); r=d['roofline']; print(d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], d['gpu_launches'], d['e2e']['value'], d['check'])"
