# GPU check of the widened rows: full -m gpu suite, X2 (paper Example 2) bench line, C2 sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_all.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gpu_tests_all.log
timeout 600 python bench.py --config X2 > gpurun_out/bench_X2.json 2> gpurun_out/bench_X2.err; echo "X2 rc=$?"
tail -1 gpurun_out/bench_X2.json | cut -c1-400
timeout 900 python tools/sweep_c2.py > gpurun_out/c2_sweep.json 2> gpurun_out/c2_sweep.err; echo "sweep rc=$?"
tail -3 gpurun_out/c2_sweep.err
