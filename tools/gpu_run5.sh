timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_tests.log
bash tools/gpu_sweep.sh default m5 m4
