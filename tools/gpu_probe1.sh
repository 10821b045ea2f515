# r02b: far-field probe + quick GPU tests + C3 timing
mkdir -p gpurun_out
./tools/far_probe > gpurun_out/far_probe.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/far_probe.txt
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
bash tools/gpu_sweep.sh default
