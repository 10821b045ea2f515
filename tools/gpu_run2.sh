./tools/rsqrt_probe > gpurun_out/rsqrt_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gpu_tests.log
cat gpurun_out/rsqrt_probe.txt
