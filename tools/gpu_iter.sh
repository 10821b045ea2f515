# one GPU iteration: parity tests on the in-tree build, then a variant sweep
# usage: bash tools/gpu_iter.sh v1 v2 ...
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_tests.log
bash tools/gpu_sweep.sh "$@"
