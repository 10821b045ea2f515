# far_small (Stokeslet P <= 8): parity on the in-tree build, eval time over n vs the previous kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/gpu_tests_small.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests_small.log
for v in default nosmall; do
  if [ "$v" = default ]; then unset KITC_LIB; else export KITC_LIB=$PWD/tools/variants/libkitc_$v.so; fi
  echo "== $v"; PM_N=1,2,3,4,5,6,7 PM_THETA=0.7 timeout 600 python tools/perf_matrix.py 2>&1 | grep '"kernel": 0'
done
unset KITC_LIB
CFG=X1 bash tools/gpu_sweep.sh default nosmall
