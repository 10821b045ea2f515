# eval variants: GPU parity on the first variant, then the Stokeslet eval over n on the C3 input per variant
# usage: bash tools/gpu_evar.sh v1 v2 ...  (tools/variants/libkitc_<v>.so); PM_N to choose degrees
mkdir -p gpurun_out
KITC_LIB=$PWD/tools/variants/libkitc_$2.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 200 > gpurun_out/ev_tests_$2.log 2>&1; echo "parity ($2) rc=$?"; tail -2 gpurun_out/ev_tests_$2.log
for v in "$@"; do echo "== $v"; KITC_LIB=$PWD/tools/variants/libkitc_$v.so PM_KERN=${PM_KERN:-0} PM_N=${PM_N:-4,5,8} PM_THETA=0.7 timeout 300 python tools/perf_matrix.py 2>&1 | tail -4; done
