# variant check: quick parity (treecode tests) per variant, then C3 timing per variant
# usage: [CFG=C3] [TESTK=expr] bash tools/gpu_var.sh v1 v2 ...
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then unset KITC_LIB; else export KITC_LIB=$PWD/tools/variants/libkitc_$v.so; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "${TESTK:-treecode_parity or degenerate or self_include}" > gpurun_out/var_$v.log 2>&1; echo "$v parity rc=$? $(tail -1 gpurun_out/var_$v.log)"
done
unset KITC_LIB
for rep in 1 2; do bash tools/gpu_sweep.sh "$@"; done
