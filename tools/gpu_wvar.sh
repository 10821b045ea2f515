# modified-weights kernel variants: parity tests on the product build, then per-phase times per variant
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 120 -k "weights or split_ranges or upward" > gpurun_out/wv_tests.log 2>&1; echo "w tests rc=$?"; tail -2 gpurun_out/wv_tests.log
for c in C3 C5 C4; do for v in "$@"; do echo -n "$c $v: "; KITC_LIB=tools/variants/libkitc_$v.so timeout 200 python tools/phase_times.py $c 10 2>&1 | tail -1; done; done
