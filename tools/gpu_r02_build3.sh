mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 60 -k "tree_bit_exact or tree_degenerate" > gpurun_out/tb_tree.log 2>&1; echo "tree tests rc=$?"; tail -15 gpurun_out/tb_tree.log
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --timeout 120 -rf > gpurun_out/tb_gpu_fast.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/tb_gpu_fast.log
for c in C3 C5 C2; do timeout 120 python tools/phase_times.py $c 10 2>&1 | tail -1; done
for c in C3 C5; do KITC_LIB=$PWD/tools/variants/libkitc_bprof.so timeout 120 python tools/build_prof.py $c; done
