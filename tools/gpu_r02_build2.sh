mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider -rf > gpurun_out/tb_gpu_fast.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/tb_gpu_fast.log
for c in C3 C5 C2; do timeout 300 python tools/phase_times.py $c 10 2>&1 | tail -1; done
for c in C3 C5; do KITC_LIB=$PWD/tools/variants/libkitc_bprof.so timeout 300 python tools/build_prof.py $c; done
