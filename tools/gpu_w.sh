mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 120 -k "weights or split_ranges or upward" > gpurun_out/w_tests.log 2>&1; echo "w tests rc=$?"; tail -2 gpurun_out/w_tests.log
for c in C3 C5; do timeout 200 python tools/phase_times.py $c 10 2>&1 | tail -1; done
bash tools/gpu_ncu_weights.sh r02db C5
python tools/ncu_summary.py gpurun_out/prof_w_r02db.ncu-rep 2>&1 | head -12
