mkdir -p gpurun_out
python tools/profile_step.py C5 2 > gpurun_out/plain_c5f.log 2>&1 && python tools/bench_direct.py 300000 > gpurun_out/plain_dir.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_final_c5 python tools/profile_step.py C5 2 > gpurun_out/ncu_final_c5.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_direct -s 1 -c 1 -o gpurun_out/prof_final_direct python tools/bench_direct.py 300000 > gpurun_out/ncu_final_direct.log 2>&1
echo "ncu rc=$?"
