python tools/profile_step.py C3 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_eval_g8 python tools/profile_step.py C3 2 > gpurun_out/ncu_eval.log 2>&1
echo rc=$?
