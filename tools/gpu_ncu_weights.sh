# ncu --set full of the modified-weights kernel (Algorithm 1): usage bash tools/gpu_ncu_weights.sh TAG CONFIG
TAG=$1; CFG=${2:-C3}
python tools/profile_step.py $CFG 2 > gpurun_out/plain_w_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k 'regex:k_weights' -s 1 -c 1 -o gpurun_out/prof_w_$TAG python tools/profile_step.py $CFG 2 > gpurun_out/ncu_w_$TAG.log 2>&1
echo "ncu rc=$?"
