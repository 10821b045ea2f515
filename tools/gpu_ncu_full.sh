# ncu --set full capture of one k_eval launch (after a clean run of the same command)
# usage: bash tools/gpu_ncu_full.sh TAG [config]
TAG=$1; CFG=${2:-C3}
mkdir -p gpurun_out
python tools/profile_step.py $CFG 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py $CFG 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
