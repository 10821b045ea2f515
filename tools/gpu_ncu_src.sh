# ncu --set full + source of one k_eval launch, and a DRAM-traffic record for the bench
# usage: bash tools/gpu_ncu_src.sh TAG [config]
TAG=$1; CFG=${2:-C3}
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id_$TAG.txt
python tools/profile_step.py $CFG 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py $CFG 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
