# ncu --set full of the non-eval kernels (tree build, modified weights) for HBM / FP64 evidence
# usage: bash tools/gpu_ncu_aux.sh TAG CONFIG
TAG=$1; CFG=${2:-C3}
mkdir -p gpurun_out
python tools/profile_step.py $CFG 2 > gpurun_out/plain_aux_$TAG.log 2>&1 && \
ncu --set full --clock-control none -k 'regex:k_weights|k_bbox_partial|k_part_scatter|k_part_count|k_leaf_order|k_gather_w|k_copy_back' -s 12 -c 14 -o gpurun_out/prof_aux_$TAG python tools/profile_step.py $CFG 2 > gpurun_out/ncu_aux_$TAG.log 2>&1
echo "ncu rc=$?"
