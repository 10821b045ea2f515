# round-2 (session 4): per-rank work of the 1/2/4/8-GPU decomposition re-timed on one GPU at the final build
mkdir -p gpurun_out
for c in C3 C5; do timeout 900 python tools/scale_emulate.py $c 3 > gpurun_out/r02i_scale_$c.log 2>&1; echo "$c rc=$?"; tail -2 gpurun_out/r02i_scale_$c.log | cut -c1-400; done
ls gpurun_out | grep -i scale
