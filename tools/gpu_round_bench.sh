# Round bench evidence: full bench lines per config, the bench launch list, ncu --set full of the eval
# (C3 and C4), and the reference (oracle) arm.  Outputs under gpurun_out/.  usage: bash tools/gpu_round_bench.sh TAG
TAG=${1:-v}
mkdir -p gpurun_out
for c in C3 C4 C5 C2 X2 X1 X1L; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_${c}_$TAG.json | cut -c1-200
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
bash tools/gpu_ncu_full.sh ${TAG}_c3 C3
bash tools/gpu_ncu_full.sh ${TAG}_c4 C4
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref_$TAG.json | cut -c1-200
