# Round bench evidence: full bench lines per config, the bench launch list, ncu --set full of the C4/C5 eval,
# and the reference (oracle) arm.  Outputs under gpurun_out/.
mkdir -p gpurun_out
for c in C3 C4 C5 C2; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_$c.json | cut -c1-300
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
bash tools/gpu_ncu_full.sh c4 C4
bash tools/gpu_ncu_full.sh c5 C5
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.json | cut -c1-300
