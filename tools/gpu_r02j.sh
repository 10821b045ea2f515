# round-2 (session 4): ncu launch list of the bench command at the final build (after the same command exited 0 without ncu)
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/r02j_b_plain.json 2> gpurun_out/r02j_b_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
python tools/ncu_summary.py gpurun_out/r02j_launches.csv > gpurun_out/r02j_bench_launches.txt; cat gpurun_out/r02j_bench_launches.txt
