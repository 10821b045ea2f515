mkdir -p gpurun_out
for c in C4n4 C4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-check > gpurun_out/ln_$c.json 2>gpurun_out/ln_$c.err; python -c "import json; d=json.load(open('gpurun_out/ln_$c.json')); r=d['roofline']; print('$c', d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], r['pairs_per_launch'])"; done
PM_N=4,5,6,8 PM_THETA=0.7 timeout 300 python tools/perf_matrix.py
python tools/profile_step.py C4n4 2 > gpurun_out/plain_ln.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_c4n4 python tools/profile_step.py C4n4 2 > gpurun_out/ncu_ln.log 2>&1; echo ncu rc=$?
