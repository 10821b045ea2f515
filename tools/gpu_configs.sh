for c in C4 C5 C2; do
  echo "== $c"
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').readlines()[-1]); r=d['roofline']; print('value %.4g ms %.2f eval_ms %.2f frac %.3f pairs %.3g E %s clusters %s depth %s'%(d['value'],d['ms_per_step'],r['launch_ms'],r['frac'],r['pairs_per_launch'],d['check'],d['config']['clusters'],d['config']['depth']))" || tail -5 gpurun_out/bench_$c.err
done
