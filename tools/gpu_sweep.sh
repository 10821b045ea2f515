# usage: [CFG=C4] bash tools/gpu_sweep.sh v1 v2 ...   (variants under tools/variants/libkitc_<v>.so; "default" = in-tree)
CFG=${CFG:-C3}
for v in "$@"; do
  if [ "$v" = default ]; then unset KITC_LIB; else export KITC_LIB=$PWD/tools/variants/libkitc_$v.so; fi
  echo "== $v $CFG"
  timeout 300 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-check 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print('value %.4g ms %.2f eval_ms %.2f frac %.3f launches %d'%(d['value'],d['ms_per_step'],r['launch_ms'],r['frac'],d['gpu_launches']))"
done
