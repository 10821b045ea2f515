# eval time over n (theta 0.7, C3 input) for the in-tree build and tuning variants:
# bash tools/pm_variants.sh default v1 v2 ...   (variants: tools/build_variant.py)
for v in "$@"; do
  if [ "$v" = default ]; then unset KITC_LIB; else export KITC_LIB=$PWD/tools/variants/libkitc_$v.so; fi
  echo "== $v"; PM_N=${PM_N:-3,4,5,6,7,8,9,10} PM_THETA=${PM_THETA:-0.7} timeout 300 python tools/perf_matrix.py | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['kernel'], d['n'], '%.2f'%d['eval_ms'], '%.3f'%d['frac'])" | paste -s -d' '
done
