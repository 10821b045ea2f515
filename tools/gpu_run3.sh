timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gpu_tests.log
for v in default tools/variants/libkitc_g2.so tools/variants/libkitc_g8.so; do
  if [ "$v" = default ]; then unset KITC_LIB; else export KITC_LIB=$PWD/$v; fi
  echo "== $v"
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-check 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print('value %.4g ms %.2f eval_ms %.2f frac %.3f launches %d'%(d['value'],d['ms_per_step'],r['launch_ms'],r['frac'],d['gpu_launches']))"
done
