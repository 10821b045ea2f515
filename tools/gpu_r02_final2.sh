# round-2 evidence after the late changes: GPU suite, smoke, bench lines, ncu of the C3 eval (traffic + build id)
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02_smoke.log
bash tools/gpu_ncu_src.sh r02final2 C3
python tools/ncu_traffic.py C3 gpurun_out/prof_r02final2.ncu-rep $(cat gpurun_out/build_id_r02final2.txt) profiles/r02_ncu_eval_C3_final.txt
for c in ${CFGS:-C3 C4 C4n4 C5 C2 X1 X1L X2}; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02_bench_$c.json')); r=d['roofline']; print('  ', d['value'], d['ms_per_step'], round(r['frac'],4), round(r['frac_of_measured'] or 0,4), r['traffic'], r['traffic_same_build'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d.get('check'))"
done
