# build with the target coordinates read from the packed records: quick GPU suite, ncu C3 eval (traffic record
# updated on the box so the bench line below ties to it), C3 / C5 bench lines
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id_r02d.txt
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider -rf > gpurun_out/r02d_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02d_gpu_tests.log
bash tools/gpu_ncu_src.sh r02d C3
python tools/ncu_summary.py gpurun_out/prof_r02d.ncu-rep > gpurun_out/r02d_ncu_eval_C3.txt 2>&1
python tools/ncu_traffic.py C3 gpurun_out/prof_r02d.ncu-rep $(cat gpurun_out/build_id_r02d.txt) profiles/r02d_ncu_eval_C3.txt
for c in C3 C5; do
  timeout 900 python bench.py --config $c > gpurun_out/r02d_bench_$c.json 2> gpurun_out/r02d_bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02d_bench_$c.json')); r=d['roofline']; print('  ', d['value'], d['ms_per_step'], round(r['frac'],4), r['traffic'], r.get('traffic_same_build'), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
