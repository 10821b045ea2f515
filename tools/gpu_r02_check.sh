# round-2 GPU check: build id, host, full GPU suite (incl. full-size parity), smoke, C3 bench line
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id.txt
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv) > gpurun_out/host.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in ${CFGS:-C3}; do timeout 900 python bench.py --config $c > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02_bench_$c.json')); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r.get('frac_of_measured'), d['clocks'], d.get('check'))"; done
