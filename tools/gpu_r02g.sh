# round-2 (session 4) confirmation at HEAD after the container was re-created: full GPU suite, smoke,
# default bench line (C3), reference arm
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id_r02g.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r02g_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02g_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02g_smoke.log
timeout 900 python bench.py > gpurun_out/r02g_bench_C3.json 2> gpurun_out/r02g_bench_C3.err; echo "C3 rc=$?"
tail -1 gpurun_out/r02g_bench_C3.json | cut -c1-600
