# build f93d8f83 (comment-only change over 164b67e4) + the far_small degree test: quick GPU suite, ncu C3 eval, C3 bench
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id_r02c.txt
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider -rf > gpurun_out/r02c_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02c_gpu_tests.log
bash tools/gpu_ncu_src.sh r02c C3
timeout 900 python bench.py --config C3 > gpurun_out/r02c_bench_C3.json 2> gpurun_out/r02c_bench_C3.err; echo "C3 rc=$?"
