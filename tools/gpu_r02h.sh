# round-2 (session 4): more fuzz seeds at the final build (700..1099 product library, 1100..1249 checked
# build), C3 repeatability (3 runs), C5 line, launch list of the default command
mkdir -p gpurun_out
python -c "from paper_1902_02250_b200 import build as B; print(B.build_id())" > gpurun_out/build_id_r02h.txt
{ echo "# python tools/fuzz_many.py 700 1100 (1 x B200, build $(cat gpurun_out/build_id_r02h.txt), product library)";
  timeout 1500 python tools/fuzz_many.py 700 1100 2>&1 | tail -8;
  echo "# KITC_LIB=paper_1902_02250_b200/libkitc_checks.so python tools/fuzz_many.py 1100 1250 (device-side checks compiled in)";
  KITC_LIB=paper_1902_02250_b200/libkitc_checks.so timeout 900 python tools/fuzz_many.py 1100 1250 2>&1 | tail -8; } > gpurun_out/r02h_fuzz.txt
tail -4 gpurun_out/r02h_fuzz.txt
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02h_bench_C3_run$i.json 2> gpurun_out/r02h_bench_C3_run$i.err; echo "C3 run$i rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02h_bench_C3_run$i.json')); r=d['roofline']; print('  ', d['value'], d['ms_per_step'], round(r['frac'],4), round(r['frac_of_measured'] or 0,4), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 900 python bench.py --config C5 --no-cpu-baseline > gpurun_out/r02h_bench_C5.json 2> gpurun_out/r02h_bench_C5.err; echo "C5 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02h_bench_C5.json')); r=d['roofline']; print('  ', d['value'], d['ms_per_step'], round(r['frac'],4), round(r['frac_of_measured'] or 0,4), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
