nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
kill $SMI
nproc > gpurun_out/host.txt; lscpu | grep -i "model name" >> gpurun_out/host.txt
nvidia-smi >> gpurun_out/host.txt
