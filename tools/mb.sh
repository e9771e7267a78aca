nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/mb_clocks.csv &
SMI=$!
./tools/microbench_fp64 > gpurun_out/mb.jsonl 2>&1
python tools/dgemm_peak.py >> gpurun_out/mb.jsonl 2>&1
kill $SMI
nproc >> gpurun_out/mb_host.txt; lscpu | head -20 >> gpurun_out/mb_host.txt; free -g >> gpurun_out/mb_host.txt
cat gpurun_out/mb.jsonl
