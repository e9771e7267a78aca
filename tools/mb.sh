# FP64 peak microbenchmarks; builds the executables from tools/*.cu if they are missing
for t in microbench_fp64 dmma_latency dmma_pattern dmma_mix rsq_test; do
  [ -x tools/$t ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/$t tools/$t.cu
done
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/mb_clocks.csv &
SMI=$!
./tools/microbench_fp64 > gpurun_out/mb.jsonl 2>&1
python tools/dgemm_peak.py >> gpurun_out/mb.jsonl 2>&1
kill $SMI
nproc >> gpurun_out/mb_host.txt; lscpu | head -20 >> gpurun_out/mb_host.txt; free -g >> gpurun_out/mb_host.txt
cat gpurun_out/mb.jsonl
