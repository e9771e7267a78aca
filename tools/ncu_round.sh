#!/bin/bash
# ncu evidence for the bench path at the config-3 recipe (m=500, m_v=30) with n=300k (cheaper input generation).
set -e
CMD="python bench.py --n 300000 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:vif:: -c 40 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"vecchia_kernel|gemm_tn_kernel|syrk_kernel|chol_inv" -s 5 -c 5 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu-done
