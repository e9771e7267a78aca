#!/bin/bash
# Round-end ncu evidence at the bench configuration (config 3, n = 1M):
#  1) launch list of the bench command (gpu__time_duration per launch, cold-cache, serialised)
#  2) ncu --set full (with source) of the dominant kernels: vecchia_reg and the integer-slice K1 / K4 kernels
# usage: bash tools/ncu_round.sh <tag>   (outputs gpurun_out/<tag>_*)
T=${1:-round}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-grad --npred 0 --no-knn --la-n 0"
$CMD > gpurun_out/${T}_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:vif:: -c 80 --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/${T}_ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"vecchia_reg_kernel|oz_gemm|oz_syrk|kx_slice" -s 4 -c 4 -o gpurun_out/${T}_prof $CMD \
    > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
