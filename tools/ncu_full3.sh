#!/bin/bash
# ncu --set full of the three dominant kernels at the bench configuration (config 3, n = 1M).
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/ncu3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"vecchia_reg_kernel|gemm_tn_kernel|syrk_kernel|kx_eval" -s 4 -c 4 -o gpurun_out/prof_r01_c3 $CMD \
    > gpurun_out/ncu3_full.log 2>&1
echo "ncu rc=$?"
