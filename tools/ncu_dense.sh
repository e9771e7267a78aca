#!/bin/bash
# ncu --set full of the dense kernels (kx_eval, gemm_tn, syrk) at n=$N (config-3 recipe).
CMD="python tools/vecchia_probe.py ${N:-300000} 0"
$CMD > gpurun_out/ncu_plain_dense.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"kx_eval|gemm_tn|syrk_kernel" -s 3 -c 3 \
   -o gpurun_out/prof_dense${TAG:-} $CMD > gpurun_out/ncu_full_dense.log 2>&1
echo "ncu rc=$?"
