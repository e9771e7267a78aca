#!/bin/bash
# ncu --set full of the integer-slice kernels (K1: kx_slice + oz_gemm; K4: oz_colmax + oz_slice + oz_syrk) at
# n=$N (config-3 recipe), one launch each after the warm-up evaluation.
CMD="python tools/vecchia_probe.py ${N:-1000000} 0"
$CMD > gpurun_out/ncu_plain_oz.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"kx_slice|oz_gemm|oz_colmax|oz_slice|oz_syrk" -s 5 -c 5 \
   -o gpurun_out/prof_oz${TAG:-} $CMD > gpurun_out/ncu_full_oz.log 2>&1
echo "ncu rc=$?"
