#!/bin/bash
# ncu --set full of the vecchia kernel at the config-3 recipe (n=300k) after a plain run of the same command.
# usage: tools/ncu_vecchia.sh TAG [kernel-regex]   (env vars such as VIF_VECCHIA_VARIANT pass through)
CMD="python bench.py --n 300000 --steps 2 --warmup 1 --no-cpu-baseline"
TAG=${1:-cur}
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"${2:-vecchia}" -s 2 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
