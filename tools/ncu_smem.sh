#!/bin/bash
# ncu --set full of the s > 32 vecchia kernel at config 5's recipe (n = 100k) after a plain run.
CMD=${CMD:-"python tools/config_probe.py 5 100000 2"}
TAG=${1:-smem}
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"${KREGEX:-vecchia_smem}" -s ${SKIP:-2} -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
