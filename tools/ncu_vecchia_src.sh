#!/bin/bash
# ncu --set full (source counters) of the vecchia kernel at n=$N for the variant given as env spec $1
# (e.g. VIF_VREG_CFG=134 or VIF_VECCHIA_VARIANT=4); report gpurun_out/prof_vecchia_<tag>.ncu-rep.
SPEC=$1; TAG=${SPEC##*=}${2:-}
CMD="python tools/vecchia_probe.py ${N:-300000} 0"
env $SPEC $CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
env $SPEC ncu --set full --clock-control none --import-source on -k regex:vecchia -s 2 -c 1 \
   -o gpurun_out/prof_vecchia_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu $SPEC rc=$?"
