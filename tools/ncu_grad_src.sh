#!/bin/bash
# ncu --set full (source) of one grad_param_kernel launch at n=$N
CMD="python tools/grad_probe.py ${N:-300000} 1"
$CMD > gpurun_out/gsrc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grad_param -s 5 -c 1 -o gpurun_out/prof_gparam $CMD \
   > gpurun_out/gsrc_ncu.log 2>&1
echo "ncu rc=$?"
