#!/bin/bash
# launch list of one vif_grad call (after a warm-up call) at n=$N
CMD="python tools/grad_probe.py ${N:-300000} 1"
$CMD > gpurun_out/grad_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/grad_launches.csv $CMD > gpurun_out/grad_ncu.log 2>&1
echo "ncu rc=$?"; tail -1 gpurun_out/grad_plain.log
