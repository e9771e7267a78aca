#!/bin/bash
# ncu --set full of the integer-slice neighbour search (one launch) at n=$N (config-3 recipe)
CMD="python tools/knn_probe.py ${N:-100000}"
$CMD > gpurun_out/knn_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"knn_i8" -s 1 -c 1 \
   -o gpurun_out/prof_knn${TAG:-} $CMD > gpurun_out/ncu_knn.log 2>&1
echo "ncu rc=$?"
