#!/bin/bash
# A/B of vecchia kernel variants at n=$N (config-3 recipe), then parity (gpu, not slow) of candidates.
#   SPECS="VIF_VREG_CFG=134 VIF_VECCHIA_VARIANT=4" CANDS="VIF_VECCHIA_VARIANT=4" bash tools/ab_vecchia.sh
N=${N:-300000}
for spec in $SPECS; do
  env $spec timeout 600 python tools/vecchia_probe.py $N ${FLAGS:-0} 2>&1 | grep '^{' | tee -a gpurun_out/ab.jsonl
done
for spec in $CANDS; do
  env $spec timeout 900 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -3 | sed "s/^/$spec: /" | tee -a gpurun_out/pytest_cand.log
done
