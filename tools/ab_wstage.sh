#!/bin/bash
# A/B of the vecchia W pass at n = 1M (VIF_WPASS: 0 register-only, 1 cp.async-staged pairs, 2 staged + early pair)
python -m paper_2507_05064_b200.build > /dev/null
for r in 1 2; do for wm in ${WMS:-0 1 2}; do
VIF_WPASS=$wm timeout 900 python tools/vecchia_probe.py ${N:-1000000} 0 2>&1 | grep '^{' | tee -a gpurun_out/ab_wstage2.jsonl
done; done
