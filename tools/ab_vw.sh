#!/bin/bash
# A/B of the vecchia register kernel's warps per block at n = 1M (VIF_VREG_VW = 4, 1, 2; 16 warps per SM)
python -m paper_2507_05064_b200.build > /dev/null
for r in 1 2; do for vw in ${VWS:-4 1 2}; do
VIF_VREG_VW=$vw timeout 900 python tools/vecchia_probe.py ${N:-1000000} 0 2>&1 | grep '^{' | tee -a gpurun_out/ab_vw.jsonl
done; done
