#!/bin/bash
# per-stage times with ablation switches (SAR_DBG bit mask; numbers only, parity off)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in ${MASKS:-0 1 2 4 3 5 6 7}; do echo "mask=$m" >> gpurun_out/ablate.log; SAR_DBG=$m timeout 300 python scripts/probe_stages.py ${CFG:-large} 2>&1 | grep " comp" >> gpurun_out/ablate.log; done
