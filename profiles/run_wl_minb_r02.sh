#!/bin/bash
# Occupancy of the AB work-list step (default 48 warps / 40 registers) vs 40
# warps / 48 registers and 56 warps / 32 registers (+32 B stack), in-process.
set -u
TAG=${1:-r02av}
mkdir -p gpurun_out
V="LBM_WL_MINB=6,LBM_WL_MINB=5,LBM_WL_MINB=7,LBM_WL_MINB=6,LBM_WL_MINB=5,LBM_WL_MINB=7"
for W in porous512@0.1 porous512@0.2 porous512 vascular1024; do
  timeout 900 python bench.py --workload $W --steps 400 --warmup 20 --variants $V 2>/dev/null | grep "^{" >> gpurun_out/wl_minb_${TAG}.txt
done
