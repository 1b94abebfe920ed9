#!/bin/bash
# Tile-shape sweep with the warp work list forced (LBM_STEP_VARIANT=8) and the
# CTA-per-tile kernel (7), across porosity and C4: the round-1 sweep had only
# measured tiles below 512 nodes with the CTA kernel.
set -u
mkdir -p gpurun_out
for W in porous512@0.1 porous512@0.2 porous512 porous512@0.9 vascular1024; do
  for T in 4,4,8 4,4,4 2,4,8 4,8,8 8,8,8 4,8,16 4,4,16 2,8,8 8,4,4; do
    timeout 300 python bench.py --workload $W --tile $T --steps 300 --warmup 20 --variants 8,7 2>/dev/null | grep "^{" >> gpurun_out/tile_sweep_r02ag.txt
  done
done
