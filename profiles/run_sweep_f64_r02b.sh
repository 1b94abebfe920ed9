#!/bin/bash
# float64 porosity sweep where the fill-based default tile is 4x4x4 (phi <= 0.3).
set -u
TAG=${1:-r02ay}
mkdir -p gpurun_out
for P in 0.1 0.2 0.3; do
  timeout 600 python bench.py --workload porous512@$P --dtype f64 --steps 300 --warmup 20 --no-cpu --no-e2e > gpurun_out/sweep_f64_${TAG}_$P.json 2>&1
done
