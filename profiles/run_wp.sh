#!/bin/bash
# persistent work list (13) vs the default work list (8); setup / e2e phases
set -u
TAG=${1:-r02l}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "launch_configuration or default_tile_kernel" > gpurun_out/pytest_wp_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_wp_${TAG}.log
for W in porous512@0.1 porous512@0.2 porous512 vascular1024; do
  timeout 900 python bench.py --workload $W --steps 300 --warmup 20 --variants 8,13,8,13 >> gpurun_out/variants_wp_${TAG}.txt 2>&1
done
LBM_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-sparse > gpurun_out/bench_${TAG}_e2e.json 2> gpurun_out/setup_phases_${TAG}.txt
