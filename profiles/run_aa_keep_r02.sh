#!/bin/bash
# A-A neighbour step with the pull addresses kept for the pushes (KEEP) at
# several register caps vs the recomputing default: parity, then in-process
# A/B (geometry built once per workload), clocks logged alongside.
set -u
TAG=${1:-r02as}
mkdir -p gpurun_out
for K in 2 3 4; do LBM_AA_KEEP=$K timeout 600 python -m pytest tests/test_gpu_aa.py -x -q 2>&1 | tail -1 | sed "s/^/keep=$K /" >> gpurun_out/keep_tests_${TAG}.txt; done
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 500 > gpurun_out/keep_clocks_${TAG}.csv &
SMI=$!
V="LBM_AA_KEEP=0,LBM_AA_KEEP=3,LBM_AA_KEEP=4,LBM_AA_KEEP=0,LBM_AA_KEEP=3,LBM_AA_KEEP=4"
for W in vascular1024 porous512@0.1 porous512; do
  timeout 900 python bench.py --workload $W --scheme aa --steps 400 --warmup 20 --variants $V 2>/dev/null | grep "^{" >> gpurun_out/ab_aa_keep_${TAG}.txt
done
V="LBM_AA_KEEP=0,LBM_AA_KEEP=2,LBM_AA_KEEP=3,LBM_AA_KEEP=4,LBM_AA_KEEP=0,LBM_AA_KEEP=2,LBM_AA_KEEP=3,LBM_AA_KEEP=4"
for W in vascular1024 porous512@0.1; do
  timeout 900 python bench.py --workload $W --scheme aa --dtype f64 --steps 300 --warmup 20 --variants $V 2>/dev/null | grep "^{" | sed 's/^{/{"dtype": "f64", /' >> gpurun_out/ab_aa_keep_${TAG}.txt
done
kill $SMI
