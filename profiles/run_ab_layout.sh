#!/bin/bash
# GPU tests + in-process-alternating A/B of the brick-record tile layout
# against the round-1 layout library (exp_lib/base/liblbm19.so).
set -u
TAG=${1:-r02d}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
rm -f gpurun_out/ab_lib.txt
for W in porous512@0.1 porous512@0.2 porous512 vascular1024; do
  echo "== $W" >> gpurun_out/ab_lib.txt
  bash profiles/ab_lib.sh exp_lib/base --workload $W --steps 300 --warmup 20
done
for W in porous512@0.1 vascular1024; do
  echo "== $W aa" >> gpurun_out/ab_lib.txt
  bash profiles/ab_lib.sh exp_lib/base --workload $W --steps 300 --warmup 20 --scheme aa
done
mv gpurun_out/ab_lib.txt gpurun_out/ab_layout_${TAG}.txt
