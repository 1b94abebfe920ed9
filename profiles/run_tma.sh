#!/bin/bash
# correctness of every tile kernel choice + TMA / work-list / CTA A/B
set -u
TAG=${1:-r02h}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
for W in porous512@0.1 porous512 porous512@0.9 vascular1024; do
  timeout 900 python bench.py --workload $W --steps 300 --warmup 20 --variants 9,8,9,8 >> gpurun_out/variants_${TAG}.txt 2>&1
done
rm -f gpurun_out/ab_lib.txt
for S in ab aa; do
  echo "== channel512 $S" >> gpurun_out/ab_lib.txt
  bash profiles/ab_lib.sh exp_lib/base --workload channel512 --steps 300 --warmup 20 --scheme $S
done
mv gpurun_out/ab_lib.txt gpurun_out/ab_dense_${TAG}.txt
