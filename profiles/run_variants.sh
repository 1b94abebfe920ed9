#!/bin/bash
# GPU tests, then in-process variant A/B of the sparse tile kernels
# (bench --variants): 8 warp work list (default below live fraction 0.85),
# 7 CTA per tile, 9 TMA-staged tiles; and the library against the round-1
# build (exp_lib/base) in alternating processes.
set -u
TAG=${1:-r02g}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
for W in porous512@0.1 porous512@0.2 porous512 porous512@0.9 vascular1024; do
  timeout 900 python bench.py --workload $W --steps 300 --warmup 20 --variants 8,7,9,8,7,9 >> gpurun_out/variants_${TAG}.txt 2>&1
done
rm -f gpurun_out/ab_lib.txt
for W in porous512@0.1 porous512 vascular1024; do
  echo "== $W" >> gpurun_out/ab_lib.txt
  bash profiles/ab_lib.sh exp_lib/base --workload $W --steps 300 --warmup 20
done
mv gpurun_out/ab_lib.txt gpurun_out/ab_vs_r01_${TAG}.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
