#!/bin/bash
# Round-2 bench lines for DESIGN §5 (one B200): GPU tests, C2 setup phases,
# A-A / f64 / C5 lines, the porosity sweep.
set -u
TAG=${1:-r02k}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
LBM_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-sparse > gpurun_out/bench_${TAG}_setup_phases.json 2> gpurun_out/setup_phases_${TAG}.txt
for W in porous512 vascular1024; do
  timeout 900 python bench.py --workload $W --scheme aa --no-cpu --no-e2e > gpurun_out/bench_${TAG}_${W}_aa.json 2>&1
done
timeout 900 python bench.py --workload channel512 --scheme aa --no-cpu > gpurun_out/bench_${TAG}_channel512_aa.json 2>&1
timeout 1500 python bench.py --workload c5 --steps 300 --warmup 10 --no-cpu > gpurun_out/bench_${TAG}_c5.json 2>&1
for W in channel512 porous512; do
  timeout 900 python bench.py --workload $W --dtype f64 --steps 300 --warmup 20 --no-cpu --no-e2e --no-sparse > gpurun_out/bench_${TAG}_${W}_f64.json 2>&1
done
for P in 0.1 0.2 0.3 0.5 0.7 0.9; do
  timeout 600 python bench.py --workload porous512@$P --steps 300 --warmup 20 --no-cpu --no-e2e > gpurun_out/sweep_${TAG}_$P.json 2>&1
done
timeout 600 python bench.py --workload cavity64 --steps 1000 --warmup 100 --no-cpu > gpurun_out/bench_${TAG}_cavity64.json 2>&1
