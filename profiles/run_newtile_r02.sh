#!/bin/bash
# The 4x4x8 default tile (work list everywhere): GPU suite, the driver's bench
# command, the porosity sweep, A-A lines, ncu captures keyed for the new tile.
set -u
TAG=${1:-r02ah}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=6 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_driver.json 2> gpurun_out/bench_${TAG}_driver.err
for P in 0.1 0.2 0.3 0.5 0.7 0.9; do
  timeout 600 python bench.py --workload porous512@$P --steps 300 --warmup 20 --no-cpu --no-e2e > gpurun_out/sweep_${TAG}_$P.json 2>&1
done
for W in porous512 vascular1024; do
  timeout 900 python bench.py --workload $W --scheme aa --no-cpu --no-e2e > gpurun_out/bench_${TAG}_${W}_aa.json 2>&1
  timeout 900 python bench.py --workload $W --dtype f64 --steps 300 --warmup 20 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_${W}_f64.json 2>&1
done
timeout 1500 bash profiles/profile.sh ${TAG} porous512 vascular1024 porous512@0.1
rm -f gpurun_out/*.ncu-rep
