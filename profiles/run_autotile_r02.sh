#!/bin/bash
# The fill-based default tile (4x4x4 when the kept 4x4x8 tiles are < 70 %
# non-solid): GPU suite, smoke, the driver's bench command, the porosity sweep
# with the default tile, ncu captures keyed by the tile each run used.
set -u
TAG=${1:-r02an}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
S=$(date +%s%N)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_driver.json 2> gpurun_out/bench_${TAG}_driver.err
echo "driver command wall $(( ($(date +%s%N) - S) / 1000000 )) ms" >> gpurun_out/bench_${TAG}_driver.err
for P in 0.1 0.2 0.3 0.5; do
  timeout 600 python bench.py --workload porous512@$P --steps 300 --warmup 20 --no-cpu --no-e2e > gpurun_out/sweep_${TAG}_$P.json 2>&1
done
timeout 1500 bash profiles/profile.sh ${TAG} porous512@0.1 porous512@0.2 vascular1024
rm -f gpurun_out/*.ncu-rep
