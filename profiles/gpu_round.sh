#!/bin/bash
# One gpurun call: gpu tests, smoke, default bench, workload sweep, ncu launch lists + full captures.
# usage: bash profiles/gpu_round.sh <tag> [skip_tests]
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_${TAG}.txt 2>&1
if [ "${2:-}" != "skip_tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
  echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
fi
timeout 900 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2>&1
for W in porous512 vascular1024 cavity64; do
  timeout 900 python bench.py --workload $W --no-cpu > gpurun_out/bench_${TAG}_${W}.json 2> gpurun_out/bench_${TAG}_${W}.err
done
timeout 900 python bench.py --workload channel512 --scheme aa --no-cpu > gpurun_out/bench_${TAG}_channel512_aa.json 2> gpurun_out/bench_${TAG}_channel512_aa.err
timeout 1500 python bench.py --workload c5 --steps 300 --warmup 10 --no-cpu > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err
for W in channel512 porous512; do
  timeout 900 python bench.py --workload $W --dtype f64 --steps 300 --warmup 20 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_${W}_f64.json 2>&1
done
for W in porous512 vascular1024; do
  timeout 900 python bench.py --workload $W --scheme aa --no-cpu --no-e2e > gpurun_out/bench_${TAG}_${W}_aa.json 2>&1
done
for P in 0.1 0.2 0.3 0.5 0.7 0.9; do
  timeout 600 python bench.py --workload porous512@$P --steps 300 --warmup 20 --no-cpu --no-e2e > gpurun_out/sweep_${TAG}_$P.json 2>&1
done
timeout 1800 bash profiles/profile.sh ${TAG} channel512 porous512 vascular1024
ls -la gpurun_out
