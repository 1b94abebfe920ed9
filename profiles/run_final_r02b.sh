#!/bin/bash
# End-of-round refresh on the final tree: GPU suite, smoke, the driver's bench
# command (sparse block now finds ncu traffic for the default tiles), the
# 1000-step default, the reference arm.
set -u
TAG=${1:-r02final3}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
S=$(date +%s%N)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_driver.json 2> gpurun_out/bench_${TAG}_driver.err
echo "driver command wall $(( ($(date +%s%N) - S) / 1000000 )) ms" >> gpurun_out/bench_${TAG}_driver.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err
timeout 900 python bench.py --no-sparse > gpurun_out/bench_${TAG}_default1000.json 2> gpurun_out/bench_${TAG}_default1000.err
