#!/bin/bash
# End-of-round check: GPU suite, smoke, the driver's bench command, the
# reference arm, C1 (clock window check), N = 2 on one GPU.
set -u
TAG=${1:-r02final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
S=$(date +%s)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_driver.json 2> gpurun_out/bench_${TAG}_driver.err
echo "wall $(( $(date +%s) - S )) s" >> gpurun_out/bench_${TAG}_driver.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_reference.json 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}_default1000.json 2> gpurun_out/bench_${TAG}_default1000.err
timeout 600 python bench.py --workload cavity64 --steps 1000 --warmup 100 --no-cpu > gpurun_out/bench_${TAG}_cavity64.json 2>&1
LBM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 5 \
  > gpurun_out/bench_${TAG}_multi2_samegpu.json 2> gpurun_out/bench_${TAG}_multi2_samegpu.err
