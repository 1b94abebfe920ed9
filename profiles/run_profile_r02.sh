#!/bin/bash
# Round-2 evidence: default bench line (with the sparse block), the reference
# arm, ncu launch lists + one --set full capture per workload, the TMA
# kernel's capture, and the multi-rank path on one GPU (2 ranks, gloo plumbing).
set -u
TAG=${1:-r02i}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_${TAG}.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2>&1
timeout 1500 bash profiles/profile.sh ${TAG} channel512 porous512 vascular1024 porous512@0.1
BENCH_EXTRA="--scheme aa" timeout 900 bash profiles/profile.sh ${TAG}aa channel512
# the TMA-staged tile kernel (variant 9) on C3
LBM_STEP_VARIANT=9 timeout 900 bash profiles/profile.sh ${TAG}tma porous512
# N = 2 on one GPU: both ranks share the device (functional check of the
# C5 duct default, the solo-rate leg and the IPC peer stores; not a scaling number)
LBM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 5 \
  > gpurun_out/bench_${TAG}_multi2_samegpu.json 2> gpurun_out/bench_${TAG}_multi2_samegpu.err

# keep the copy-back under gpurun's 64 MiB: the raw/source CSVs carry the numbers
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
