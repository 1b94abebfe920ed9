#!/bin/bash
# cudaLimitMaxL2FetchGranularity (the L2's DRAM fetch size hint): in-process
# A/B per workload (geometry built once), then ncu DRAM bytes per setting.
set -u
TAG=${1:-r02au}
mkdir -p gpurun_out
V="LBM_L2FETCH=128,LBM_L2FETCH=32,LBM_L2FETCH=64,LBM_L2FETCH=128,LBM_L2FETCH=32,LBM_L2FETCH=64"
for W in porous512@0.1 porous512 vascular1024 channel512; do
  timeout 900 python bench.py --workload $W --steps 300 --warmup 20 --variants $V 2>> gpurun_out/l2fetch_${TAG}.err | grep "^{" >> gpurun_out/l2fetch_${TAG}.txt
done
for F in 128 32; do
  LBM_L2FETCH=$F ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -s 20 -c 2 --csv \
      --log-file gpurun_out/launches_l2fetch_${F}_${TAG}.csv \
      python bench.py --workload porous512@0.1 --steps 2 --warmup 20 --no-cpu --no-e2e --no-sparse > /dev/null 2>&1
done
