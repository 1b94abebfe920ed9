#!/bin/bash
# Slab overhead on ONE GPU (in-process slabs, one stream each): dense AB / A-A
# channel 512^3, porous 512^3 tile slabs AB (work list + boundary-first) and A-A;
# plus the per-phase launch list of the A-A tile steps.
set -u
TAG=${1:-r02p}
mkdir -p gpurun_out
timeout 900 python profiles/slab_overhead.py ab > gpurun_out/slab_overhead_${TAG}.txt 2>&1
timeout 900 python profiles/slab_overhead.py aa > gpurun_out/slab_overhead_aa_${TAG}.txt 2>&1
timeout 900 python profiles/tile_slab_overhead.py ab > gpurun_out/tile_slab_overhead_${TAG}.txt 2>&1
timeout 900 python profiles/tile_slab_overhead.py aa > gpurun_out/tile_slab_overhead_aa_${TAG}.txt 2>&1
for W in vascular1024 porous512; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -s 40 -c 4 --csv \
    --log-file gpurun_out/launches_aa_${TAG}_${W}.csv python bench.py --workload $W --scheme aa --steps 5 --warmup 40 --no-cpu --no-e2e > /dev/null 2>&1
done
