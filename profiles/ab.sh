#!/bin/bash
# in-process interleaved A/B of library switches, then ncu DRAM bytes per variant
# usage: bash profiles/ab.sh "<variantA>,<variantB>,..." workload...
V=$1; shift
for W in "$@"; do
  timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --variants "$V" 2>>gpurun_out/ab.err
done
