#!/bin/bash
# Full ncu capture of both A-A tile steps (node-local and neighbour) on C4,
# to compare with the AB work-list step's capture (ncu_r02an.md).
set -u
mkdir -p gpurun_out
LBM_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:k_step_tiles_aa_w -s 600 -c 2 \
    -o gpurun_out/prof_aa_r02aq -f \
    python bench.py --workload vascular1024 --scheme aa --steps 2 --warmup 600 --no-cpu --no-e2e --no-sparse > gpurun_out/ncu_aa_r02aq.log 2>&1
ncu -i gpurun_out/prof_aa_r02aq.ncu-rep --page raw --csv > gpurun_out/raw_aa_r02aq.csv 2>/dev/null
ncu -i gpurun_out/prof_aa_r02aq.ncu-rep --page details --csv > gpurun_out/details_aa_r02aq.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
