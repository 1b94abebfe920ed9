#!/bin/bash
# ncu evidence for the step kernels (run under gpurun, one GPU):
#   1. launch list with device times (cold-cache, serialised: compare shares)
#   2. one `--set full` capture of the step kernel per workload
# usage: [BENCH_EXTRA="--dtype f64 --scheme aa"] bash profiles/profile.sh <tag> [workload ...]
# then: python profiles/summarize_ncu.py <tag> [--dtype ..] [--scheme ..] [workload ...]
set -u
TAG=${1:-r01}; shift || true
WLS=${@:-channel512}
mkdir -p gpurun_out
for W in $WLS; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
      --log-file gpurun_out/launches_${TAG}_${W}.csv \
      python bench.py --workload $W --steps 5 --warmup 3 --no-cpu --no-e2e --no-sparse ${BENCH_EXTRA:-} > /dev/null 2>&1
  # one step-kernel launch after 600 steps: the flow has reached the whole
  # domain (early steps are mostly fluid at rest, whose zero momenta take
  # cheaper arithmetic paths)
  LBM_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:k_step -s 600 -c 1 \
      -o gpurun_out/prof_${TAG}_${W} -f \
      python bench.py --workload $W --steps 2 --warmup 600 --no-cpu --no-e2e --no-sparse ${BENCH_EXTRA:-} > gpurun_out/ncu_${TAG}_${W}.log 2>&1
  # export the raw page and the source-line hot spots; keep the .ncu-rep only
  # for the first workload (gpurun copies back at most 64 MiB)
  ncu -i gpurun_out/prof_${TAG}_${W}.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_${W}.csv 2>/dev/null
  if [ "$W" != "${WLS%% *}" ]; then rm -f gpurun_out/prof_${TAG}_${W}.ncu-rep; fi
done
