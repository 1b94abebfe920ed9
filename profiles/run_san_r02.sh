#!/bin/bash
# compute-sanitizer over the round-2 code paths (one B200): memcheck on the
# TMA kernel, the A-A tile slabs (peer stores into neighbour tile storage),
# the boundary-first / graph-replayed slabs and the reference-tile pipeline;
# racecheck + synccheck on the TMA kernel (shared memory + mbarrier ring).
set -u
mkdir -p gpurun_out
S="compute-sanitizer --error-exitcode 9 --print-limit 20"
LBM_STEP_VARIANT=9 timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise_vs_oracle and tile and 1" > gpurun_out/san_tma_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san_tma_memcheck.log
LBM_STEP_VARIANT=9 timeout 1500 $S --tool racecheck python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise_vs_oracle and tile and 1" > gpurun_out/san_tma_racecheck.log 2>&1; echo "exit $?" >> gpurun_out/san_tma_racecheck.log
LBM_STEP_VARIANT=9 timeout 1500 $S --tool synccheck python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise_vs_oracle and tile and 1" > gpurun_out/san_tma_synccheck.log 2>&1; echo "exit $?" >> gpurun_out/san_tma_synccheck.log
timeout 2400 $S --tool memcheck python -m pytest tests/test_gpu_halo.py -x -q -k "aa_tile_slabs and tile0 or slabs_in_process_bitwise and 2-False" > gpurun_out/san_slabs_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san_slabs_memcheck.log
timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_reference_tiles.py tests/test_gpu_aa.py -x -q -k "reference or bitwise_vs_oracle and 1" > gpurun_out/san_misc_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san_misc_memcheck.log
