#!/bin/bash
# compute-sanitizer memcheck over the fill-based default tile (4x4x4 work
# list, AB; the A-A default) and the slab default-tile test.
set -u
mkdir -p gpurun_out
S="compute-sanitizer --error-exitcode 9 --print-limit 20"
timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q -k "default_tile_kernel_choice" > gpurun_out/san_deftile_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san_deftile_memcheck.log
timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_halo.py -x -q -k "default_tile_on_slabs" > gpurun_out/san_deftile_slabs_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san_deftile_slabs_memcheck.log
