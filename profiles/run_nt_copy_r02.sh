#!/bin/bash
# Non-temporal host copy (default) vs plain memcpy (LBM_NT=0) for the staged
# transfers, alternating processes: e2e phases of the driver's command (C2,
# K = 20) with the library's readback breakdown; then the readback parity tests.
set -u
TAG=${1:-r02aw}
mkdir -p gpurun_out
for rep in 1 2 3; do
  for NT in 1 0; do
    LBM_NT=$NT LBM_TIMING=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-sparse \
      2> gpurun_out/nt_${TAG}_${NT}_${rep}.err | grep "^{" | sed "s/^{/{\"nt\": $NT, /" >> gpurun_out/nt_copy_${TAG}.txt
    grep "readback:" gpurun_out/nt_${TAG}_${NT}_${rep}.err | sed "s/^/nt=$NT /" >> gpurun_out/nt_copy_${TAG}.log
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py::test_c2_channel512_bitwise_vs_oracle -x -q > gpurun_out/nt_tests_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/nt_tests_${TAG}.log
