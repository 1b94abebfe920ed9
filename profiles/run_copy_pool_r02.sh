#!/bin/bash
# Persistent copy workers (default) vs a thread spawn per staging chunk
# (LBM_COPY_POOL=0), alternating processes: e2e phases of the driver's
# command with the library's readback breakdown; then the readback / halo /
# binding tests that go through the staged copies.
set -u
TAG=${1:-r02ax}
mkdir -p gpurun_out
for rep in 1 2 3; do
  for P in 1 0; do
    LBM_COPY_POOL=$P LBM_TIMING=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-sparse \
      2> gpurun_out/cp_${TAG}_${P}_${rep}.err | grep "^{" | sed "s/^{/{\"pool\": $P, /" >> gpurun_out/copy_pool_${TAG}.txt
    grep "readback:" gpurun_out/cp_${TAG}_${P}_${rep}.err | sed "s/^/pool=$P /" >> gpurun_out/copy_pool_${TAG}.log
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py tests/test_gpu_reference_binding.py tests/test_gpu_fullsize.py::test_c2_channel512_bitwise_vs_oracle -x -q > gpurun_out/copy_pool_tests_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/copy_pool_tests_${TAG}.log
