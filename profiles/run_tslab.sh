set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_halo.py -x -q > gpurun_out/pytest_tslab.log 2>&1; echo "exit $?" >> gpurun_out/pytest_tslab.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_all2.log
timeout 600 python bench.py --workload porous512 --steps 200 --warmup 20 --variants "0,0" > gpurun_out/tslab_bench.txt 2>&1
