set -u
mkdir -p gpurun_out
free -g > gpurun_out/free.txt 2>&1; nproc >> gpurun_out/free.txt
timeout 900 python -m pytest tests/test_gpu_aa.py -x -q > gpurun_out/pytest_aa.log 2>&1; echo "exit $?" >> gpurun_out/pytest_aa.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_all.log
for W in channel512 porous512 vascular1024; do
  timeout 600 python bench.py --workload $W --steps 300 --warmup 20 --variants "LBM_GRAPH=1" --scheme aa > gpurun_out/ab_aa_$W.txt 2>&1
  timeout 600 python bench.py --workload $W --steps 300 --warmup 20 --variants "LBM_GRAPH=1" --scheme ab >> gpurun_out/ab_aa_$W.txt 2>&1
done
timeout 1500 python bench.py --workload c5 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
