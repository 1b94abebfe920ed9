set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_e2e.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_e2e.log
python profiles/e2e_phases.py > gpurun_out/e2e_phases2.txt 2>&1
timeout 1500 python bench.py --workload c5 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
