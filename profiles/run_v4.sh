# 128-bit dense kernel (variant 8) vs scalar (0): parity + A/B + ncu
set -u
mkdir -p gpurun_out
LBM_STEP_VARIANT=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_aa.py -x -q -k "dense or cavity or box or uniform or perturbed or launch or poiseuille or duct or ghia" > gpurun_out/pytest_v4.log 2>&1; echo "exit $?" >> gpurun_out/pytest_v4.log
timeout 900 python bench.py --workload channel512 --steps 300 --warmup 20 --variants "0,8,0,8" > gpurun_out/v4.txt 2>&1
timeout 900 python bench.py --workload channel512 --steps 1000 --warmup 100 --variants "0,8,0,8" >> gpurun_out/v4.txt 2>&1
for V in 0 8; do
LBM_STEP_VARIANT=$V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/v4_$V.csv python bench.py --workload channel512 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
