# shared-memory tile staging (variant 6) vs direct (0): parity + A/B + L2 traffic
set -u
mkdir -p gpurun_out
LBM_STEP_VARIANT=6 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tile" > gpurun_out/pytest_smem.log 2>&1; echo "exit $?" >> gpurun_out/pytest_smem.log
for W in porous512@0.1 porous512@0.2 porous512@0.5 porous512@0.9 vascular1024; do
timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --variants "0,6,0,6" >> gpurun_out/smem.txt 2>&1
done
for V in 0 6; do
LBM_STEP_VARIANT=$V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/smem_$V.csv python bench.py --workload porous512 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
