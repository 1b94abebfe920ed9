# warp work-list tile kernel (variant 5) vs per-tile CTAs (variant 0)
set -u
mkdir -p gpurun_out
LBM_STEP_VARIANT=5 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tile" > gpurun_out/pytest_w.log 2>&1; echo "exit $?" >> gpurun_out/pytest_w.log
for W in porous512@0.1 porous512@0.2 porous512@0.5 porous512@0.9 vascular1024; do
timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --variants "0,5,0,5" >> gpurun_out/wl.txt 2>&1
done
for V in 0 5; do
LBM_STEP_VARIANT=$V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/wl_$V.csv python bench.py --workload porous512@0.2 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
