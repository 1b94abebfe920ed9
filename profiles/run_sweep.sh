# porosity sweep (C3) x step-kernel variant, in-process A/B (one B200)
set -u
mkdir -p gpurun_out
for W in porous512@0.1 porous512@0.2 porous512@0.3 porous512@0.5 porous512@0.7 porous512@0.9 vascular1024; do
timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --variants "0,3,4,0" >> gpurun_out/sweep.txt 2>&1
done
timeout 900 python bench.py --workload channel512 --steps 200 --warmup 20 --variants "0,1,0" >> gpurun_out/sweep.txt 2>&1
for V in 0 4; do
LBM_STEP_VARIANT=$V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/launches_sweep_$V.csv python bench.py --workload porous512@0.2 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
