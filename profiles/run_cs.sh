# streaming (evict-first) stores of the post buffer, A/B in process
set -u
mkdir -p gpurun_out
for W in channel512 porous512@0.2 porous512 vascular1024; do
timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --variants "LBM_STORE_CS=0,LBM_STORE_CS=1,LBM_STORE_CS=0,LBM_STORE_CS=1" >> gpurun_out/cs.txt 2>&1
done
for C in 0 1; do
LBM_STORE_CS=$C ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/cs_$C.csv python bench.py --workload porous512 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
