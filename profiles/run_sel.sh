# exact-select gathers without spills vs speculative (DRAM bytes + time)
set -u
mkdir -p gpurun_out
for W in porous512@0.2 porous512@0.5; do
timeout 600 python bench.py --workload $W --steps 200 --warmup 20 --variants "0,3,4,0" >> gpurun_out/sel.txt 2>&1
for V in 0 3 4; do
LBM_STEP_VARIANT=$V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/sel_${W}_$V.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
done
