# tile launch order: rank vs z-groups of B tile layers (x/y streaming kept)
set -u
mkdir -p gpurun_out
for W in porous512@0.2 porous512@0.5 vascular1024; do
timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --variants "LBM_TILE_ORDER=row,LBM_TILE_ORDER=z:2,LBM_TILE_ORDER=z:4,LBM_TILE_ORDER=z:8,LBM_TILE_ORDER=row" >> gpurun_out/zgroup.txt 2>&1
for O in row z:2 z:4; do
LBM_TILE_ORDER=$O ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/zg_${W}_$O.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
done
LBM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/multi2.json 2> gpurun_out/multi2.err
