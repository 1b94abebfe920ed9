# tile launch order: rank (row) vs y-pencils of B rows vs Morton -- time and DRAM bytes
set -u
mkdir -p gpurun_out
for W in porous512@0.2 porous512@0.5 vascular1024; do
timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --variants "LBM_TILE_ORDER=row,LBM_TILE_ORDER=pencil:2,LBM_TILE_ORDER=pencil:4,LBM_TILE_ORDER=pencil:8,LBM_TILE_ORDER=pencil:16,LBM_TILE_ORDER=row" >> gpurun_out/pencil.txt 2>&1
for O in row pencil:4 pencil:8; do
LBM_TILE_ORDER=$O ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -c 1 --csv --log-file gpurun_out/pencil_${W}_$O.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
done
