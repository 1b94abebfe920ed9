set -u
mkdir -p gpurun_out
for W in vascular1024 porous512@0.1; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -s 20 -c 4 --csv \
    --log-file gpurun_out/launches_aa_${W}_r02ap.csv \
    python bench.py --workload $W --scheme aa --steps 4 --warmup 20 --no-cpu --no-e2e --no-sparse > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -s 20 -c 2 --csv \
    --log-file gpurun_out/launches_ab_${W}_r02ap.csv \
    python bench.py --workload $W --steps 2 --warmup 20 --no-cpu --no-e2e --no-sparse > /dev/null 2>&1
done
