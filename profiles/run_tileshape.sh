# tile shape sweep on the sparse workloads (in-process, one B200)
set -u
mkdir -p gpurun_out
for W in porous512@0.2 porous512@0.5 vascular1024; do
for T in 8,8,8 8,4,16 4,4,32 16,4,8 8,8,4 16,8,4 4,8,16; do
timeout 600 python bench.py --workload $W --steps 200 --warmup 20 --tile $T --variants "0" >> gpurun_out/tileshape.txt 2>&1
done
done
