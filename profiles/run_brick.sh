# in-tile order: 2x2x2 bricks (LBM_BRICK=1, default) vs x-rows (0), tile 8^3 and 4x8x16
set -u
mkdir -p gpurun_out
for W in porous512@0.2 porous512@0.5 porous512@0.9 vascular1024; do
for T in 8,8,8 4,8,16 16,8,4; do
timeout 900 python bench.py --workload $W --steps 200 --warmup 20 --tile $T --variants "LBM_BRICK=1,LBM_BRICK=0" >> gpurun_out/brick.txt 2>&1
done
done
