"""Read bytes of the phi = 0.1 step predicted for 32/64/128-B DRAM granules
(live 2x2x2 bricks per granule, 19 directions; sparse_r02.md)."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
import bench
g,*_=bench.build_workload('porous512@0.1'); live=g.descriptors.type_tag!=0
nz,ny,nx=live.shape
B=live.reshape(nz//2,2,ny//2,2,nx//2,2).any(axis=(1,3,5))   # (bz,by,bx)
lb=B.sum(); print('live bricks',lb, 'sector floor read GB', lb*19*32/1e9)
# 64-B granule = x pair of bricks (tile 2 bricks wide in x)
g64=B.reshape(B.shape[0],B.shape[1],B.shape[2]//2,2).any(axis=3).sum()
print('64B granules', g64, 'read GB', g64*19*64/1e9)
# 128-B granule = 2x2 (bx,by) bricks at one bz inside a 4x4x4 tile
g128=B.reshape(B.shape[0],B.shape[1]//2,2,B.shape[2]//2,2).any(axis=(2,4)).sum()
print('128B granules', g128, 'read GB', g128*19*128/1e9)
# alternative orders for 64B: y pairs, z pairs
gy=B.reshape(B.shape[0],B.shape[1]//2,2,B.shape[2]).any(axis=2).sum(); print('64B y-pairs read GB', gy*19*64/1e9)
gz=B.reshape(B.shape[0]//2,2,B.shape[1],B.shape[2]).any(axis=1).sum(); print('64B z-pairs read GB', gz*19*64/1e9)
