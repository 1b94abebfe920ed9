"""DRAM fetch-granularity estimate for the sparse tile layout (design aid):
reads of the live-brick sectors if DRAM/L2 fetch whole 64-B or 128-B
granules of each (tile, direction) block.  python profiles/model/line_granularity.py"""
import sys; import os; R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, 'profiles', 'model'))
import numpy as np, paper_2108_13241_b200 as lb
from l2_model import build_items
for phi in (0.1, 0.2, 0.5):
    geom = lb.build_porous_random(512, phi, seed=0, radius_range=(4, 32))
    ns = geom.descriptors.type_tag != 0
    ex,ey,ez=4,8,16
    gz,gy,gx = 512//ez,512//ey,512//ex
    bx,by,bz=ex//2,ey//2,ez//2
    live = ns.reshape(gz, bz, 2, gy, by, 2, gx, bx, 2).any(axis=(2, 5, 8)).transpose(0,2,4,1,3,5).reshape(gz,gy,gx,bz*by*bx)
    keep = live.any(axis=3)
    lt = live[keep]
    nlive = lt.sum()
    for gran in (2,4):
        g = lt.reshape(lt.shape[0], -1, gran)
        chunks = g.any(axis=2).sum()
        print(phi, gran*32, "B granules: fetched", chunks*gran*19*32/1e9, "GB vs live", nlive*19*32/1e9)
