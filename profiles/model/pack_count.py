"""128-B lines per direction touched by 4x4x4 tiles at phi = 0.1 / 0.2, as stored
and with each tile's live bricks packed to the front."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
import bench
for w in ('porous512@0.1','porous512@0.2'):
    g,*_=bench.build_workload(w); live=g.descriptors.type_tag!=0
    nz,ny,nx=live.shape
    B=live.reshape(nz//2,2,ny//2,2,nx//2,2).any(axis=(1,3,5))
    T=B.reshape(B.shape[0]//2,2,B.shape[1]//2,2,B.shape[2]//2,2)   # 4x4x4 tiles: (tz,bz,ty,by,tx,bx)
    cnt=T.sum(axis=(1,3,5))
    lines_now=T.any(axis=(3,5)).sum()          # per tile: line = bz half
    lines_pack=np.ceil(cnt/4).sum()
    print(w, 'lines now', int(lines_now), 'packed', int(lines_pack), 'read GB now %.3f packed %.3f' % (lines_now*19*128/1e9, lines_pack*19*128/1e9))
