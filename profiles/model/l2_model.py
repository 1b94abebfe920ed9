"""Sector-level L2 model of the sparse tile step (design aid, not a test).

Replays the DRAM-relevant accesses of the warp work-list kernel
(k_step_tiles_w, exact per-link select) over a geometry: items in launch
order, per item the unique 32-B sectors its loads touch (one warp
instruction per direction) and the 19 full sectors per live brick it stores.
A sector read misses L2 when more than `window` bytes of distinct-ish
traffic passed since its previous access (LRU approximated by a reuse
window).  Prints modelled DRAM read bytes against the live-brick minimum.

    python profiles/model/l2_model.py porous512@0.1 [--window-mb 100] [--tile 4,8,16]
"""
import argparse
import os
import sys

import numpy as np
from numba import njit

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

CX = np.array([0, 1, 0, -1, 0, 1, -1, -1, 1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0])
CY = np.array([0, 0, 1, 0, -1, 1, 1, -1, -1, 0, 0, 0, 0, 0, 0, 1, -1, -1, 1])
CZ = np.array([0, 0, 0, 0, 0, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 1, -1])
OPP = np.array([0, 3, 4, 1, 2, 7, 8, 5, 6, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17])


@njit(cache=True)
def replay(ns, rank, tiles, items_t, items_b, items_n, ex, ey, ez, window_sectors, nbr_sector_base):
    """ns: (nz,ny,nx) bool non-solid. Returns (dram_read_sectors, read_accesses, write_sectors)."""
    nz, ny, nx = ns.shape
    gz, gy, gx = rank.shape
    bx, by, bz = ex // 2, ey // 2, ez // 2
    nbrick = bx * by * bz
    T = tiles.shape[0]
    last = np.full(T * 19 * nbrick, -(1 << 62), dtype=np.int64)
    clock = 0
    miss = 0
    reads = 0
    writes = 0
    touched = np.empty(32 * 19, dtype=np.int64)
    for it in range(items_t.shape[0]):
        t = items_t[it]
        tx, ty, tz = tiles[t, 0], tiles[t, 1], tiles[t, 2]
        for i in range(19):
            nt = 0
            for k in range(items_n[it]):
                b = items_b[it, k]
                bxi = b % bx
                byi = (b // bx) % by
                bzi = b // (bx * by)
                for q in range(8):
                    x = tx * ex + bxi * 2 + (q & 1)
                    y = ty * ey + byi * 2 + ((q >> 1) & 1)
                    z = tz * ez + bzi * 2 + (q >> 2)
                    if x >= nx or y >= ny or z >= nz or not ns[z, y, x]:
                        continue
                    ux, uy, uz = x - CX[i], y - CY[i], z - CZ[i]
                    present = (0 <= ux < nx) and (0 <= uy < ny) and (0 <= uz < nz) and ns[uz, uy, ux]
                    if i == 0 or not present:
                        d = i if i == 0 else OPP[i]
                        sec = (t * 19 + d) * nbrick + b
                    else:
                        ut = rank[uz // ez, uy // ey, ux // ex]
                        lb = ((ux % ex) // 2) + bx * (((uy % ey) // 2) + by * ((uz % ez) // 2))
                        sec = (ut * 19 + i) * nbrick + lb
                    dup = False
                    for m in range(nt):
                        if touched[m] == sec:
                            dup = True
                            break
                    if not dup:
                        touched[nt] = sec
                        nt += 1
            for m in range(nt):
                sec = touched[m]
                reads += 1
                if clock - last[sec] > window_sectors:
                    miss += 1
                last[sec] = clock
                clock += 1
        # stores: 19 full sectors per live brick (post buffer: capacity only)
        w = 19 * items_n[it]
        writes += w
        clock += w
    return miss, reads, writes


def build_items(ns, ex, ey, ez, order="rank"):
    nz, ny, nx = ns.shape
    gx, gy, gz = -(-nx // ex), -(-ny // ey), -(-nz // ez)
    pad = np.zeros((gz * ez, gy * ey, gx * ex), dtype=bool)
    pad[:nz, :ny, :nx] = ns
    keep = pad.reshape(gz, ez, gy, ey, gx, ex).any(axis=(1, 3, 5))
    rank = np.full((gz, gy, gx), -1, dtype=np.int64)
    rank[keep] = np.arange(int(keep.sum()))
    kz, ky, kx = np.nonzero(keep)
    tiles = np.stack([kx, ky, kz], axis=1)
    # live bricks per tile: (gz, bz, 2, gy, by, 2, gx, bx, 2)
    bx, by, bz = ex // 2, ey // 2, ez // 2
    live = pad.reshape(gz, bz, 2, gy, by, 2, gx, bx, 2).any(axis=(2, 5, 8))  # gz,bz,gy,by,gx,bx
    live = live.transpose(0, 2, 4, 1, 3, 5).reshape(gz, gy, gx, bz * by * bx)
    lt = live[kz, ky, kx]   # (T, nbrick) in brick order x-fastest
    its_t, its_b, its_n = [], [], []
    seq = range(len(tiles))
    for t in seq:
        bs = np.nonzero(lt[t])[0]
        for k in range(0, len(bs), 4):
            g = bs[k:k + 4]
            its_t.append(t)
            row = np.zeros(4, dtype=np.int64)
            row[:len(g)] = g
            its_b.append(row)
            its_n.append(len(g))
    return (rank, tiles, np.array(its_t), np.array(its_b), np.array(its_n), int(lt.sum()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--window-mb", type=float, default=100.0)
    ap.add_argument("--tile", default="4,8,16")
    a = ap.parse_args()
    import paper_2108_13241_b200 as lb
    phi = float(a.workload.split("@")[1]) if "@" in a.workload else 0.5
    if a.workload.startswith("porous"):
        geom = lb.build_porous_random(512, phi, seed=0, radius_range=(4, 32))
    else:
        geom = lb.build_vascular(1024, seed=0, fluid_fraction=0.05)
    ns = geom.descriptors.type_tag != 0
    ex, ey, ez = (int(v) for v in a.tile.split(","))
    rank, tiles, it_t, it_b, it_n, nlive = build_items(ns, ex, ey, ez)
    win = int(a.window_mb * 1e6 / 32)
    miss, reads, writes = replay(ns, rank, tiles, it_t, it_b, it_n, ex, ey, ez, win, 0)
    nons = int(ns.sum())
    alg = nons * 76
    print(f"{a.workload} tile {a.tile} window {a.window_mb} MB: non-solid {nons}, live bricks {nlive} "
          f"(fill {nons / (8 * nlive):.3f}), items {len(it_t)}")
    print(f"  DRAM read {miss * 32 / 1e9:.3f} GB (min live sectors {nlive * 19 * 32 / 1e9:.3f}, alg {alg / 1e9:.3f}); "
          f"L2 read requests {reads * 32 / 1e9:.3f} GB; writes {writes * 32 / 1e9:.3f} GB")


if __name__ == "__main__":
    main()
