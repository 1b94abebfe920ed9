"""Host side of the readback (DESIGN §8 e2e): copy 4 x 1.07 GB out of a 64 MB
pinned slot into caller arrays with 16 threads -- fresh arrays (page faults,
with / without MADV_HUGEPAGE) vs arrays already faulted in -- to separate
fault-in cost from copy bandwidth."""
import ctypes
import mmap
import threading
import time

import numpy as np
import torch

N = 1 << 27            # f64 elements per field (512^3)
SLOT = 64 << 20
libc = ctypes.CDLL("libc.so.6")
src = torch.empty(SLOT, dtype=torch.uint8, pin_memory=True).numpy()
src[:] = 7


def advise(a):
    p = a.ctypes.data
    lo = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
    hi = (p + a.nbytes) & ~((2 << 20) - 1)
    libc.madvise(ctypes.c_void_p(lo), ctypes.c_size_t(hi - lo), 14)   # MADV_HUGEPAGE


def fill(dsts, nt=16):
    views = [d.view(np.uint8) for d in dsts]
    jobs = [(v, o) for v in views for o in range(0, v.size, SLOT)]

    def work(k):
        for j in range(k, len(jobs), nt):
            v, o = jobs[j]
            n = min(SLOT, v.size - o)
            np.copyto(v[o:o + n], src[:n])
    th = [threading.Thread(target=work, args=(k,)) for k in range(nt)]
    t0 = time.perf_counter()
    [t.start() for t in th]
    [t.join() for t in th]
    return time.perf_counter() - t0


for case in ("fresh", "fresh+thp", "prefaulted", "fresh+thp", "prefaulted"):
    dsts = [np.empty(N) for _ in range(4)]
    if "thp" in case:
        [advise(d) for d in dsts]
    if case == "prefaulted":
        fill(dsts)
    dt = fill(dsts)
    print(f"{case:12s} {4 * N * 8 / dt / 1e9:6.1f} GB/s ({dt * 1e3:.0f} ms)", flush=True)
    del dsts
