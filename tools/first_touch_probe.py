"""First-touch cost of fresh pageable output arrays (the reference's
render() allocates np.zeros per call): plain 4 KB faults vs madvise(MADV_HUGEPAGE)
before the first write.    python tools/first_touch_probe.py"""
import ctypes
import mmap
import time

import numpy as np

print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      "defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
N = 1080 * 1920 * 3
src = np.random.default_rng(0).random(N)
for advise in (False, True, False, True):
    ts = []
    for _ in range(5):
        a = np.zeros(N)
        t0 = time.perf_counter()
        if advise:
            p = a.ctypes.data
            lo = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
            hi = (p + a.nbytes) & ~((2 << 20) - 1)
            if hi > lo:
                libc.madvise(lo, hi - lo, 14)  # MADV_HUGEPAGE
        np.copyto(a, src)
        ts.append(time.perf_counter() - t0)
        del a
    print(f"madvise={advise}: first-touch copy of {N * 8 / 1e6:.0f} MB: median {sorted(ts)[2] * 1e3:.2f} ms")
