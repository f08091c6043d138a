"""render() output buffers and the mapped-store e2e time: one page-locked
buffer reused vs two alternating (a loop that holds the previous frame), and
cudaHostAlloc blocks vs 2 MB-page (THP) anonymous memory registered with
srt_host_register.    python tools/e2e_pool_probe.py"""
import ctypes
import mmap
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06598_b200 import RenderSettings, _lib, front_camera  # noqa: E402
from paper_2504_06598_b200.render import _PINNED, prepare  # noqa: E402
from paper_2504_06598_b200.scene import camera_tuple  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

W, H = 1920, 1080
st = RenderSettings(width=W, height=H, spp=1)
sc = prepare(density_cloud(1_000_000), st)
ct = camera_tuple(front_camera(), W, H)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
S2 = st.cutoff_s ** 2


def huge(shape):
    nbytes = int(np.prod(shape)) * 8
    size = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    mm = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(mm))
    off = (-base) % (2 << 20)
    try:
        mm.madvise(mmap.MADV_HUGEPAGE, off, size)
    except Exception as e:  # noqa: BLE001
        print("madvise failed", e)
    arr = np.frombuffer(mm, dtype=np.float64, count=nbytes // 8, offset=off).reshape(shape)
    arr.fill(0.0)
    _lib.check(_lib.load().srt_host_register(ctypes.c_void_p(arr.ctypes.data), arr.nbytes))
    return arr, mm


def run(bufs, reps=30):
    ts = []
    for i in range(reps + 2):
        rgb, op = bufs[i % len(bufs)]
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc.render(ct, W, H, 1, 1, 0, S2, True, st.seed, st.background, out_rgb=rgb, out_op=op)
        if i >= 2:
            ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, min(ts) * 1e3


pin = [(_PINNED.array((H, W, 3)), _PINNED.array((H, W))) for _ in range(3)]
hp = [(huge((H, W, 3))[0], huge((H, W))[0]) for _ in range(3)]
for name, bufs in [("cudaHostAlloc x1", pin[:1]), ("cudaHostAlloc x2", pin[:2]), ("cudaHostAlloc x3", pin),
                   ("THP registered x1", hp[:1]), ("THP registered x2", hp[:2]), ("THP registered x3", hp),
                   ("cudaHostAlloc x1", pin[:1]), ("cudaHostAlloc x2", pin[:2])]:
    med, mn = run(bufs)
    print(f"{name:22s} median {med:.3f} ms  min {mn:.3f} ms", flush=True)
