"""INTEGRATION.md Option A timed: the unmodified reference's render()
(baseline/_ref) with its kernel module swapped for
paper_2504_06598_b200.kernels, at C3-target (1M SH-3, 1080p, 1 spp), beside
our own render().  The reference's SAH tree comes from the oracle's C build
(bitwise the reference's bvh.build).   python tools/time_option_a.py"""
import importlib
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/srt_numba_cache")
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2504_06598_b200 import RenderSettings as Settings  # noqa: E402
from paper_2504_06598_b200 import kernels as gpu_kernels  # noqa: E402
from paper_2504_06598_b200 import render as our_render  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

sr = importlib.import_module("splatray.render")
sr.kernels = gpu_kernels
from splatray.bvh import Bvh  # noqa: E402
from splatray.config import RenderSettings  # noqa: E402
from splatray.synthetic import front_camera, random_cloud  # noqa: E402

f = (1e4 / 1e6) ** (1 / 3)
ref_asset = random_cloud(1_000_000, seed=0, scale_range=(0.02 * f, 0.25 * f), sh_degree=3)
ours = density_cloud(1_000_000)
lo, hi = ref_asset.aabb_arrays(RenderSettings().cutoff_s)
ob = O.sah_build(lo, hi)
bvh = Bvh(ob.node_lo, ob.node_hi, ob.node_left, ob.node_right, ob.node_count, ob.prim_order, ob.prim_lo, ob.prim_hi, 4)
st = RenderSettings(width=1920, height=1080, spp=1)


def timed(name, fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ms = float(np.median(ts)) * 1e3
    print(f"{name:58s} {ms:8.2f} ms  {1920 * 1080 / ms / 1e3:8.1f} Mrays/s", flush=True)


timed("reference render() with the kernels shim (Option A)", lambda: sr.render(ref_asset, front_camera(), st, bvh=bvh))
timed("paper_2504_06598_b200.render()", lambda: our_render(ours, front_camera(), Settings(width=1920, height=1080, spp=1)))
