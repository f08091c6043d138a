"""Generate tests/golden/*.npz from the UNMODIFIED reference (run in the build
container, where /root/reference exists; the fixtures travel, the reference
does not).  TEST INFRASTRUCTURE.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden.py

Every fixture is produced by the reference's own public functions:
sampling.hash_position / pixel_jitter, synthetic.random_cloud, assets.packed
/ aabb_arrays, bvh.build, kernels.trace_batch / transmittance_batch /
render_stochastic (via render.render).
"""

from __future__ import annotations

import hashlib
import importlib
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from splatray import kernels, sampling, synthetic
    from splatray import bvh as B
    from splatray.config import RenderSettings

    R = importlib.import_module("splatray.render")
    OUT.mkdir(parents=True, exist_ok=True)
    tmax = float(np.finfo(np.float64).max)
    s = 2.0 * np.sqrt(2.0)

    # 1. randomness ------------------------------------------------------
    rng = np.random.default_rng(2024)
    pts = rng.uniform(-20, 20, size=(512, 3))
    slots = rng.integers(0, 8, size=512)
    hv = np.array([sampling.hash_position(p, int(k)) for p, k in zip(pts, slots)])
    jit_args = np.array([[px, py, f, sd] for px, py, f, sd in
                         zip(rng.integers(0, 4000, 256), rng.integers(0, 3000, 256), rng.integers(0, 5000, 256),
                             rng.integers(0, 100, 256))], dtype=np.int64)
    jit = np.array([sampling.pixel_jitter((a[0], a[1]), int(a[2]), int(a[3])) for a in jit_args])
    np.savez_compressed(OUT / "sampling.npz", points=pts, slots=slots, hash=hv, jitter_args=jit_args, jitter=jit)

    # 2. synthetic assets and packing (digests only; arrays are regenerated)
    digests = {}
    for name, kw in {"c1_10k_sh0": dict(n=10_000, seed=0, sh_degree=0),
                     "c2_100k_sh3_density": dict(n=100_000, seed=0, sh_degree=3,
                                                 scale_range=(0.02 * (0.1) ** (1 / 3), 0.25 * (0.1) ** (1 / 3))),
                     "small_400_s31": dict(n=400, seed=31)}.items():
        a = synthetic.random_cloud(**kw)
        pk = a.packed
        lo, hi = a.aabb_arrays(s)
        digests[name] = {"asset": _digest(a.means, a.rotations, a.scales, a.opacities, a.sh),
                         "packed": _digest(pk.means, pk.cov_inv6, pk.opacities, pk.sh),
                         "aabb": _digest(lo, hi)}
    np.savez_compressed(OUT / "assets.npz", **{f"{k}__{f}": np.array(v[f]) for k, v in digests.items() for f in v})

    # 3. BVH build (bvh.py:87-193) on a 3000-primitive SH3 cloud
    a = synthetic.random_cloud(3000, seed=3, sh_degree=3)
    lo, hi = a.aabb_arrays(s)
    b = B.build((lo, hi))
    np.savez_compressed(OUT / "bvh_3000.npz", lo=lo, hi=hi, node_lo=b.node_lo, node_hi=b.node_hi,
                        node_left=b.node_left, node_right=b.node_right, node_count=b.node_count,
                        prim_order=b.prim_order)

    # 4. explicit-ray traces (kernels.py:527-540), trig hash, both depth modes
    a = synthetic.random_cloud(400, seed=31)
    pk = a.packed
    bb = R.scene_bvh(a, s)
    rr = np.random.default_rng(1234)
    n = 600
    origins = rr.uniform(-3, 3, size=(n, 3))
    dirs = rr.normal(size=(n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    res = {}
    for mode in (0, 1):
        for ns in (1, 4):
            ot = np.empty((n, ns))
            oi = np.empty((n, ns), np.int64)
            kernels.trace_batch(*R._bvh_args(bb), pk.means, pk.cov_inv6, pk.opacities, origins, dirs, 0.0, tmax,
                                mode, s * s, True, ot, oi)
            res[f"t_m{mode}_n{ns}"] = ot
            res[f"id_m{mode}_n{ns}"] = oi
    tr = np.empty(n)
    kernels.transmittance_batch(*R._bvh_args(bb), pk.means, pk.cov_inv6, pk.opacities, origins, dirs, 0.0, tmax,
                                0, s * s, tr)
    np.savez_compressed(OUT / "trace_400.npz", origins=origins, dirs=dirs, transmittance=tr, **res)

    # 5. full-frame render (render.py:125-174 -> kernels.py:622-673)
    a = synthetic.random_cloud(300, seed=53, sh_degree=3)
    cam = synthetic.front_camera()
    st = RenderSettings(width=24, height=20, spp=6, multisample=2, seed=5, background=[0.1, 0.2, 0.3])
    buf = R.render(a, cam, st)
    st2 = RenderSettings(width=16, height=12, spp=3, seed=11, depth_mode="center")
    a2 = synthetic.anisotropic_sheets(60, seed=3)
    buf2 = R.render(a2, cam, st2)
    np.savez_compressed(OUT / "render_small.npz", rgb=buf.rgb, opacity=buf.opacity, spp=buf.spp,
                        rgb_center=buf2.rgb, opacity_center=buf2.opacity)

    # 6. configs[0] (C1): random_cloud(10k, seed 0, SH0) as-is, 64x64, 1 spp,
    #    and the same frame at 4 passes x N=2 with SH degree 3
    a = synthetic.random_cloud(10_000, seed=0, sh_degree=0)
    c1 = R.render(a, cam, RenderSettings(width=64, height=64, spp=1))
    a3 = synthetic.random_cloud(10_000, seed=0, sh_degree=3)
    c1b = R.render(a3, cam, RenderSettings(width=48, height=40, spp=8, multisample=2, seed=7,
                                           background=[0.05, 0.1, 0.2]))
    np.savez_compressed(OUT / "render_c1.npz", rgb=c1.rgb, opacity=c1.opacity,
                        rgb_ms=c1b.rgb, opacity_ms=c1b.opacity)

    # 7. exact compositing (kernels.py:584-604, 677-723)
    a = synthetic.random_cloud(500, seed=41, sh_degree=2)
    pk = a.packed
    bg = np.array([0.15, 0.25, 0.35])
    ex_rgb = np.empty((n, 3))
    ex_op = np.empty(n)
    kernels.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, origins, dirs, 0.0, tmax, 0,
                        s * s, bg[0], bg[1], bg[2], ex_rgb, ex_op)
    fr = R.render(a, cam, RenderSettings(width=20, height=16, spp=3, seed=2, reference_mode=True,
                                         background=bg))
    np.savez_compressed(OUT / "exact_500.npz", rgb=ex_rgb, opacity=ex_op, frame_rgb=fr.rgb, frame_opacity=fr.opacity,
                        frame_spp=fr.spp)

    # 8. PLY ingest (assets.py:257-370): files written by the reference and the
    #    arrays its loader returns for them
    from splatray.assets import load_ply, save_ply

    a = synthetic.random_cloud(300, seed=5, sh_degree=3)
    save_ply(a, OUT / "splats_300_sh3.ply", binary=True)
    b = synthetic.random_cloud(60, seed=6, sh_degree=1)
    save_ply(b, OUT / "splats_60_sh1_ascii.ply", binary=False)
    out = {}
    for tag, fname in (("bin", "splats_300_sh3.ply"), ("ascii", "splats_60_sh1_ascii.ply")):
        got = load_ply(OUT / fname)
        for f in ("means", "rotations", "scales", "opacities", "sh"):
            out[f"{tag}_{f}"] = getattr(got, f)
    np.savez_compressed(OUT / "ply_loaded.npz", **out)
    biased()
    print("golden fixtures written to", OUT)


def biased() -> None:
    """9. biased k-nearest composite (kernels.py:479-518, 561-580): the
    reference's `--compare-biased` baseline on the trace_400 rays."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from splatray import kernels, synthetic

    tmax = float(np.finfo(np.float64).max)
    s2 = 8.0
    t = np.load(OUT / "trace_400.npz")
    origins, dirs = t["origins"], t["dirs"]
    a = synthetic.random_cloud(500, seed=41, sh_degree=2)
    pk = a.packed
    bg = np.array([0.15, 0.25, 0.35])
    res = {}
    for mode in (0, 1):
        for kk in (1, 2, 5):
            out = np.empty((origins.shape[0], 3))
            kernels.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, origins, dirs, 0.0, tmax,
                                 mode, s2, kk, bg[0], bg[1], bg[2], out)
            res[f"rgb_m{mode}_k{kk}"] = out
    # the cli's frame-level baseline (cli.py:164-203) on a small frame
    from splatray import cli
    from splatray.config import RenderSettings

    cam = synthetic.front_camera()
    for kk in (1, 3):
        st = RenderSettings(width=20, height=16, spp=2, seed=5, background=bg)
        res[f"frame_k{kk}"] = cli._biased_frame(a, cam, st, kk)
    np.savez_compressed(OUT / "biased_500.npz", **res)


def c3target() -> None:
    """10. The headline workload at full scale, from the unmodified reference:
    density-preserving random_cloud(1M, SH3, f = (1e4/n)^(1/3)), its own SAH
    BVH, trace_batch ids/depths of the pass-0 camera rays of a 16-pixel grid
    of the 1920x1080 frame, and render()'s rgb/opacity on the same grid."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from splatray import kernels, synthetic
    from splatray.config import RenderSettings

    R = importlib.import_module("splatray.render")
    n = 1_000_000
    f = (1e4 / n) ** (1.0 / 3.0)
    a = synthetic.random_cloud(n, seed=0, scale_range=(0.02 * f, 0.25 * f), sh_degree=3)
    cam = synthetic.front_camera()
    st = RenderSettings(width=1920, height=1080, spp=1)
    bvh = R.scene_bvh(a, st.cutoff_s)
    xs, ys = np.meshgrid(np.arange(8, 1920, 16), np.arange(8, 1080, 16))
    rays = [R.generate_camera_ray(cam, st, (int(x), int(y)), 0) for x, y in zip(xs.ravel(), ys.ravel())]
    origins = np.array([r.origin for r in rays])
    dirs = np.array([r.direction for r in rays])
    pk = a.packed
    tmax = float(np.finfo(np.float64).max)
    out_t = np.empty((len(rays), 1))
    out_id = np.empty((len(rays), 1), np.int64)
    kernels.trace_batch(*R._bvh_args(bvh), pk.means, pk.cov_inv6, pk.opacities, origins, dirs, 0.0, tmax, 0,
                        st.cutoff_s ** 2, True, out_t, out_id)
    buf = R.render(a, cam, st, bvh=bvh)
    np.savez_compressed(OUT / "c3target_grid.npz", px=xs.ravel(), py=ys.ravel(), origins=origins, dirs=dirs,
                        t=out_t, id=out_id, rgb=buf.rgb[ys, xs].reshape(-1, 3), opacity=buf.opacity[ys, xs].ravel())


if __name__ == "__main__":
    if sys.argv[1:] == ["biased"]:
        biased()
    elif sys.argv[1:] == ["c3target"]:
        c3target()
    else:
        main()
