"""Small workload touching every libsrt kernel, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_workload.py
    compute-sanitizer --tool racecheck python tools/sanitize_workload.py
    compute-sanitizer --tool synccheck python tools/sanitize_workload.py

Builds (PLOC, LBVH, upload), splat packing, fused and split frames (mapped
and pageable outputs, N = 1/2/4, both depth modes, odd widths), explicit rays
(counter, table, trig64; per lane and as packets), transmittance, exact and
biased composites (per lane and as packets), host arrays through the staging
ring.
"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])

import numpy as np

from paper_2504_06598_b200 import RenderSettings, front_camera, render, render_biased
from paper_2504_06598_b200.assets import SplatAsset
from paper_2504_06598_b200.render import PinnedPool
from paper_2504_06598_b200.scene import DeviceScene, camera_tuple
from paper_2504_06598_b200.synthetic import random_cloud, two_layer_scene

S2 = 8.0
TMAX = float(np.finfo(np.float64).max)


def main() -> None:
    a = random_cloud(2_000, seed=5, sh_degree=3)
    W, H = 40, 24
    cam = camera_tuple(front_camera(), W, H)
    pool = PinnedPool()
    for method in ("ploc", "lbvh"):
        sc = DeviceScene.from_packed(a.packed)
        sc.build_bvh(np.sqrt(S2), method=method)
        for mode in (0, 1):
            for nslots in (1, 2, 4):
                sc.render(cam, W, H, 2, nslots, mode, S2, True, 1, (0.1, 0.2, 0.3))
                sc.render(cam, W, H, 2, nslots, mode, S2, True, 1, (0.1, 0.2, 0.3), out_rgb=pool.array((H, W, 3)),
                          out_op=pool.array((H, W)), want_ids=True)
        rng = np.random.default_rng(1)
        o = rng.uniform(-3, 3, (300, 3))
        d = rng.normal(size=(300, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        sc.trace_rays(o, d, 0.0, TMAX, 0, S2, True, 2)
        sc.trace_rays(o, d, 0.0, TMAX, 1, S2, True, 1, rng="table", table=rng.uniform(size=(2_000, 1)))
        sc.trace_rays(o, d, 0.0, TMAX, 0, S2, True, 2, rng="trig64")
        sc.transmittance(o, d, 0.0, TMAX, 0, S2)
        sc.exact_rays(o, d, s2=S2)
        sc.render_exact(cam, W, H, 2, 0, S2, 3)
        for rng_name in ("counter", "trig64"):
            sc.biased_rays(o, d, 3, s2=S2, rng=rng_name)
            sc.render_biased(cam, W, H, 2, 2, 0, S2, rng=rng_name)
        sc.biased_rays(o, d, 2, s2=S2, rng="table", table=np.zeros(2_000))
        # one-hemisphere batches of >= 4096 rays: the packet routes (trace,
        # transmittance, exact and biased composites; distinct origins sorted)
        hd = rng.normal(size=(5000, 3)) * [0.2, 0.2, 0.0] + [0.0, 0.0, 1.0]
        hd /= np.linalg.norm(hd, axis=1, keepdims=True)
        ho = rng.uniform(-1, 1, (5000, 3)) * [1, 1, 0] + [0, 0, -4]
        sc.trace_rays(ho, hd, 0.0, TMAX, 0, S2, True, 1)
        sc.transmittance(ho, hd, 0.0, TMAX, 0, S2)
        sc.exact_rays(ho, hd, s2=S2)
        for kk in (1, 4, 12):
            sc.biased_rays(ho, hd, kk, s2=S2)
        sc.biased_rays(ho, hd, 3, s2=S2, rng="table", table=rng.uniform(size=2_000))
        sc.render_biased(cam, W, H, 12, 2, 0, S2)
        # odd width: partial packets store the f64 frame per lane
        cam_odd = camera_tuple(front_camera(), 37, 23)
        sc.render(cam_odd, 37, 23, 1, 1, 0, S2, True, 1, (0.1, 0.2, 0.3), out_rgb=pool.array((23, 37, 3)),
                  out_op=pool.array((23, 37)))
        sc.close()
    # host arrays above 2 MB: the page-locked staging ring
    big = DeviceScene.from_packed(a.packed)
    big.build_bvh(np.sqrt(S2))
    bo = np.random.default_rng(2).uniform(-3, 3, (120_000, 3))
    bd = np.random.default_rng(3).normal(size=(120_000, 3))
    bd /= np.linalg.norm(bd, axis=1, keepdims=True)
    big.trace_rays(bo, bd, 0.0, TMAX, 0, S2, True, 1)
    big.close()
    # raw splats packed on the GPU, and a scene from the reference's own BVH layout
    sp = DeviceScene.from_splats(a)
    sp.build_bvh(np.sqrt(S2))
    sp.render(cam, W, H, 1, 1, 0, S2, True, 0, (0.0, 0.0, 0.0))
    sp.close()
    # the closest-hit walks' split tree (>= 16,384 primitives), with a few
    # degenerate primitives whose unbounded boxes land in every cell
    from paper_2504_06598_b200.synthetic import density_cloud

    pk = density_cloud(20_000, seed=2).packed
    cov = pk.cov_inv6.copy()
    cov[::4001] = 0.0
    sp2 = DeviceScene(pk.means, cov, pk.opacities, pk.sh, pk.sh_degree)
    sp2.build_bvh(np.sqrt(S2))
    assert sp2.split_info()["num_refs"] >= 20_000
    for nslots in (1, 4):
        sp2.render(cam, W, H, 1, nslots, 0, S2, True, 0, (0.0, 0.0, 0.0), out_rgb=pool.array((H, W, 3)),
                   out_op=pool.array((H, W)))
        sp2.render(cam, W, H, 3, nslots, 1, S2, True, 0, (0.0, 0.0, 0.0), want_ids=True)
    sp2.trace_rays(o, d, 0.0, TMAX, 0, S2, True, 1)
    sp2.trace_rays(o, d, 0.0, TMAX, 0, S2, True, 4)
    sp2.trace_rays(ho, hd, 0.0, TMAX, 0, S2, True, 2)
    sp2.trace_rays(o, d, 0.0, TMAX, 0, S2, True, 2, rng="trig64")
    sp2.close()
    t = two_layer_scene()
    render(t, front_camera(), RenderSettings(width=16, height=16, spp=2))
    render(t, front_camera(), RenderSettings(width=16, height=16, spp=2, reference_mode=True))
    render_biased(t, front_camera(), RenderSettings(width=16, height=16, spp=1), 1)
    one = SplatAsset(means=np.zeros((1, 3)), rotations=np.array([[1.0, 0, 0, 0]]), scales=np.full((1, 3), 0.3),
                     opacities=np.array([0.5]), sh=np.zeros((1, 3, 1)))
    render(one, front_camera(), RenderSettings(width=8, height=8, spp=1))
    from paper_2504_06598_b200 import _lib

    print("sanitize workload ok,", getattr(_lib.load(), "_name", "?"))


if __name__ == "__main__":
    main()
