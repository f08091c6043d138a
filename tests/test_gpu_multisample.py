"""multisample N > 8 (the reference allows N <= 256: config.py:18,79-80, the
slot loop of kernels.py:353-364) through frames and explicit rays, and frames
whose (pixel, pass) work items exceed one persistent launch.

A walk holds at most 8 slots; N > 8 runs as ceil(N/8) walks of <= 8 slots
over the same ray, slot 8 g + k drawing sample pass * N + 8 g + k (the trig64
walk uses groups of 16, hashing slot index 16 g + k).  Every
slot is independent (the clip culls only beyond the farthest slot bound), so
the split reproduces the N-slot walk of the reference exactly.
"""

import numpy as np
import pytest

from conftest import CUTOFF, S2, TMAX, random_rays

pytestmark = pytest.mark.gpu

ID_AGREE = 0.999


def _oracle_bvh(O, asset):
    lo, hi = asset.aabb_arrays(CUTOFF)
    return O.sah_build(lo, hi)


@pytest.mark.parametrize("spp,nslots", [(64, 64), (256, 256), (40, 20)])
def test_render_multisample_beyond_16_vs_oracle(oracle, spp, nslots):
    """render() with N = 20, 64, 256: slot ids of pass 0 and the frame means
    against the counter-mode oracle."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, render
    from paper_2504_06598_b200.render import prepare
    from paper_2504_06598_b200.scene import camera_tuple
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(4_000, seed=11, sh_degree=2)
    w, h = 40, 24
    st = RenderSettings(width=w, height=h, spp=spp, multisample=nslots, seed=3, background=[0.1, 0.0, 0.2])
    buf = render(a, front_camera(), st)
    assert buf.spp == st.passes * nslots
    sc = prepare(a, st)
    ct = camera_tuple(front_camera(), w, h)
    _, _, ids = sc.render(ct, w, h, 1, nslots, 0, S2, True, st.seed, st.background, want_ids=True)
    pk = a.packed
    ref = oracle.render(_oracle_bvh(oracle, a), pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree,
                        np.array(ct), w, h, passes=st.passes, nslots=nslots, s2=S2, seed=st.seed, rng="counter",
                        background=st.background)
    ref1 = oracle.render(_oracle_bvh(oracle, a), pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree,
                         np.array(ct), w, h, passes=1, nslots=nslots, s2=S2, seed=st.seed, rng="counter",
                         background=st.background, want_ids=True)
    agree = np.mean(ids == ref1["ids"])
    assert agree >= ID_AGREE, agree
    ok = np.all(np.abs(buf.rgb - ref["rgb"]) <= 1e-5 * np.abs(ref["rgb"]) + 1e-6, axis=2)
    ok &= np.abs(buf.opacity - ref["opacity"]) <= 1e-12
    assert ok.mean() >= 0.99, ok.mean()


def test_single_pass_multisample_beyond_16_mapped_and_device_paths_agree():
    """One pass of N = 48 slots: the fused per-pass path (first/last group
    flags, mapped f64 store on the last group) equals the one-launch
    fixed-point frame up to fp32 summation rounding."""
    import torch

    from paper_2504_06598_b200 import front_camera
    from paper_2504_06598_b200.render import PinnedPool
    from paper_2504_06598_b200.scene import DeviceScene, camera_tuple, make_camera, make_render_params, shard_tiles
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(3_000, seed=5, sh_degree=1)
    sc = DeviceScene.from_packed(a.packed)
    sc.build_bvh(CUTOFF)
    W, H, N = 56, 40, 48
    ct = camera_tuple(front_camera(), W, H)
    pool = PinnedPool()
    rgb_m, op_m, _ = sc.render(ct, W, H, 1, N, 0, S2, True, 2, (0.0, 0.0, 0.0), out_rgb=pool.array((H, W, 3)),
                               out_op=pool.array((H, W)))
    rgb_c, op_c, _ = sc.render(ct, W, H, 1, N, 0, S2, True, 2, (0.0, 0.0, 0.0))
    np.testing.assert_array_equal(rgb_m, rgb_c)
    np.testing.assert_array_equal(op_m, op_c)
    prm = make_render_params(W, H, 1, N, 0, S2, True, 2)
    acc64 = torch.empty((shard_tiles(W, H) * 256, 4), dtype=torch.int64, device="cuda")
    out = torch.zeros((W * H, 4), device="cuda")
    sc.render_frame_device(make_camera(ct), prm, acc64.data_ptr(), out.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(H, W, 4)
    np.testing.assert_allclose(o[..., :3], rgb_c, rtol=2e-6, atol=2e-6)
    np.testing.assert_allclose(o[..., 3], op_c, rtol=2e-6, atol=2e-6)
    assert op_c.max() > 0


@pytest.mark.parametrize("rng", ["table", "trig64"])
def test_trace_batch_beyond_16_slots_table_and_trig64(oracle, rng):
    """Explicit rays with N = 20 slots under scripted uniforms (table columns
    8 g + k) and under the reference's own trig-hash draw (slot index 16 g + k
    in the hash, kernels.py:354)."""
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(3_000, seed=8, sh_degree=0)
    pk = a.packed
    o, d = random_rays(np.random.default_rng(4), 3_000)
    N = 20
    table = np.random.default_rng(5).uniform(size=(3_000, N)) if rng == "table" else None
    sc = DeviceScene.from_packed(pk)
    sc.build_bvh(CUTOFF)
    t, ids = sc.trace_rays(o, d, 0.0, TMAX, 0, S2, True, N, rng=rng, table=table)
    sc.close()
    ot, oid = oracle.trace_batch(_oracle_bvh(oracle, a), pk.means, pk.cov_inv6, pk.opacities, o, d, 0.0, TMAX, 0,
                                 S2, True, N, rng="table" if rng == "table" else "trig", table=table)
    agree = np.mean(ids == oid)
    assert agree >= ID_AGREE, agree
    same = (ids == oid) & (oid >= 0)
    np.testing.assert_allclose(t[same], ot[same], rtol=2e-5, atol=1e-5)


def test_frame_beyond_2_31_work_items_is_not_double_counted():
    """A 1x1 frame of 2^24 + 5 passes is 2^32 + 1280 (tile pixel, pass) work
    items: it runs as 2^31-item launches whose 32-bit work counters never wrap
    (a wrapped counter re-walks items and adds their samples twice).
    Every sample misses (the only primitive is behind the camera), so the mean
    must be the background exactly and the opacity zero."""
    from paper_2504_06598_b200 import SplatAsset
    from paper_2504_06598_b200.scene import DeviceScene, camera_tuple
    from paper_2504_06598_b200.synthetic import front_camera

    a = SplatAsset(np.array([[0.0, 0.0, -20.0]]), np.array([[1.0, 0.0, 0.0, 0.0]]), np.full((1, 3), 0.1),
                   np.array([0.9]), np.zeros((1, 3, 1)))
    sc = DeviceScene.from_packed(a.packed)
    sc.build_bvh(CUTOFF)
    bg = (0.25, 0.5, 0.125)  # dyadic: bg * 2^32 is exact in the fixed-point sums
    passes = (1 << 24) + 5
    rgb, op, _ = sc.render(camera_tuple(front_camera(), 1, 1), 1, 1, passes, 1, 0, S2, True, 0, bg)
    sc.close()
    np.testing.assert_array_equal(rgb.reshape(3), np.array(bg))
    assert op[0, 0] == 0.0
