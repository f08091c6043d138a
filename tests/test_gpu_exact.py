"""Exact sorted compositing on the GPU (render_exact / exact_batch,
kernels.py:441-475, 584-604, 677-723) against the reference's own outputs
(tests/golden/exact_500.npz) and the oracle.  fp32 alphas and colours: 1e-5
relative; a pixel whose two candidates lie within fp32 resolution in depth
may composite in swapped order, so a small fraction may deviate more."""

import numpy as np
import pytest

from conftest import S2, random_rays

pytestmark = pytest.mark.gpu
RTOL, ATOL = 2e-5, 2e-6


def _close_fraction(a, b):
    ok = np.abs(a - b) <= RTOL * np.abs(b) + ATOL
    return float(np.mean(ok.reshape(ok.shape[0], -1).all(axis=1) if ok.ndim > 1 else ok))


def test_exact_batch_matches_reference(golden):
    from paper_2504_06598_b200 import kernels
    from paper_2504_06598_b200.synthetic import random_cloud

    g = golden("exact_500")
    t = golden("trace_400")
    a = random_cloud(500, seed=41, sh_degree=2)
    pk = a.packed
    n = t["origins"].shape[0]
    rgb = np.empty((n, 3))
    op = np.empty(n)
    kernels.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, t["origins"], t["dirs"], 0.0,
                        float(np.finfo(np.float64).max), 0, S2, 0.15, 0.25, 0.35, rgb, op)
    assert _close_fraction(rgb, g["rgb"]) >= 0.995
    assert _close_fraction(op, g["opacity"]) >= 0.995


def test_render_reference_mode_matches_reference(golden):
    from paper_2504_06598_b200 import RenderSettings, front_camera, render
    from paper_2504_06598_b200.synthetic import random_cloud

    g = golden("exact_500")
    a = random_cloud(500, seed=41, sh_degree=2)
    buf = render(a, front_camera(), RenderSettings(width=20, height=16, spp=3, seed=2, reference_mode=True,
                                                   background=[0.15, 0.25, 0.35]))
    assert buf.spp == 3
    assert _close_fraction(buf.rgb.reshape(-1, 3), g["frame_rgb"].reshape(-1, 3)) >= 0.995
    assert _close_fraction(buf.opacity.reshape(-1), g["frame_opacity"].reshape(-1)) >= 0.995


def test_exact_vs_oracle_larger(oracle):
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(5_000, seed=3, sh_degree=3)
    pk = a.packed
    o, d = random_rays(np.random.default_rng(4), 4_000)
    sc = DeviceScene.from_packed(pk)
    sc.build_bvh(np.sqrt(S2))
    rgb, op = sc.exact_rays(o, d, s2=S2, background=(0.1, 0.0, 0.2))
    want_rgb, want_op = oracle.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 3, o, d, s2=S2,
                                           background=(0.1, 0.0, 0.2))
    assert _close_fraction(rgb, want_rgb) >= 0.995
    assert _close_fraction(op, want_op) >= 0.995


def test_exact_closed_forms():
    """tests/test_render.py:113-124 and tests/test_kernels.py:163-175 of the reference."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, kernels, pancake_stack, render, two_layer_scene

    buf = render(two_layer_scene(), front_camera(), RenderSettings(width=8, height=8, spp=4, reference_mode=True))
    np.testing.assert_allclose(buf.rgb[..., 0], 0.5, atol=1e-6)
    np.testing.assert_allclose(buf.rgb[..., 1], 0.0, atol=1e-6)
    np.testing.assert_allclose(buf.rgb[..., 2], 0.25, atol=1e-6)
    np.testing.assert_allclose(buf.opacity, 0.75, atol=1e-6)
    assert buf.spp == 4
    tie = pancake_stack([0.5, 0.5], [[1, 0, 0], [0, 0, 1]], spacing=0.0)  # equal depths: id order
    pk = tie.packed
    rgb = np.empty((1, 3))
    op = np.empty(1)
    kernels.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 0, np.array([[0.1, 0.0, 0.0]]),
                        np.array([[0.0, 0.0, 1.0]]), 0.0, float(np.finfo(np.float64).max), 0, S2, 0.0, 0.0, 0.0, rgb, op)
    np.testing.assert_allclose(rgb[0], [0.5, 0.0, 0.25], atol=1e-6)


def test_stochastic_mean_approaches_exact():
    """tests/test_kernels.py:255-266: the estimator's mean closes in on the exact image."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, render
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(100, seed=59)
    errs = {}
    for spp in (1, 512):
        exact = render(a, front_camera(), RenderSettings(width=8, height=8, spp=spp, seed=5, reference_mode=True))
        noisy = render(a, front_camera(), RenderSettings(width=8, height=8, spp=spp, seed=5))
        errs[spp] = float(np.mean((noisy.rgb - exact.rgb) ** 2))
    assert errs[512] < errs[1] / 20


@pytest.mark.parametrize("kk", [1, 3, 300])
def test_biased_counter_vs_oracle(oracle, kk):
    """Biased k-nearest composite under the counter draw (seed, ray i, sample
    0) against the oracle; kk=300 > the 256-entry kept list is legal while
    fewer than 256 candidates are accepted."""
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(5_000, seed=3, sh_degree=3)
    pk = a.packed
    o, d = random_rays(np.random.default_rng(5), 4_000)
    sc = DeviceScene.from_packed(pk)
    sc.build_bvh(np.sqrt(S2))
    rgb = sc.biased_rays(o, d, kk, s2=S2, background=(0.1, 0.0, 0.2), seed=11)
    sc.close()
    want = oracle.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 3, o, d, kk, s2=S2,
                               background=(0.1, 0.0, 0.2), rng="counter", seed=11)
    assert _close_fraction(rgb, want) >= 0.995


def test_biased_shim_signature():
    """kernels.biased_batch keeps the reference's positional signature
    (kernels.py:561-565) and writes out_rgb in place."""
    from paper_2504_06598_b200 import kernels
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(300, seed=2)
    pk = a.packed
    o, d = random_rays(np.random.default_rng(1), 64)
    out = np.full((64, 3), np.nan)
    kernels.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, o, d, 0.0,
                         float(np.finfo(np.float64).max), 0, S2, 2, 0.0, 0.0, 0.0, out)
    assert np.isfinite(out).all() and (out >= 0).all()


def test_biased_frame_counter_matches_explicit_rays():
    """render_biased's counter draw of pixel (px,py), pass f is (seed, py*W+px,
    f): one pass equals biased_rays over the same camera rays, row-major."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, generate_camera_ray, render_biased
    from paper_2504_06598_b200.render import prepare
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(2_000, seed=8, sh_degree=1)
    cam = front_camera()
    st = RenderSettings(width=24, height=18, spp=1, seed=3)
    frame = render_biased(a, cam, st, 2)
    rays = [generate_camera_ray(cam, st, (x, y), 0) for y in range(18) for x in range(24)]
    o = np.array([r[0] for r in rays])
    d = np.array([r[1] for r in rays])
    sc = prepare(a, st)
    per_ray = sc.biased_rays(o, d, 2, s2=st.cutoff_s ** 2, seed=3, ray_id0=0, sample0=0)
    ok = np.all(np.abs(frame.reshape(-1, 3) - per_ray) <= 1e-6, axis=1)
    assert ok.mean() >= 0.99


def test_exact_and_biased_peel_many_candidates(oracle):
    """A ray through 700 layers (more than any chunk): exact compositing peels
    the candidates 256 at a time and matches the closed form and the oracle;
    the biased composite with every candidate accepted and k = 600 (several
    128-chunks) equals the exact composite truncated after 600 layers."""
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import pancake_stack

    n = 700
    rs = np.random.default_rng(3)
    alphas = rs.uniform(0.001, 0.01, n)
    colors = rs.uniform(0.0, 1.0, (n, 3))
    a = pancake_stack(alphas, colors, z0=1.0, spacing=0.05, thickness=0.004)
    pk = a.packed
    o = np.array([[0.01, -0.02, 0.0], [0.3, 0.1, 0.0]])
    d = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0]])
    sc = DeviceScene.from_packed(pk)
    sc.build_bvh(np.sqrt(S2))
    rgb, op = sc.exact_rays(o, d, s2=S2, background=(0.2, 0.3, 0.4))
    want_rgb, want_op = oracle.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, o, d, s2=S2,
                                           background=(0.2, 0.3, 0.4))
    np.testing.assert_allclose(rgb, want_rgb, rtol=2e-5, atol=2e-6)
    np.testing.assert_allclose(op, want_op, rtol=2e-5, atol=2e-6)
    trans = np.cumprod(np.concatenate([[1.0], 1.0 - alphas]))
    closed = (trans[:n, None] * alphas[:, None] * colors).sum(axis=0) + trans[n] * np.array([0.2, 0.3, 0.4])
    np.testing.assert_allclose(rgb[0], closed, rtol=1e-4)
    got = sc.biased_rays(o, d, 600, s2=S2, background=(0.2, 0.3, 0.4), rng="table", table=np.zeros(n))
    sc.close()
    k = 600
    trunc = (trans[:k, None] * alphas[:k, None] * colors[:k]).sum(axis=0) + trans[k] * np.array([0.2, 0.3, 0.4])
    np.testing.assert_allclose(got[0], trunc, rtol=1e-4)


def test_exact_frame_packets_vs_oracle(oracle):
    """render(reference_mode=True) walks 8x4 pixel blocks as packets
    (k_exact_packet, every pass of a block in one warp): a 20k SH-3
    density-preserving cloud at 72x44 (partial blocks at the right and bottom
    edges), 2 passes, against the brute-force oracle render_exact."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, render
    from paper_2504_06598_b200.scene import camera_tuple
    from paper_2504_06598_b200.synthetic import density_cloud

    a = density_cloud(20_000, seed=5)
    pk = a.packed
    st = RenderSettings(width=72, height=44, spp=2, seed=4, reference_mode=True, background=[0.1, 0.2, 0.05])
    buf = render(a, front_camera(), st)
    want_rgb, want_op = oracle.render_exact(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree,
                                            np.array(camera_tuple(front_camera(), 72, 44)), 72, 44, frames=2,
                                            s2=S2, seed=4, background=(0.1, 0.2, 0.05))
    assert _close_fraction(buf.rgb.reshape(-1, 3), want_rgb.reshape(-1, 3)) >= 0.995
    assert _close_fraction(buf.opacity.reshape(-1), want_op.reshape(-1)) >= 0.995
    np.testing.assert_allclose(buf.rgb, want_rgb, atol=2e-3)


@pytest.mark.parametrize("one_origin", [True, False])
def test_exact_rays_packets_vs_oracle(oracle, one_origin):
    """One-hemisphere exact_batch batches of >= 4096 rays take the packet
    kernel (coherence-sorted when the origins differ)."""
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import density_cloud

    a = density_cloud(10_000, seed=6)
    pk = a.packed
    rs = np.random.default_rng(7)
    R = 5000
    d = rs.normal(size=(R, 3)) * [0.2, 0.2, 0.0] + [0.0, 0.0, 1.0]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.tile([0.1, -0.2, -4.0], (R, 1)) if one_origin else rs.uniform(-1.0, 1.0, (R, 3)) * [1, 1, 0] + [0, 0, -4]
    sc = DeviceScene.from_packed(pk)
    sc.build_bvh(np.sqrt(S2))
    rgb, op = sc.exact_rays(o, d, s2=S2, background=(0.3, 0.1, 0.2))
    sc.close()
    want_rgb, want_op = oracle.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, o, d, s2=S2,
                                           background=(0.3, 0.1, 0.2))
    assert _close_fraction(rgb, want_rgb) >= 0.995
    assert _close_fraction(op, want_op) >= 0.995


@pytest.mark.parametrize("layers", [1000, 1100])
def test_exact_frame_long_lists(layers):
    """Camera rays through every layer of a 1000- / 1100-layer stack: 1000
    fits a packet lane's candidate list (sorted there), 1100 exceeds it and
    the lane composites by chunked peeling; both equal the closed form."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, render
    from paper_2504_06598_b200.synthetic import pancake_stack

    rs = np.random.default_rng(11)
    alphas = rs.uniform(0.001, 0.004, layers)
    colors = rs.uniform(0.0, 1.0, (layers, 3))
    a = pancake_stack(alphas, colors, z0=1.0, spacing=0.004, thickness=0.0005)
    buf = render(a, front_camera(), RenderSettings(width=16, height=8, spp=1, reference_mode=True,
                                                   background=[0.2, 0.3, 0.4]))
    trans = np.cumprod(np.concatenate([[1.0], 1.0 - alphas]))
    closed = (trans[:layers, None] * alphas[:, None] * colors).sum(axis=0) + trans[layers] * np.array([0.2, 0.3, 0.4])
    np.testing.assert_allclose(buf.rgb.reshape(-1, 3), np.broadcast_to(closed, (128, 3)), rtol=1e-4)
    np.testing.assert_allclose(buf.opacity, 1.0 - trans[layers], rtol=1e-5)


@pytest.mark.parametrize("kk", [1, 4, 12])
def test_biased_frame_packets_vs_oracle(oracle, kk):
    """render_biased walks 8x4 pixel blocks as packets (k <= 8: clipped at
    the k-th accepted depth; 12: unclipped) -- 2 passes of a 20k SH-3
    cloud at 56x40 against the oracle's biased_batch over the same camera
    rays, draw (seed, py*W+px, pass)."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, generate_camera_ray, render_biased
    from paper_2504_06598_b200.synthetic import density_cloud

    a = density_cloud(20_000, seed=9)
    pk = a.packed
    cam = front_camera()
    W, H = 56, 40
    st = RenderSettings(width=W, height=H, spp=2, seed=5, background=[0.2, 0.1, 0.0])
    frame = render_biased(a, cam, st, kk)
    want = np.zeros((H * W, 3))
    for f in range(2):
        rays = [generate_camera_ray(cam, st, (x, y), f) for y in range(H) for x in range(W)]
        o = np.array([r[0] for r in rays])
        d = np.array([r[1] for r in rays])
        want += oracle.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 3, o, d, kk, s2=S2,
                                    background=(0.2, 0.1, 0.0), rng="counter", seed=5, ray_id0=0, sample0=f)
    want /= 2
    assert _close_fraction(frame.reshape(-1, 3), want) >= 0.995


@pytest.mark.parametrize("rng,kk", [("counter", 1), ("counter", 6), ("counter", 20), ("table", 3)])
def test_biased_rays_packets_vs_oracle(oracle, rng, kk):
    """One-hemisphere biased_batch batches of >= 4096 rays from distinct
    origins walk as coherence-sorted packets; draws keyed by the caller's ray
    index (counter) or read from the table."""
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import density_cloud

    a = density_cloud(10_000, seed=12)
    pk = a.packed
    rs = np.random.default_rng(13)
    R = 5000
    d = rs.normal(size=(R, 3)) * [0.2, 0.2, 0.0] + [0.0, 0.0, 1.0]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = rs.uniform(-1.0, 1.0, (R, 3)) * [1, 1, 0] + [0, 0, -4]
    table = rs.uniform(0.0, 1.0, pk.means.shape[0]) if rng == "table" else None
    sc = DeviceScene.from_packed(pk)
    sc.build_bvh(np.sqrt(S2))
    kw = dict(table=table) if table is not None else dict(seed=21, ray_id0=7, sample0=3)
    rgb = sc.biased_rays(o, d, kk, s2=S2, background=(0.1, 0.3, 0.2), rng=rng, **kw)
    sc.close()
    want = oracle.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 3, o, d, kk, s2=S2,
                               background=(0.1, 0.3, 0.2), rng=rng, **kw)
    assert _close_fraction(rgb, want) >= 0.995


def test_biased_frame_long_accepted_lists_fall_back(oracle):
    """k = 12 walks unclipped and keeps every accepted candidate in the ray's
    list: through 1,100 near-opaque layers a list overflows its 1,024
    entries and the ray composites through the per-lane peeling path --
    same result as the oracle's brute-force biased composite."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, generate_camera_ray, render_biased
    from paper_2504_06598_b200.synthetic import pancake_stack

    layers = 1100
    rs = np.random.default_rng(17)
    alphas = rs.uniform(0.97, 0.99, layers)
    colors = rs.uniform(0.0, 1.0, (layers, 3))
    a = pancake_stack(alphas, colors, z0=1.0, spacing=0.004, thickness=0.0005)
    pk = a.packed
    cam = front_camera()
    st = RenderSettings(width=16, height=8, spp=1, seed=3, background=[0.2, 0.3, 0.4])
    frame = render_biased(a, cam, st, 12)
    rays = [generate_camera_ray(cam, st, (x, y), 0) for y in range(8) for x in range(16)]
    o = np.array([r[0] for r in rays])
    d = np.array([r[1] for r in rays])
    want = oracle.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, o, d, 12, s2=S2,
                               background=(0.2, 0.3, 0.4), rng="counter", seed=3, ray_id0=0, sample0=0)
    np.testing.assert_allclose(frame.reshape(-1, 3), want, rtol=1e-4, atol=1e-6)
