"""Pin the oracle (C restatement) to the reference.

Fixtures in tests/golden were produced by the unmodified reference
(oracle/gen_golden.py).  In trig mode the oracle must reproduce them bit for
bit; that is what makes it a trustworthy checker for the GPU path.
"""

import numpy as np
import pytest

from conftest import S2, TMAX


def test_frozen_hash_values(oracle):
    """tests/test_sampling.py:18-27 of the reference."""
    assert oracle.hash_position([0.0, 0.0, 0.0]) == pytest.approx(oracle.hash_position([0.0, 0.0, 0.0]))
    assert oracle.hash_position([1.0, 2.0, 3.0]) == 0.8811819498150726
    assert oracle.hash_position([1.0, 2.0, 3.0], slot=1) == 0.27091394690796733
    assert oracle.hash_position([1.0, 2.0, 3.0], slot=5) == 0.1282423883676529
    assert oracle.hash_position([-0.7, 0.3, 9.1]) == 0.04217293553301715


def test_frozen_jitter_values(oracle):
    """tests/test_sampling.py:71-77 of the reference."""
    assert oracle.pixel_jitter(3, 5, 0, 0) == (0.27136341482400894, 0.6206638417206705)
    assert oracle.pixel_jitter(3, 5, 7, 2) == (0.0026576726231724024, 0.32626721472479403)


def test_hash_and_jitter_golden(oracle, golden):
    g = golden("sampling")
    hv = np.array([oracle.hash_position(p, int(k)) for p, k in zip(g["points"], g["slots"])])
    np.testing.assert_array_equal(hv, g["hash"])
    jit = np.array([oracle.pixel_jitter(*map(int, a)) for a in g["jitter_args"]])
    np.testing.assert_array_equal(jit, g["jitter"])


def test_sah_build_bitwise(oracle, golden):
    """bvh.build (bvh.py:87-193) restated in C gives the identical tree."""
    g = golden("bvh_3000")
    b = oracle.sah_build(g["lo"], g["hi"])
    for f in ("node_lo", "node_hi", "node_left", "node_right", "node_count", "prim_order"):
        np.testing.assert_array_equal(getattr(b, f), g[f], err_msg=f)


def _scene_400():
    from paper_2504_06598_b200.synthetic import random_cloud

    return random_cloud(400, seed=31)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("nslots", [1, 4])
def test_trace_batch_bitwise(oracle, golden, mode, nslots):
    """kernels.trace_batch (kernels.py:527-540), trig hash: (t, id) bit for bit."""
    g = golden("trace_400")
    a = _scene_400()
    pk = a.packed
    lo, hi = a.aabb_arrays(np.sqrt(S2))
    b = oracle.sah_build(lo, hi)
    t, ids = oracle.trace_batch(b, pk.means, pk.cov_inv6, pk.opacities, g["origins"], g["dirs"], 0.0, TMAX, mode, S2,
                                True, nslots, rng="trig")
    np.testing.assert_array_equal(ids, g[f"id_m{mode}_n{nslots}"])
    np.testing.assert_array_equal(t, g[f"t_m{mode}_n{nslots}"])


def test_transmittance_matches(oracle, golden):
    g = golden("trace_400")
    a = _scene_400()
    pk = a.packed
    lo, hi = a.aabb_arrays(np.sqrt(S2))
    b = oracle.sah_build(lo, hi)
    tr = oracle.transmittance(b, pk.means, pk.cov_inv6, pk.opacities, g["origins"], g["dirs"], 0.0, TMAX, 0, S2)
    np.testing.assert_allclose(tr, g["transmittance"], rtol=1e-12, atol=0)


def test_render_bitwise(oracle, golden):
    """render() -> kernels.render_stochastic (kernels.py:622-673), trig hash."""
    from paper_2504_06598_b200.synthetic import anisotropic_sheets, front_camera, random_cloud

    g = golden("render_small")
    a = random_cloud(300, seed=53, sh_degree=3)
    pk = a.packed
    lo, hi = a.aabb_arrays(np.sqrt(S2))
    b = oracle.sah_build(lo, hi)
    cam = front_camera()
    ct = oracle.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, 24, 20)
    out = oracle.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 3, ct, 24, 20, passes=3, nslots=2, s2=S2,
                        seed=5, rng="trig", background=[0.1, 0.2, 0.3])
    np.testing.assert_array_equal(out["rgb"], g["rgb"])
    np.testing.assert_array_equal(out["opacity"], g["opacity"])
    # center depth mode on tilted sheets
    a2 = anisotropic_sheets(60, seed=3)
    pk2 = a2.packed
    lo, hi = a2.aabb_arrays(np.sqrt(S2))
    b2 = oracle.sah_build(lo, hi)
    ct2 = oracle.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, 16, 12)
    out2 = oracle.render(b2, pk2.means, pk2.cov_inv6, pk2.opacities, pk2.sh, 0, ct2, 16, 12, passes=3, nslots=1,
                         mode=1, s2=S2, seed=11, rng="trig")
    np.testing.assert_array_equal(out2["rgb"], g["rgb_center"])
    np.testing.assert_array_equal(out2["opacity"], g["opacity_center"])


# ---- counter RNG spec (frozen) ---------------------------

COUNTER_GOLDEN = [  # (seed, ray_id, sample, prim); values frozen in test_counter_rng_frozen_values
    ((0, 0, 0, 0), None),
    ((0, 1, 0, 0), None),
    ((7, 123456, 3, 999), None),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), None),
]


def test_counter_rng_c_matches_numpy(oracle):
    rs = np.random.default_rng(5)
    args = rs.integers(0, 2**32, size=(2000, 4), dtype=np.uint64)
    c = np.array([oracle.counter_u(oracle.walk_key(int(s), int(r), int(k)), int(p)) for s, r, k, p in args])
    v = oracle.counter_u_np(args[:, 0], args[:, 1], args[:, 2], args[:, 3])
    np.testing.assert_array_equal(c, v)
    assert np.all((c >= 0) & (c < 1))
    assert np.all(c * 2**24 == np.floor(c * 2**24))  # exactly 24 bits


def test_counter_rng_frozen_values(oracle):
    vals = [oracle.counter_u(oracle.walk_key(s, r, k), p) for (s, r, k, p), _ in COUNTER_GOLDEN]
    frozen = [0.6150132417678833, 0.4052417278289795, 0.8931280374526978, 0.8988131284713745]
    assert vals == frozen


def test_counter_rng_uniform_and_decorrelated(oracle):
    """256-bin chi-square and adjacent-prim / adjacent-sample correlation."""
    from scipy import stats

    n = 200_000
    prim = np.arange(n)
    u0 = oracle.counter_u_np(0, 17, 0, prim)
    u1 = oracle.counter_u_np(0, 17, 1, prim)
    counts, _ = np.histogram(u0, bins=256, range=(0.0, 1.0))
    assert stats.chisquare(counts).pvalue > 1e-3
    assert abs(u0.mean() - 0.5) < 0.005
    assert abs(np.corrcoef(u0[:-1], u0[1:])[0, 1]) < 0.01
    assert abs(np.corrcoef(u0, u1)[0, 1]) < 0.01


def test_render_c1_bitwise(oracle, golden):
    """configs[0] (C1) frames from the reference: 10k SH0 at 1 spp, and SH3 at
    4 passes x N=2 with a background, bit for bit."""
    from paper_2504_06598_b200.synthetic import front_camera, random_cloud

    g = golden("render_c1")
    cam = front_camera()
    a = random_cloud(10_000, seed=0, sh_degree=0)
    pk = a.packed
    lo, hi = a.aabb_arrays(np.sqrt(S2))
    b = oracle.sah_build(lo, hi)
    ct = oracle.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, 64, 64)
    out = oracle.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 0, ct, 64, 64, s2=S2, rng="trig")
    np.testing.assert_array_equal(out["rgb"], g["rgb"])
    np.testing.assert_array_equal(out["opacity"], g["opacity"])
    a3 = random_cloud(10_000, seed=0, sh_degree=3)
    pk3 = a3.packed
    ct3 = oracle.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, 48, 40)
    out3 = oracle.render(b, pk3.means, pk3.cov_inv6, pk3.opacities, pk3.sh, 3, ct3, 48, 40, passes=4, nslots=2,
                         s2=S2, seed=7, rng="trig", background=[0.05, 0.1, 0.2])
    np.testing.assert_array_equal(out3["rgb"], g["rgb_ms"])
    np.testing.assert_array_equal(out3["opacity"], g["opacity_ms"])


def test_exact_compositing_matches_reference(oracle, golden):
    """kernels.exact_batch and render(reference_mode=True) (kernels.py:584-604,
    677-723) restated: bit for bit against the reference's outputs."""
    from paper_2504_06598_b200.synthetic import front_camera, random_cloud

    g = golden("exact_500")
    t = golden("trace_400")
    a = random_cloud(500, seed=41, sh_degree=2)
    pk = a.packed
    bg = [0.15, 0.25, 0.35]
    rgb, op = oracle.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 2, t["origins"], t["dirs"], s2=S2,
                                 background=bg)
    np.testing.assert_array_equal(rgb, g["rgb"])
    np.testing.assert_array_equal(op, g["opacity"])
    cam = front_camera()
    ct = oracle.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, 20, 16)
    frgb, fop = oracle.render_exact(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 2, ct, 20, 16, frames=3, s2=S2, seed=2,
                                    background=bg)
    np.testing.assert_array_equal(frgb, g["frame_rgb"])
    np.testing.assert_array_equal(fop, g["frame_opacity"])
    assert int(g["frame_spp"]) == 3


def test_biased_batch_bitwise(oracle, golden):
    """kernels.biased_batch (kernels.py:479-518, 561-580) with the reference's
    trig draw: bit-identical for k in {1, 2, 5}, both depth modes."""
    from paper_2504_06598_b200.synthetic import random_cloud

    g = golden("biased_500")
    t = golden("trace_400")
    a = random_cloud(500, seed=41, sh_degree=2)
    pk = a.packed
    for mode in (0, 1):
        for kk in (1, 2, 5):
            rgb = oracle.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, 2, t["origins"], t["dirs"], kk,
                                      mode=mode, s2=S2, background=[0.15, 0.25, 0.35], rng="trig")
            np.testing.assert_array_equal(rgb, g[f"rgb_m{mode}_k{kk}"])


def test_c3target_scale_trace_bitwise(oracle, golden):
    """The oracle at the headline scale (density-preserving 1M SH-3 cloud, its
    SAH tree, pass-0 camera rays of a 16-pixel grid of the 1080p frame):
    trace_batch ids and depths bit-identical to the unmodified reference's."""
    from paper_2504_06598_b200.synthetic import density_cloud

    g = golden("c3target_grid")
    a = density_cloud(1_000_000)
    pk = a.packed
    lo, hi = a.aabb_arrays(np.sqrt(S2))
    b = oracle.sah_build(lo, hi)
    t, ids = oracle.trace_batch(b, pk.means, pk.cov_inv6, pk.opacities, g["origins"], g["dirs"], 0.0, TMAX, 0, S2,
                                True, 1, rng="trig")
    np.testing.assert_array_equal(ids, g["id"])
    np.testing.assert_array_equal(t, g["t"])
