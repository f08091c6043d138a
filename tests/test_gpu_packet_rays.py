"""Explicit rays (trace_batch, kernels.py:527-540; transmittance_batch,
kernels.py:544-557) walked as warp packets.

Batches of >= 4096 rays whose probed directions share a hemisphere (camera
batches, the reference's parallel jittered rays, validate.py:36-43) go to the
packet kernel with per-lane origins; SRT_PACKET_RAYS=1 forces it for any
batch, 0 disables it.  Every route must give the oracle's ids on the same
counter stream (>= 99.9%, ties only) and its depths within fp32 tolerance.
"""

import numpy as np
import pytest

from conftest import CUTOFF, S2, TMAX, axis_rays, random_rays

pytestmark = pytest.mark.gpu


def camera_rays(w, h, origin=(0.0, 0.0, -6.0), half=0.45):
    """Row-major pinhole rays from one origin towards the cloud (unit dirs)."""
    xs = (np.arange(w) + 0.5) / w * 2.0 - 1.0
    ys = 1.0 - (np.arange(h) + 0.5) / h * 2.0
    gx, gy = np.meshgrid(xs * half * w / h, ys * half)
    d = np.stack([gx.ravel(), gy.ravel(), np.ones(w * h)], axis=1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.tile(np.asarray(origin, dtype=np.float64), (w * h, 1))
    return o, d


def _scene(n, seed, deg=0):
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import random_cloud

    a = random_cloud(n, seed=seed, sh_degree=deg)
    sc = DeviceScene.from_packed(a.packed)
    sc.build_bvh(CUTOFF)
    return a, sc


def _check(oracle, a, sc, o, d, t_min, t_max, mode, nslots, seed=3, ray_id0=11, sample0=2):
    t, ids = sc.trace_rays(o, d, t_min, t_max, mode, S2, True, nslots, "counter", seed=seed, ray_id0=ray_id0,
                           sample0=sample0)
    pk = a.packed
    lo, hi = a.aabb_arrays(CUTOFF)
    tr, ir = oracle.trace_batch(oracle.sah_build(lo, hi), pk.means, pk.cov_inv6, pk.opacities, o, d, t_min, t_max,
                                mode, S2, True, nslots, rng="counter", seed=seed, ray_id0=ray_id0, sample0=sample0)
    agree = np.mean(ids == ir)
    assert agree >= 0.999, agree
    hit = (ids == ir) & (ir >= 0)
    assert hit.sum() > 0.05 * ids.size  # the batch actually hits the cloud
    np.testing.assert_allclose(t[hit], tr[hit], rtol=2e-5, atol=1e-5)
    assert np.all(np.isinf(t[ids < 0]))
    return t, ids


@pytest.mark.parametrize("nslots", [1, 4])
@pytest.mark.parametrize("mode", [0, 1])
def test_forced_packets_on_incoherent_rays(oracle, monkeypatch, nslots, mode):
    """Correctness never depends on coherence: random origins and directions."""
    monkeypatch.setenv("SRT_PACKET_RAYS", "1")
    a, sc = _scene(20_000, 9)
    o, d = random_rays(np.random.default_rng(2), 20_000)
    _check(oracle, a, sc, o, d, 0.0, TMAX, mode, nslots)
    sc.close()


@pytest.mark.parametrize("nslots", [1, 2, 16])
def test_camera_batch_auto_route(oracle, nslots):
    a, sc = _scene(30_000, 4, deg=1)
    o, d = camera_rays(128, 96)
    _check(oracle, a, sc, o, d, 0.0, TMAX, 0, nslots)
    sc.close()


@pytest.mark.parametrize("nslots,nrays", [(1, 70_000), (4, 70_000), (1, 20_000)])
def test_jittered_parallel_rays_sorted_packets(oracle, monkeypatch, nslots, nrays):
    """The reference's validate.py ray batch (distinct origins, one direction)
    as packets (forced: the default takes them from PACKET_MIN_DISTINCT rays):
    sorted at any size >= 4096, outputs keyed by input index."""
    monkeypatch.setenv("SRT_PACKET_RAYS", "1")
    a, sc = _scene(10_000, 6)
    o, d = axis_rays(np.random.default_rng(5), nrays, lateral=1.5)
    o[:, 2] = -5.0
    _check(oracle, a, sc, o, d, 0.0, TMAX, 0, nslots)
    sc.close()


def test_packets_non_unit_directions_and_finite_interval(oracle, monkeypatch):
    """1/|d|^2 and the (t_min, t_max) interval travel per batch / per lane."""
    monkeypatch.setenv("SRT_PACKET_RAYS", "1")
    a, sc = _scene(20_000, 12)
    o, d = camera_rays(80, 60)
    # center mode's depth is (mu - o).d (kernels.py:171-173): a scaled d moves
    # the evaluation point off the peak, so the reference hits almost nothing
    _check(oracle, a, sc, o, d, 5.0, 7.0, 1, 4)
    d *= np.linspace(0.5, 3.0, d.shape[0])[:, None]
    _check(oracle, a, sc, o, d, 0.3, 4.0, 0, 1)
    _check(oracle, a, sc, o, d, 0.3, 4.0, 0, 4)
    sc.close()


def test_routes_agree(monkeypatch):
    """Packet and per-lane walks of the same camera batch: same ids and depths
    up to threshold ties."""
    a, sc = _scene(30_000, 7)
    o, d = camera_rays(160, 120)
    monkeypatch.setenv("SRT_PACKET_RAYS", "0")
    t0, i0 = sc.trace_rays(o, d, 0.0, TMAX, 0, S2, True, 2, "counter", seed=1)
    monkeypatch.setenv("SRT_PACKET_RAYS", "1")
    t1, i1 = sc.trace_rays(o, d, 0.0, TMAX, 0, S2, True, 2, "counter", seed=1)
    sc.close()
    assert np.mean(i0 == i1) >= 0.9999
    same = (i0 == i1) & (i0 >= 0)
    np.testing.assert_allclose(t0[same], t1[same], rtol=1e-6, atol=1e-7)


# ---- transmittance_batch (kernels.py:544-557) as packets --------------------

def _check_trans(oracle, a, sc, o, d, t_min, t_max, mode):
    got = sc.transmittance(o, d, t_min, t_max, mode, S2)
    pk = a.packed
    lo, hi = a.aabb_arrays(CUTOFF)
    want = oracle.transmittance(oracle.sah_build(lo, hi), pk.means, pk.cov_inv6, pk.opacities, o, d, t_min, t_max,
                                mode, S2)
    assert np.mean(want < 0.999) > 0.05  # the batch actually crosses the cloud
    np.testing.assert_allclose(got, want, rtol=2e-4, atol=2e-6)  # fp32 alphas (test_gpu_parity.py)
    return got


@pytest.mark.parametrize("mode", [0, 1])
def test_transmittance_camera_batch_auto_route(oracle, mode):
    a, sc = _scene(20_000, 3)
    o, d = camera_rays(96, 64)
    _check_trans(oracle, a, sc, o, d, 0.0, TMAX, mode)
    _check_trans(oracle, a, sc, o, d, 5.0, 7.0, mode)
    sc.close()


def test_transmittance_forced_packets_incoherent_and_sorted(oracle, monkeypatch):
    a, sc = _scene(10_000, 5)
    monkeypatch.setenv("SRT_PACKET_RAYS", "1")
    o, d = random_rays(np.random.default_rng(4), 8_000)
    _check_trans(oracle, a, sc, o, d, 0.0, TMAX, 0)
    o, d = axis_rays(np.random.default_rng(6), 70_000, lateral=1.5)  # sorted packets
    o[:, 2] = -5.0
    _check_trans(oracle, a, sc, o, d, 0.0, TMAX, 0)
    sc.close()


def test_transmittance_routes_agree(monkeypatch):
    """Packet and per-lane walks multiply the same factors in another order."""
    a, sc = _scene(30_000, 8)
    o, d = camera_rays(128, 96)
    monkeypatch.setenv("SRT_PACKET_RAYS", "0")
    t0 = sc.transmittance(o, d, 0.0, TMAX, 0, S2)
    monkeypatch.setenv("SRT_PACKET_RAYS", "1")
    t1 = sc.transmittance(o, d, 0.0, TMAX, 0, S2)
    sc.close()
    np.testing.assert_allclose(t1, t0, rtol=1e-12, atol=1e-300)


# ---- more than 16 slots (multisample up to 256, config.py:18) ---------------

@pytest.mark.parametrize("kind,nslots", [("random", 40), ("camera", 33), ("camera", 256)])
def test_trace_rays_beyond_16_slots(oracle, kind, nslots):
    """Slot groups of <= 8 (sample0 + 8 g + k): identical to one walk of
    all slots, since each slot's closest accepted hit is independent."""
    a, sc = _scene(8_000, 14)
    if kind == "random":
        o, d = random_rays(np.random.default_rng(3), 3_000)
    else:
        o, d = camera_rays(96, 64) if nslots < 100 else camera_rays(32, 24)
    _check(oracle, a, sc, o, d, 0.0, TMAX, 0, nslots)
    sc.close()
