"""Stochastic-tracer semantics, run on BOTH backends: the CPU oracle (checker
itself, not gpu-marked) and the GPU product through the libsrt C ABI
(gpu-marked).  Mirrors the reference's tests/test_tracer.py (scripted walk)
and tests/test_acceptance.py (A02, A03, A04, A05, A07) under the counter RNG.
"""

import math

import numpy as np
import pytest

from conftest import CUTOFF, S2, TMAX, axis_rays, random_rays
from paper_2504_06598_b200.synthetic import pancake_stack, random_cloud, two_layer_scene


class OracleBackend:
    name = "oracle"

    def __init__(self, oracle):
        self.O = oracle

    def trace(self, asset, origins, dirs, nslots=1, rng="counter", table=None, seed=0, ray_id0=0, sample0=0,
              clip=True, mode=0, t_min=0.0, t_max=TMAX, counters=False):
        pk = asset.packed
        lo, hi = asset.aabb_arrays(CUTOFF)
        b = self.O.sah_build(lo, hi)
        return self.O.trace_batch(b, pk.means, pk.cov_inv6, pk.opacities, origins, dirs, t_min, t_max, mode, S2, clip,
                                  nslots, rng=rng, seed=seed, ray_id0=ray_id0, sample0=sample0, table=table,
                                  counters=counters)

    def transmittance(self, asset, origins, dirs):
        pk = asset.packed
        lo, hi = asset.aabb_arrays(CUTOFF)
        b = self.O.sah_build(lo, hi)
        return self.O.transmittance(b, pk.means, pk.cov_inv6, pk.opacities, origins, dirs, 0.0, TMAX, 0, S2)

    def biased(self, asset, origins, dirs, kk, rng="counter", table=None, seed=0, mode=0, background=(0, 0, 0)):
        pk = asset.packed
        return self.O.biased_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, origins, dirs, kk,
                                   mode=mode, s2=S2, background=background, rng=rng, seed=seed, table=table)

    def exact(self, asset, origins, dirs, background=(0, 0, 0)):
        pk = asset.packed
        return self.O.exact_batch(pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, origins, dirs, s2=S2,
                                  background=background)[0]


class GpuBackend:
    name = "gpu"

    def __init__(self):
        from paper_2504_06598_b200.scene import DeviceScene

        self.DeviceScene = DeviceScene

    def scene(self, asset):
        sc = self.DeviceScene.from_packed(asset.packed)
        sc.build_bvh(CUTOFF)
        return sc

    def trace(self, asset, origins, dirs, nslots=1, rng="counter", table=None, seed=0, ray_id0=0, sample0=0,
              clip=True, mode=0, t_min=0.0, t_max=TMAX, counters=False):
        assert not counters
        sc = self.scene(asset)
        try:
            return sc.trace_rays(origins, dirs, t_min, t_max, mode, S2, clip, nslots, rng, seed, ray_id0, sample0,
                                 table)
        finally:
            sc.close()

    def transmittance(self, asset, origins, dirs):
        sc = self.scene(asset)
        try:
            return sc.transmittance(origins, dirs, 0.0, TMAX, 0, S2)
        finally:
            sc.close()

    def biased(self, asset, origins, dirs, kk, rng="counter", table=None, seed=0, mode=0, background=(0, 0, 0)):
        sc = self.scene(asset)
        try:
            return sc.biased_rays(origins, dirs, kk, 0.0, TMAX, mode, S2, background, rng, seed, 0, 0, table)
        finally:
            sc.close()

    def exact(self, asset, origins, dirs, background=(0, 0, 0)):
        sc = self.scene(asset)
        try:
            return sc.exact_rays(origins, dirs, 0.0, TMAX, 0, S2, background)[0]
        finally:
            sc.close()


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def backend(request, oracle):
    if request.param == "oracle":
        return OracleBackend(oracle)
    return GpuBackend()


# ---- scripted walks (reference tests/test_tracer.py:80-121) -------------------

def _six_layers():
    return pancake_stack([0.5] * 6, [[1, 0, 0]] * 6)


def test_first_accept_wins(backend):
    """Draws 0.6, 0.7, 0.2 on layers 0..2 (alpha 0.5): prim 2 at t = 4."""
    a = _six_layers()
    table = np.array([[0.6], [0.7], [0.2], [0.9], [0.9], [0.9]])
    t, ids = backend.trace(a, [[0, 0, 0]], [[0, 0, 1]], 1, rng="table", table=table)
    assert ids[0, 0] == 2
    assert t[0, 0] == pytest.approx(4.0, abs=1e-5)


def test_all_rejections_miss(backend):
    a = _six_layers()
    t, ids = backend.trace(a, [[0, 0, 0]], [[0, 0, 1]], 1, rng="table", table=np.full((6, 1), 0.9))
    assert ids[0, 0] == -1 and t[0, 0] == math.inf


def test_boundary_is_strict(backend):
    """u == alpha rejects (tracer.py:75-78): alpha 0.5 with u = 0.5 never accepts."""
    a = _six_layers()
    t, ids = backend.trace(a, [[0, 0, 0]], [[0, 0, 1]], 1, rng="table", table=np.full((6, 1), 0.5))
    assert ids[0, 0] == -1


def test_multi_slot_interleave_and_clip(backend):
    """layer 0: slot 0 rejects (0.8), slot 1 accepts (0.1); layer 1: slot 0
    accepts; the walk clips at max(3, 2) = 3 so layer 2 is never accepted."""
    a = _six_layers()
    table = np.array([[0.8, 0.1], [0.1, 0.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0]])
    t, ids = backend.trace(a, [[0, 0, 0]], [[0, 0, 1]], 2, rng="table", table=table)
    assert list(ids[0]) == [1, 0]
    np.testing.assert_allclose(t[0], [3.0, 2.0], atol=1e-5)


def test_oracle_draw_count_matches_reference_walk(oracle):
    """The scripted walkthrough consumes exactly 3 draws (reference
    test_tracer.py:90-97) and 3 in the two-slot case (:108-121)."""
    be = OracleBackend(oracle)
    a = _six_layers()
    table = np.array([[0.6], [0.7], [0.2], [0.9], [0.9], [0.9]])
    _, _, c = be.trace(a, [[0, 0, 0]], [[0, 0, 1]], 1, rng="table", table=table, counters=True)
    assert c["draws"] == 3
    table2 = np.array([[0.8, 0.1], [0.1, 0.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0]])
    _, _, c2 = be.trace(a, [[0, 0, 0]], [[0, 0, 1]], 2, rng="table", table=table2, counters=True)
    assert c2["draws"] == 3


def test_open_range(backend):
    """Candidates exactly at t_min or t_max are excluded (kernels.py:349)."""
    a = pancake_stack([1.0], [[1, 0, 0]], z0=4.0)
    o, d = [[0.1, 0.2, 0.0]], [[0, 0, 1]]
    _, ids = backend.trace(a, o, d, 1, rng="table", table=np.zeros((1, 1)))
    assert ids[0, 0] == 0
    _, ids = backend.trace(a, o, d, 1, rng="table", table=np.zeros((1, 1)), t_max=3.999)
    assert ids[0, 0] == -1
    _, ids = backend.trace(a, o, d, 1, rng="table", table=np.zeros((1, 1)), t_min=4.001)
    assert ids[0, 0] == -1


# ---- statistical acceptance (reference tests/test_acceptance.py) --------------

def test_a02_unbiased_single_hit(backend):
    """Two layers (alpha .5/.5, red over blue): mean of 1e6 samples within 3 SE
    of (0.5, 0, 0.25), hit rate within 3 sigma of 0.75."""
    a = two_layer_scene()
    n = 1_000_000
    o, d = axis_rays(np.random.default_rng(7), n)
    _, ids = backend.trace(a, o, d, 1, seed=7)
    ids = ids[:, 0]
    lut = np.array([[0, 0, 0], [1, 0, 0], [0, 0, 1]], float)
    samples = lut[ids + 1]
    mean = samples.mean(axis=0)
    se = samples.std(axis=0, ddof=1) / math.sqrt(n)
    assert np.all(np.abs(mean - [0.5, 0, 0.25]) <= 3 * se + 1e-12)
    p = float(np.mean(ids >= 0))
    assert abs(p - 0.75) <= 3 * math.sqrt(0.75 * 0.25 / n)


def test_a03_miss_rate_and_transmittance(backend):
    geom = np.random.default_rng(42)
    zs = np.sort(geom.uniform(1.5, 12.0, 8))
    alphas = geom.uniform(0.1, 0.5, 8)
    a = pancake_stack(alphas, [[1, 1, 1]] * 8)
    a.means[:, 2] = zs
    n = 200_000
    o, d = axis_rays(np.random.default_rng(0), n)
    _, ids = backend.trace(a, o, d, 1, seed=3)
    p_miss = float(np.prod(1 - alphas))
    sigma = math.sqrt(p_miss * (1 - p_miss) / n)
    assert abs(float(np.mean(ids[:, 0] < 0)) - p_miss) <= 3 * sigma
    tr = backend.transmittance(a, [[0.07, -0.03, -1.0]], [[0.0, 0.0, 1.0]])
    tol = 1e-12 if backend.name == "oracle" else 2e-6
    assert tr[0] == pytest.approx(p_miss, abs=tol)


def test_a04_clip_neutral(backend):
    """Clipping on/off: identical (t, id) over 2e4 rays through 1e4 prims."""
    a = random_cloud(10_000, seed=11)
    o, d = random_rays(np.random.default_rng(1), 20_000)
    r1 = backend.trace(a, o, d, 2, seed=5, clip=True)
    r2 = backend.trace(a, o, d, 2, seed=5, clip=False)
    np.testing.assert_array_equal(r1[1], r2[1])
    np.testing.assert_array_equal(r1[0], r2[0])


def test_a07_multisample_matches_independent(backend):
    """16 slots of one walk vs 16 independent walks (chi-square p > 1e-3,
    variance ratio in [0.8, 1.25])."""
    from scipy import stats

    alphas = [0.35, 0.5, 0.2, 0.65, 0.4]
    colors = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 1, 1)]
    a = pancake_stack(alphas, colors)
    n = 10_000
    o, d = axis_rays(np.random.default_rng(31), n)
    _, ids_m = backend.trace(a, o, d, 16, seed=1)
    o1, d1 = axis_rays(np.random.default_rng(32), n * 16)
    _, ids_s = backend.trace(a, o1, d1, 1, seed=2)
    outcomes = np.arange(-1, len(alphas))
    h_m = np.array([(ids_m == v).sum() for v in outcomes])
    h_s = np.array([(ids_s == v).sum() for v in outcomes])
    _, p, _, _ = stats.chi2_contingency(np.vstack([h_m, h_s]))
    assert p > 1e-3
    red = np.zeros(len(alphas) + 1)
    red[1:] = [c[0] for c in colors]
    ratio = red[ids_m + 1].mean(axis=1).var(ddof=1) / (red[ids_s + 1].var(ddof=1) / 16.0)
    assert 0.8 <= ratio <= 1.25


def test_trace_batch_empty_and_miss(backend):
    a = random_cloud(100, seed=1)
    t, ids = backend.trace(a, np.zeros((0, 3)), np.zeros((0, 3)), 1)
    assert t.shape == (0, 1)
    t, ids = backend.trace(a, [[0, 0, -10]], [[0, 0, -1]], 3)  # facing away
    assert np.all(ids == -1) and np.all(np.isinf(t))


# ---- biased k-nearest composite (reference tests/test_tracer.py:270-299) -----

def test_biased_truncation_composites_only_k_nearest(backend):
    """Both layers accepted by script: k=1 shades only the red front layer,
    k=2 adds blue with the compositing weight (test_tracer.py:271-283)."""
    a = two_layer_scene()
    table = np.array([[0.1], [0.1]])
    k1 = backend.biased(a, [[0, 0, 0]], [[0, 0, 1]], 1, rng="table", table=table)
    k2 = backend.biased(a, [[0, 0, 0]], [[0, 0, 1]], 2, rng="table", table=table)
    np.testing.assert_allclose(k1[0], [0.5, 0.0, 0.0], atol=1e-6)
    np.testing.assert_allclose(k2[0], [0.5, 0.0, 0.25], atol=1e-6)


def test_biased_background_fills_the_rest(backend):
    """Front accepted, back rejected, k=4: half red, half background (:285-291)."""
    a = two_layer_scene()
    out = backend.biased(a, [[0, 0, 0]], [[0, 0, 1]], 4, rng="table", table=np.array([[0.1], [0.9]]),
                         background=(0.0, 1.0, 0.0))
    np.testing.assert_allclose(out[0], [0.5, 0.5, 0.0], atol=1e-6)


def test_biased_all_accepted_is_exact_composite(backend):
    """Every candidate accepted (u = 0) and k above the candidate count: the
    biased composite IS the exact sorted composite (kernels.py:441-518)."""
    a = random_cloud(500, seed=41, sh_degree=2)
    o, d = random_rays(np.random.default_rng(9), 300)
    bg = (0.15, 0.25, 0.35)
    got = backend.biased(a, o, d, 200, rng="table", table=np.zeros((500, 1)), background=bg)
    want = backend.exact(a, o, d, background=bg)
    np.testing.assert_allclose(got, want, atol=2e-5)


def test_biased_counter_k_nesting(backend):
    """One draw per candidate, independent of k: k composites a prefix of the
    same accepted list, so a ray whose k=1 and k=8 results agree accepted at
    most one candidate and every larger k gives the same colour."""
    a = random_cloud(500, seed=41, sh_degree=0)
    o, d = random_rays(np.random.default_rng(4), 300)
    k1 = backend.biased(a, o, d, 1, seed=7)
    k8 = backend.biased(a, o, d, 8, seed=7)
    k99 = backend.biased(a, o, d, 99, seed=7)
    same = np.all(np.isclose(k1, k8), axis=1)
    assert np.isfinite(k99).all()
    assert same.mean() < 1.0  # some rays accept more than one candidate
    np.testing.assert_allclose(k8[same], k99[same], atol=1e-12)  # k1 == k8 -> at most one accepted
