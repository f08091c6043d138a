"""The closest-hit walks' spatially split tree (csrc/split.cu).

PLOC builds of >= 16,384 primitives give the closest-hit walks (packets, per
lane, cooperative) a tree over leaf references clipped at a uniform cell grid.
A duplicated reference evaluates the same primitive with the same (ray, slot,
primitive) draw, so the closest accepted hit of every slot must be the
unsplit tree's (LBVH builds and uploaded reference BVHs have none): ids and
shaded frames bit for bit, depths to the screen's tolerance.  The oracle
parity tests at scale (test_gpu_scale.py, test_gpu_parity.py) run on it too.
"""

import numpy as np
import pytest

from conftest import CUTOFF, S2

pytestmark = pytest.mark.gpu


def _scenes(asset):
    from paper_2504_06598_b200.scene import DeviceScene

    a = DeviceScene.from_packed(asset.packed)
    a.build_bvh(CUTOFF)  # PLOC: split tree for the packet walk
    b = DeviceScene.from_packed(asset.packed)
    b.build_bvh(CUTOFF, method="lbvh")  # no split tree
    return a, b


def _frame(sc, w, h, passes=1, nslots=1, mode=0, want_ids=True, seed=0):
    from paper_2504_06598_b200 import front_camera
    from paper_2504_06598_b200.scene import camera_tuple

    ct = camera_tuple(front_camera(), w, h)
    return sc.render(ct, w, h, passes, nslots, mode, S2, True, seed, (0.1, 0.2, 0.3), want_ids=want_ids)


def test_split_tree_is_built_for_ploc_scenes_only():
    from paper_2504_06598_b200.synthetic import density_cloud, random_cloud

    a, b = _scenes(density_cloud(50_000, seed=4))
    info = a.split_info()
    assert info["cells"] >= 2 and info["num_refs"] >= 50_000 and info["num_nodes4"] > 0
    assert info["num_refs"] < 4 * 50_000
    assert b.split_info() == {"num_refs": 0, "num_nodes4": 0, "cells": 0}
    small = a.__class__.from_packed(random_cloud(2_000, seed=1).packed)
    small.build_bvh(CUTOFF)
    assert small.split_info()["num_refs"] == 0
    for s in (a, b, small):
        s.close()


@pytest.mark.parametrize("nslots,mode,passes", [(1, 0, 1), (4, 0, 1), (1, 1, 1), (2, 0, 3)])
def test_split_tree_frames_equal_unsplit_bitwise(nslots, mode, passes):
    """Fused frames (no ids: the bench path) and id frames (pass 0 ids) on the
    split tree equal the LBVH tree's bit for bit."""
    from paper_2504_06598_b200.synthetic import density_cloud

    a, b = _scenes(density_cloud(120_000, seed=7))
    w, h = 320, 200
    ra = _frame(a, w, h, passes, nslots, mode, want_ids=False)
    rb = _frame(b, w, h, passes, nslots, mode, want_ids=False)
    np.testing.assert_array_equal(ra[0], rb[0])
    np.testing.assert_array_equal(ra[1], rb[1])
    ia = _frame(a, w, h, 1, nslots, mode, want_ids=True)[2]
    ib = _frame(b, w, h, 1, nslots, mode, want_ids=True)[2]
    np.testing.assert_array_equal(ia, ib)
    assert (ia >= 0).mean() > 0.2  # the frame hits the cloud
    a.close()
    b.close()


def test_split_tree_with_degenerate_primitives():
    """Unbounded boxes of degenerate primitives land in every cell; the walk
    still skips them and matches the unsplit tree."""
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import density_cloud

    pk = density_cloud(30_000, seed=3).packed
    cov = pk.cov_inv6.copy()
    bad = np.arange(0, 30_000, 997)
    cov[bad[0::2]] = 0.0
    cov[bad[1::2], 0] = np.nan
    a = DeviceScene(pk.means, cov, pk.opacities, pk.sh, pk.sh_degree)
    a.build_bvh(CUTOFF)
    b = DeviceScene(pk.means, cov, pk.opacities, pk.sh, pk.sh_degree)
    b.build_bvh(CUTOFF, method="lbvh")
    assert a.split_info()["num_refs"] >= 30_000
    ia = _frame(a, 256, 160)[2]
    ib = _frame(b, 256, 160)[2]
    np.testing.assert_array_equal(ia, ib)
    assert not np.isin(ia, bad).any()
    a.close()
    b.close()


# Depths: a candidate the fp32 screen decides is accepted at the screen depth,
# one the screen cannot decide (its far bound depends on the visit order) at
# the exact stage's depth, ~1e-7 relative apart: the ids
# are order-independent, the depths equal to that tolerance.
T_RTOL = 2e-6


@pytest.mark.parametrize("kind,nslots", [("hemisphere", 2), ("hemisphere", 1), ("random", 1), ("random", 4)])
def test_split_tree_explicit_rays_equal_unsplit(kind, nslots):
    """Explicit-ray batches on the split tree -- one-hemisphere batches as
    packets with per-lane origins, incoherent ones per lane (single slot) or
    cooperatively (several slots) -- equal the unsplit tree's."""
    from conftest import random_rays
    from paper_2504_06598_b200.synthetic import density_cloud

    a, b = _scenes(density_cloud(60_000, seed=2))
    rng = np.random.default_rng(5)
    R = 50_000
    if kind == "hemisphere":
        o = np.column_stack([rng.uniform(-0.3, 0.3, R), rng.uniform(-0.3, 0.3, R), np.full(R, -4.0)])
        d = np.column_stack([rng.normal(0, 0.15, R), rng.normal(0, 0.15, R), np.ones(R)])
        d /= np.linalg.norm(d, axis=1, keepdims=True)
    else:
        o, d = random_rays(rng, R)
    ta, ida = a.trace_rays(o, d, nslots=nslots, seed=9)
    tb, idb = b.trace_rays(o, d, nslots=nslots, seed=9)
    np.testing.assert_array_equal(ida, idb)
    hit = ida >= 0
    assert hit.mean() > 0.1
    np.testing.assert_allclose(ta[hit], tb[hit], rtol=T_RTOL, atol=0)
    assert np.isinf(ta[~hit]).all() and np.isinf(tb[~hit]).all()
    a.close()
    b.close()


def test_split_tree_follows_the_bvh_lifecycle(oracle):
    """A rebuild with LBVH or an uploaded reference BVH drops the split tree
    (the walks then use the tree they were given); a PLOC rebuild restores it."""
    from paper_2504_06598_b200.scene import DeviceScene
    from paper_2504_06598_b200.synthetic import density_cloud

    asset = density_cloud(20_000, seed=8)
    sc = DeviceScene.from_packed(asset.packed)
    sc.build_bvh(CUTOFF)
    assert sc.split_info()["num_refs"] >= 20_000
    ref_ids = _frame(sc, 64, 48)[2]
    sc.build_bvh(CUTOFF, method="lbvh")
    assert sc.split_info()["num_refs"] == 0
    np.testing.assert_array_equal(_frame(sc, 64, 48)[2], ref_ids)
    lo, hi = asset.aabb_arrays(CUTOFF)
    sc.upload_bvh(oracle.sah_build(lo, hi))
    assert sc.split_info()["num_refs"] == 0
    np.testing.assert_array_equal(_frame(sc, 64, 48)[2], ref_ids)
    sc.build_bvh(CUTOFF)
    assert sc.split_info()["num_refs"] >= 20_000
    sc.close()


@pytest.mark.parametrize("w,h", [(37, 23), (161, 90)])
def test_split_tree_odd_frames_equal_unsplit(w, h):
    """Partial edge packets (per-lane f64 stores) on the split tree."""
    from paper_2504_06598_b200.render import PinnedPool
    from paper_2504_06598_b200.synthetic import density_cloud

    a, b = _scenes(density_cloud(40_000, seed=5))
    pool = PinnedPool()
    from paper_2504_06598_b200 import front_camera
    from paper_2504_06598_b200.scene import camera_tuple

    ct = camera_tuple(front_camera(), w, h)
    ra = a.render(ct, w, h, 1, 1, 0, S2, True, 3, (0.2, 0.1, 0.0), out_rgb=pool.array((h, w, 3)),
                  out_op=pool.array((h, w)))
    rb = b.render(ct, w, h, 1, 1, 0, S2, True, 3, (0.2, 0.1, 0.0), out_rgb=pool.array((h, w, 3)),
                  out_op=pool.array((h, w)))
    np.testing.assert_array_equal(ra[0], rb[0])
    np.testing.assert_array_equal(ra[1], rb[1])
    a.close()
    b.close()
