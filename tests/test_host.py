"""Host-side logic of the drop-in surface (no GPU): input types, generators,
packing, jitter and counter stream, camera, metrics, ABI exports."""

import hashlib
import math
import re

import numpy as np
import pytest

from conftest import CUTOFF, ROOT
from paper_2504_06598_b200 import (AccumBuffer, CameraConfig, ConfigError, RenderSettings, SplatAsset,
                                   camera_basis, counter_uniform, generate_camera_ray, image_metrics, pixel_jitter)
from paper_2504_06598_b200.synthetic import density_factor, front_camera, random_cloud, two_layer_scene


def _digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name,kw", [
    ("c1_10k_sh0", dict(n=10_000, seed=0, sh_degree=0)),
    ("c2_100k_sh3_density", dict(n=100_000, seed=0, sh_degree=3,
                                 scale_range=(0.02 * density_factor(100_000), 0.25 * density_factor(100_000)))),
    ("small_400_s31", dict(n=400, seed=31)),
])
def test_synthetic_and_packing_match_reference(golden, name, kw):
    """random_cloud, .packed and aabb_arrays reproduce the reference's arrays
    bit for bit (digests from oracle/gen_golden.py)."""
    g = golden("assets")
    a = random_cloud(**kw)
    assert _digest(a.means, a.rotations, a.scales, a.opacities, a.sh) == str(g[f"{name}__asset"])
    pk = a.packed
    assert _digest(pk.means, pk.cov_inv6, pk.opacities, pk.sh) == str(g[f"{name}__packed"])
    lo, hi = a.aabb_arrays(CUTOFF)
    assert _digest(lo, hi) == str(g[f"{name}__aabb"])


def test_pixel_jitter_golden(golden):
    g = golden("sampling")
    jit = np.array([pixel_jitter((a[0], a[1]), int(a[2]), int(a[3])) for a in g["jitter_args"]])
    np.testing.assert_array_equal(jit, g["jitter"])
    np.testing.assert_array_equal(pixel_jitter((3, 5), 0), [0.27136341482400894, 0.6206638417206705])
    with pytest.raises(ValueError, match="frame"):
        pixel_jitter((0, 0), -1)


def test_counter_uniform_matches_oracle(oracle):
    rs = np.random.default_rng(3)
    args = rs.integers(0, 2**32, size=(500, 4), dtype=np.uint64)
    want = np.array([oracle.counter_u(oracle.walk_key(int(s), int(r), int(k)), int(p)) for s, r, k, p in args])
    got = np.array([counter_uniform(int(s), int(r), int(k), int(p)) for s, r, k, p in args])
    np.testing.assert_array_equal(got, want)


class TestSettings:
    def test_defaults_and_passes(self):
        st = RenderSettings(spp=10, multisample=4)
        assert st.passes == 3 and st.samples_per_pixel == 12
        assert st.cutoff_s == pytest.approx(2 * math.sqrt(2))

    @pytest.mark.parametrize("kw", [dict(width=0), dict(spp=0), dict(depth_mode="peak"), dict(multisample=257),
                                    dict(cutoff_s=-1.0), dict(background=[-1, 0, 0])])
    def test_invalid(self, kw):
        with pytest.raises(ConfigError):
            RenderSettings(**kw)

    def test_camera_validation(self):
        with pytest.raises(ConfigError):
            CameraConfig(position=[0, 0, 0], look_at=[0, 0, 0])
        with pytest.raises(ConfigError):
            CameraConfig(position=[0, 0, -1], fov_deg=180)


class TestAsset:
    def test_validation(self):
        with pytest.raises(ValueError):
            SplatAsset(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3, 1)))
        with pytest.raises(ValueError, match="scales"):
            SplatAsset(np.zeros((1, 3)), [[1, 0, 0, 0]], [[1, 0, 1]], [0.5], np.zeros((1, 3, 1)))
        with pytest.raises(ValueError, match="opacities"):
            SplatAsset(np.zeros((1, 3)), [[1, 0, 0, 0]], [[1, 1, 1]], [1.5], np.zeros((1, 3, 1)))

    def test_quaternions_normalised(self):
        a = SplatAsset(np.zeros((1, 3)), [[2, 0, 0, 0]], [[1, 1, 1]], [0.5], np.zeros((1, 3, 4)))
        np.testing.assert_allclose(a.rotations, [[1, 0, 0, 0]])
        assert a.sh_degree == 1

    def test_packed_inverse(self):
        a = random_cloud(50, seed=2)
        pk = a.packed
        cov = np.einsum("nij,nj,nkj->nik", pk.rot, a.scales**2, pk.rot)
        np.testing.assert_allclose(np.einsum("nij,njk->nik", cov, pk.cov_inv), np.tile(np.eye(3), (50, 1, 1)),
                                   atol=1e-8)

    def test_aabb_contains_ellipsoid_extent(self):
        """The rotated-box AABB contains the tight ellipsoid AABB the GPU LBVH uses."""
        a = random_cloud(200, seed=4)
        lo, hi = a.aabb_arrays(CUTOFF)
        cov = np.linalg.inv(a.packed.cov_inv)
        half = CUTOFF * np.sqrt(np.einsum("nii->ni", cov))
        assert np.all(a.means - half >= lo - 1e-12) and np.all(a.means + half <= hi + 1e-12)


class TestCamera:
    def test_basis_orthonormal(self):
        cam = CameraConfig(position=[2, 1, -5], look_at=[0, 0.3, 0])
        fwd, right, up = camera_basis(cam)
        for v in (fwd, right, up):
            assert np.linalg.norm(v) == pytest.approx(1.0)
        np.testing.assert_allclose(np.cross(right, fwd), up, atol=1e-12)
        with pytest.raises(ValueError, match="parallel"):
            camera_basis(CameraConfig(position=[0, -5, 0], up=[0, 1, 0]))

    def test_ray_matches_oracle_formula(self, oracle):
        """generate_camera_ray == the 14-scalar camera of the kernel boundary."""
        cam = CameraConfig(position=[0.5, -1, -6], look_at=[0, 0, 1], fov_deg=48)
        st = RenderSettings(width=40, height=30, seed=3)
        o, d = generate_camera_ray(cam, st, (13, 22), 5)
        ct = oracle.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, 40, 30)
        jx, jy = oracle.pixel_jitter(13, 22, 5, 3)
        u = 2.0 * (13 + jx) / 40 - 1.0
        v = 1.0 - 2.0 * (22 + jy) / 30
        dd = ct[9:12] + u * ct[12] * ct[3:6] + v * ct[13] * ct[6:9]
        np.testing.assert_allclose(d, dd / np.linalg.norm(dd), rtol=1e-14)
        np.testing.assert_array_equal(o, cam.position)
        with pytest.raises(ValueError, match="outside"):
            generate_camera_ray(cam, st, (40, 0), 0)


def test_accum_buffer_and_metrics():
    with pytest.raises(ValueError, match="shapes"):
        AccumBuffer(np.zeros((4, 4, 3)), np.zeros((4, 5)), 1)
    with pytest.raises(ValueError, match="positive"):
        AccumBuffer(np.zeros((4, 4, 3)), np.zeros((4, 4)), 0)
    a = AccumBuffer(np.full((2, 3, 3), 0.5), np.ones((2, 3)), 4)
    b = AccumBuffer(np.full((2, 3, 3), 0.6), np.ones((2, 3)), 4)
    assert a.width == 3 and a.height == 2
    m = image_metrics(a, b)
    assert m["mse"] == pytest.approx(0.01)
    assert m["psnr"] == pytest.approx(20.0)
    assert image_metrics(a, a)["psnr"] == math.inf


def test_abi_header_symbols_exported():
    """libsrt.so loads and exports every entry point include/srt.h declares; the
    ctypes binding covers all of them (no compute calls: no GPU here)."""
    header = (ROOT / "include" / "srt.h").read_text()
    declared = set(re.findall(r"\b(srt_[a-z0-9_]+)\s*\(", header))
    from paper_2504_06598_b200 import _lib

    bound = {name for name, _, _ in _lib.SYMBOLS}
    assert declared == bound, declared ^ bound
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.srt_version()


def test_product_has_no_oracle_import():
    """The product package never imports the oracle (it is only the checker)."""
    for p in (ROOT / "paper_2504_06598_b200").rglob("*.py"):
        src = p.read_text()
        assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", src), p


def test_two_layer_closed_form():
    a = two_layer_scene()
    assert len(a) == 2 and a.sh_degree == 0
    cam = front_camera()
    assert cam.fov_deg == 45.0


def test_biased_k_must_be_positive():
    """tracer.py:325-326: k < 1 is a ValueError, raised before any device work."""
    from paper_2504_06598_b200 import kernels

    z = np.zeros((1, 3))
    with pytest.raises(ValueError, match="k"):
        kernels.biased_batch(z, np.zeros((1, 6)), np.zeros(1), np.zeros((1, 3, 1)), 0, z, z + [0, 0, 1], 0.0, 1.0,
                             0, 8.0, 0, 0.0, 0.0, 0.0, np.zeros((1, 3)))
