"""PLY ingest (ply.py) against files written and loaded by the reference
(assets.py:257-370; fixtures from oracle/gen_golden.py), plus the reference's
error cases (tests/test_assets.py:132-255)."""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2504_06598_b200 import EmptyAssetError, PlyFormatError, load_ply, save_ply
from paper_2504_06598_b200.synthetic import random_cloud


@pytest.mark.parametrize("tag,fname", [("bin", "splats_300_sh3.ply"), ("ascii", "splats_60_sh1_ascii.ply")])
def test_load_matches_reference(golden, tag, fname):
    g = golden("ply_loaded")
    a = load_ply(GOLDEN / fname)
    for f in ("means", "rotations", "scales", "opacities", "sh"):
        np.testing.assert_array_equal(getattr(a, f), g[f"{tag}_{f}"], err_msg=f)


def test_save_is_byte_identical_to_reference(tmp_path):
    a = random_cloud(300, seed=5, sh_degree=3)
    save_ply(a, tmp_path / "x.ply", binary=True)
    assert (tmp_path / "x.ply").read_bytes() == (GOLDEN / "splats_300_sh3.ply").read_bytes()
    b = random_cloud(60, seed=6, sh_degree=1)
    save_ply(b, tmp_path / "y.ply", binary=False)
    assert (tmp_path / "y.ply").read_bytes() == (GOLDEN / "splats_60_sh1_ascii.ply").read_bytes()


def _write(path, header_lines, body=b""):
    path.write_bytes(("\n".join(header_lines) + "\n").encode() + body)


def test_errors(tmp_path):
    p = tmp_path / "bad.ply"
    _write(p, ["plx"])
    with pytest.raises(PlyFormatError, match="magic"):
        load_ply(p)
    _write(p, ["ply", "format binary_big_endian 1.0", "element vertex 1", "end_header"])
    with pytest.raises(PlyFormatError, match="unsupported format"):
        load_ply(p)
    _write(p, ["ply", "format ascii 1.0", "element vertex 0", "property float x", "end_header"])
    with pytest.raises(EmptyAssetError):
        load_ply(p)
    _write(p, ["ply", "format ascii 1.0", "element vertex 1", "property list uchar int idx", "end_header"])
    with pytest.raises(PlyFormatError, match="list"):
        load_ply(p)
    _write(p, ["ply", "format ascii 1.0", "element vertex 1", "property float x", "end_header"], b"1.0\n")
    with pytest.raises(PlyFormatError, match="missing vertex property"):
        load_ply(p)


def test_tiny_scales_clamped_and_roundtrip(tmp_path):
    a = random_cloud(50, seed=2, sh_degree=2)
    a.scales[0] = 1e-30
    save_ply(a, tmp_path / "t.ply")
    b = load_ply(tmp_path / "t.ply")
    extent = float(np.linalg.norm(b.means.max(axis=0) - b.means.min(axis=0)))
    assert b.scales[0].min() >= 1e-8 * extent * (1 - 1e-12)
    np.testing.assert_allclose(b.means, a.means, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(b.opacities, a.opacities, rtol=1e-5, atol=1e-6)
    assert b.sh_degree == 2


@pytest.mark.gpu
def test_gpu_packing_matches_host_packing():
    """srt_scene_create_from_splats (closed-form A = R diag(1/s^2) R^T on the
    GPU) vs asset.packed (numpy inverse): same frame ids on a 50k scene."""
    from paper_2504_06598_b200 import RenderSettings, front_camera
    from paper_2504_06598_b200.scene import DeviceScene, camera_tuple

    a = load_ply(GOLDEN / "splats_300_sh3.ply")
    big = random_cloud(50_000, seed=3, sh_degree=3)
    st = RenderSettings(width=96, height=64, spp=2, multisample=2)
    ct = camera_tuple(front_camera(), st.width, st.height)
    outs = []
    for asset in (a, big):
        for gpu_pack in (False, True):
            sc = DeviceScene.from_splats(asset) if gpu_pack else DeviceScene.from_packed(asset.packed)
            sc.build_bvh(st.cutoff_s)
            outs.append(sc.render(ct, st.width, st.height, st.passes, 2, 0, st.cutoff_s ** 2, want_ids=True))
    for host, gpu in ((outs[0], outs[1]), (outs[2], outs[3])):
        assert np.mean(host[2] == gpu[2]) >= 0.999
        np.testing.assert_allclose(host[0], gpu[0], rtol=1e-3, atol=1e-3)
