"""At-scale parity of the exact code paths the benchmark times, against the
counter-mode oracle on strided pixel grids (BASELINE.json configs at full
size; north-star gates: accepted ids agree on >= 99.9% of rays, colours of
agreeing rays within 1e-4 relative, 1024-spp converged means >= 45 dB).

* C3-target (the headline): 1M density-preserving SH-3 cloud, 1920x1080,
  1 spp, N = 1, through BOTH timed paths -- ``render()`` (the e2e leg: the
  fused walk+shade stores the f64 frame into mapped host memory) and
  ``srt_render_pass_device`` (the device-resident leg, float4 means) -- with
  no slot ids requested, so the fused single-pass store is what is checked.
* C4: 3M cloud, 3840x2160, 4 spp (one-launch fixed-point frame), and the same
  frame tile-sharded over 4 "devices" (interleaved 16x16 tiles) bit for bit.
* C5: 6M cloud, 1080p, 1024 spp against the committed oracle fixture
  (oracle/gen_scale_fixtures.py).

A pixel "agrees" when its colour is within 1e-4 relative (+1e-6 absolute for
clamped-at-zero SH channels, kernels.py:250-255) and its opacity is equal:
with N = 1 and one pass that is exactly the accepted-id agreement.
"""

import numpy as np
import pytest

from conftest import CUTOFF, GOLDEN, S2

pytestmark = pytest.mark.gpu

AGREE = 0.999
RTOL, ATOL = 1e-4, 1e-6


def _oracle_frame(O, asset, w, h, passes, stride, nslots=1, seed=0):
    from paper_2504_06598_b200.scene import camera_tuple
    from paper_2504_06598_b200.synthetic import front_camera

    lo, hi = asset.aabb_arrays(CUTOFF)
    pk = asset.packed
    ct = np.array(camera_tuple(front_camera(), w, h))
    r = O.render(O.sah_build(lo, hi), pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, ct, w, h,
                 passes=passes, nslots=nslots, s2=S2, seed=seed, rng="counter", stride=stride)
    sub = (slice(None, None, stride[1]), slice(None, None, stride[0]))
    return r["rgb"][sub], r["opacity"][sub], sub


def _agreement(rgb, op, ref_rgb, ref_op, op_tol=0.0):
    ok = np.all(np.abs(rgb - ref_rgb) <= RTOL * np.abs(ref_rgb) + ATOL, axis=-1)
    ok &= np.abs(op - ref_op) <= op_tol
    return float(ok.mean())


@pytest.fixture(scope="module")
def c3_asset():
    from paper_2504_06598_b200.synthetic import density_cloud

    return density_cloud(1_000_000, seed=0, sh_degree=3)


def test_c3target_render_api_vs_oracle(oracle, c3_asset):
    """The e2e leg of bench.py: render() at C3-target, no ids requested."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, render

    st = RenderSettings(width=1920, height=1080, spp=1, multisample=1)
    buf = render(c3_asset, front_camera(), st)
    ref_rgb, ref_op, sub = _oracle_frame(oracle, c3_asset, 1920, 1080, 1, (8, 8))
    agree = _agreement(buf.rgb[sub], buf.opacity[sub], ref_rgb, ref_op)
    assert agree >= AGREE, agree
    assert 0.5 < buf.opacity.mean() < 0.9  # ~68% of rays hit


def test_c3target_device_pass_vs_oracle(oracle, c3_asset):
    """The device-resident leg of bench.py: srt_render_pass_device (fused walk
    + SH shade + accumulate, float4 means in HBM), as timed."""
    import torch

    from paper_2504_06598_b200 import RenderSettings, front_camera
    from paper_2504_06598_b200.render import prepare
    from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles

    W, H = 1920, 1080
    st = RenderSettings(width=W, height=H, spp=1, multisample=1)
    sc = prepare(c3_asset, st)
    cam = make_camera(camera_tuple(front_camera(), W, H))
    prm = make_render_params(W, H, 1, 1, 0, S2)
    acc = torch.empty(shard_tiles(W, H) * 256 * 4, device="cuda")
    out = torch.zeros(W * H * 4, device="cuda")
    sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    sc.check_status()
    f = out.cpu().numpy().reshape(H, W, 4).astype(np.float64)
    ref_rgb, ref_op, sub = _oracle_frame(oracle, c3_asset, W, H, 1, (8, 8))
    agree = _agreement(f[sub][..., :3], f[sub][..., 3], ref_rgb, ref_op)
    assert agree >= AGREE, agree


@pytest.fixture(scope="module")
def c4_asset():
    from paper_2504_06598_b200.synthetic import density_cloud

    return density_cloud(3_000_000, seed=0, sh_degree=3)


def test_c4_3m_4k_4spp_vs_oracle(oracle, c4_asset):
    """configs[3]: 3M Gaussians, 3840x2160, 4 spp (one launch over every
    (packet, pass), 2^-32 fixed-point sums) on a 32x32-strided grid."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, render

    st = RenderSettings(width=3840, height=2160, spp=4, multisample=1)
    buf = render(c4_asset, front_camera(), st)
    assert buf.spp == 4
    ref_rgb, ref_op, sub = _oracle_frame(oracle, c4_asset, 3840, 2160, 4, (32, 32))
    agree = _agreement(buf.rgb[sub], buf.opacity[sub], ref_rgb, ref_op, op_tol=1e-12)
    assert agree >= AGREE, agree


def test_c4_tile_shards_equal_single_gpu(c4_asset):
    """The C4 tile sharding (16x16 tile t -> shard t % G, G = 4) rendered
    shard by shard and resolved into one frame equals the single-GPU frame
    bit for bit (exact integer sums; every shard's samples keyed per pixel)."""
    from paper_2504_06598_b200 import RenderSettings, front_camera, render

    st = RenderSettings(width=3840, height=2160, spp=4, multisample=1)
    one = render(c4_asset, front_camera(), st)
    many = render(c4_asset, front_camera(), st, devices=[0, 0, 0, 0])
    np.testing.assert_array_equal(many.rgb, one.rgb)
    np.testing.assert_array_equal(many.opacity, one.opacity)


def test_c5_6m_1024spp_converged_vs_oracle_fixture():
    """configs[4]: 6M Gaussians, 1080p, 1024 spp in one launch; the 16x16 grid
    of the converged mean against the oracle's counter-mode fixture at
    >= 45 dB (image_metrics, render.py:177-195), and beside it the
    reference's own trig-stream converged output (independent stream:
    Monte-Carlo noise of 1024 samples bounds that PSNR)."""
    from paper_2504_06598_b200 import AccumBuffer, RenderSettings, front_camera, image_metrics, render
    from paper_2504_06598_b200.synthetic import density_cloud

    fx = np.load(GOLDEN / "c5_converged_grid.npz")
    n, w, h, spp, stride = (int(fx[k]) for k in ("n", "width", "height", "spp", "stride"))
    asset = density_cloud(n, seed=0, sh_degree=3)
    buf = render(asset, front_camera(), RenderSettings(width=w, height=h, spp=spp, multisample=1))
    sub = (slice(None, None, stride), slice(None, None, stride))
    got = AccumBuffer(buf.rgb[sub], buf.opacity[sub], spp)
    same = image_metrics(got, AccumBuffer(fx["counter_rgb"], fx["counter_opacity"], spp))
    ref = image_metrics(got, AccumBuffer(fx["trig_rgb"], fx["trig_opacity"], spp))
    print(f"C5 1024 spp: same stream {same['psnr']:.2f} dB, reference trig stream {ref['psnr']:.2f} dB")
    assert same["psnr"] >= 45.0, same
    # independent streams agree only to the noise of 1024 samples: the oracle measures 41.0 dB
    # between its own counter and trig images (oracle/gen_scale_fixtures.py)
    assert ref["psnr"] >= 38.0, ref
