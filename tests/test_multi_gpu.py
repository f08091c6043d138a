"""Multi-GPU driver host logic (paper_2504_06598_b200/multi_gpu.py), run on CPU:
tile ownership, compact-buffer pixel order, pass ranges, assembly, and a
world_size-2 gloo run of the same gather the NCCL path does.  The per-rank
renderer here is the CPU oracle (checker), standing in for libsrt."""

import os
import socket

import numpy as np
import pytest

from conftest import S2
from paper_2504_06598_b200 import multi_gpu as mg


@pytest.mark.parametrize("w,h,world", [(64, 64, 2), (70, 50, 3), (1920, 1080, 8), (17, 5, 4)])
def test_tiles_partition_the_frame(w, h, world):
    seen = np.zeros((h, w), np.int64)
    for r in range(world):
        px, py, ok = mg.compact_pixels(w, h, r, world)
        assert px.shape[0] <= mg.max_shard_tiles(w, h, world) * 256
        np.add.at(seen, (py[ok], px[ok]), 1)
    assert np.all(seen == 1)


def test_assemble_roundtrip():
    rs = np.random.default_rng(0)
    w, h, world = 70, 50, 3
    frame = rs.random((h, w, 4)).astype(np.float32)
    bufs = []
    n = mg.max_shard_tiles(w, h, world) * 256
    for r in range(world):
        px, py, ok = mg.compact_pixels(w, h, r, world)
        b = np.zeros((n, 4), np.float32)
        b[: px.shape[0]][ok] = frame[py[ok], px[ok]]
        bufs.append(b)
    np.testing.assert_array_equal(mg.assemble_tiles(bufs, w, h), frame)


def test_pass_ranges_and_combine():
    for passes in (1, 7, 1024):
        for world in (1, 2, 3, 8):
            rngs = [mg.pass_range(passes, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == passes
            assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
    means = [np.full(3, 1.0), np.full(3, 4.0)]
    np.testing.assert_allclose(mg.combine_samples(means, [1, 3]), np.full(3, 3.25))
    with pytest.raises(ValueError):
        mg.plan("rows", 0, 1, 4, 4, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2504_06598_b200.synthetic import front_camera, random_cloud

        asset = random_cloud(800, seed=4, sh_degree=1)
        pk = asset.packed
        lo, hi = asset.aabb_arrays(np.sqrt(S2))
        b = O.sah_build(lo, hi)
        w, h, passes = 40, 24, 5
        cam = front_camera()
        ct = O.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, w, h)

        def shard_render(p):
            if p.mode == "tiles" and p.world == 1:
                full = O.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 1, ct, w, h, passes=passes, s2=S2,
                                seed=3, rng="counter")
                return torch.from_numpy(np.dstack([full["rgb"], full["opacity"]]).astype(np.float32).reshape(-1, 4))
            if p.mode == "tiles":
                full = O.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 1, ct, w, h, passes=passes, s2=S2,
                                seed=3, rng="counter")
                rgba = np.dstack([full["rgb"], full["opacity"]]).astype(np.float32)
                px, py, ok = mg.compact_pixels(w, h, p.rank, p.world)
                buf = np.zeros((p.buffer_pixels, 4), np.float32)
                buf[: px.shape[0]][ok] = rgba[py[ok], px[ok]]
                return torch.from_numpy(buf)
            part = O.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 1, ct, w, h, passes=p.local_passes,
                            pass0=p.pass0, s2=S2, seed=3, rng="counter")
            return torch.from_numpy(np.dstack([part["rgb"], part["opacity"]]).astype(np.float32).reshape(-1, 4))

        p = mg.plan(mode, rank, world, w, h, passes)
        frame = mg.render_frame(p, shard_render)
        if rank == 0:
            ref = O.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 1, ct, w, h, passes=passes, s2=S2, seed=3,
                           rng="counter")
            want = np.dstack([ref["rgb"], ref["opacity"]])
            q.put(float(np.abs(frame.numpy() - want).max()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["tiles", "samples"])
def test_gloo_world2_gather_matches_single_render(mode):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
        assert pr.exitcode == 0
    err = q.get(timeout=5)
    assert err <= 1e-6, err


def _sums_worker(rank, world, port, mode, q):
    """Fixed-point-sum frames over gloo: per-sample colours from the oracle,
    2^-32 integer sums per rank, gathered ("tiles") or reduced ("samples")."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2504_06598_b200.synthetic import front_camera, random_cloud

        asset = random_cloud(800, seed=4, sh_degree=1)
        pk = asset.packed
        lo, hi = asset.aabb_arrays(np.sqrt(S2))
        b = O.sah_build(lo, hi)
        w, h, passes = 40, 24, 5
        cam = front_camera()
        ct = O.camera_tuple(cam.position, cam.look_at, cam.up, cam.fov_deg, w, h)
        per_pass = []
        for f in range(passes):
            r = O.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 1, ct, w, h, passes=1, pass0=f, s2=S2,
                         seed=3, rng="counter")
            fx = np.rint(np.dstack([r["rgb"], np.zeros((h, w))]) * mg.FIXED_ONE).astype(np.int64)
            fx[..., 3] = np.rint(r["opacity"]).astype(np.int64) << 32
            per_pass.append(fx)

        def compact(frame_sums, r, g):
            px, py, ok = mg.compact_pixels(w, h, r, g)
            buf = np.zeros((mg.max_shard_tiles(w, h, g) * 256, 4), np.int64)
            buf[: px.shape[0]][ok] = frame_sums[py[ok], px[ok]]
            return buf

        def shard_sums(p):
            if p.mode == "tiles":
                return torch.from_numpy(compact(sum(per_pass), p.rank, p.world))
            a, e = mg.pass_range(p.passes, p.rank, p.world)
            part = sum(per_pass[a:e]) if e > a else np.zeros((h, w, 4), np.int64)
            return torch.from_numpy(compact(part, 0, 1))

        p = mg.plan(mode, rank, world, w, h, passes)
        frame = mg.render_frame_sums(p, shard_sums, 1)
        if rank == 0:
            single = np.zeros((h, w, 4))
            mg.resolve_sums(compact(sum(per_pass), 0, 1), w, h, 0, 1, passes, 1, single)
            ref = O.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 1, ct, w, h, passes=passes, s2=S2, seed=3,
                           rng="counter")
            want = np.dstack([ref["rgb"], ref["opacity"]])
            q.put((bool(np.array_equal(frame.numpy(), single)), float(np.abs(frame.numpy() - want).max())))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["tiles", "samples"])
def test_gloo_world2_fixed_point_sums_are_bitwise_single_frame(mode):
    """render_frame_sums (the GPU driver's multi-pass path): integer sums make
    the world-2 frame bit for bit the one-rank frame, in both shardings."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sums_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
        assert pr.exitcode == 0
    same, err = q.get(timeout=5)
    assert same
    assert err <= 1e-9, err


def _shared_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, h = 70, 50
        pool = mg.SharedFramePool(register=False)
        keys = []

        def write(p, rgb, op):
            # each rank writes exactly its own tiles (as srt_render does for a shard)
            px, py, ok = mg.compact_pixels(p.width, p.height, p.rank, p.world)
            rgb[py[ok], px[ok]] = [p.rank + 1.0, frame_no, 0.5]
            op[py[ok], px[ok]] = p.rank + 1.0

        results = []
        for frame_no in range(3):
            p = mg.plan("tiles", rank, world, w, h, 1)
            got = mg.render_frame_shared(p, write, pool)
            if rank == 0:
                rgb, op = got
                results.append((rgb.copy(), op.copy()))
                keys.append(rgb.__array_interface__["data"][0])
                if frame_no == 0:
                    keep = got  # frame 0 stays referenced: frame 1 must use another block
                del got, rgb, op
        if rank == 0:
            q.put((results, keys))
        dist.barrier()
        pool.close()
    finally:
        dist.destroy_process_group()


def test_gloo_world3_shared_host_frame_assembles_every_tile():
    """multi_gpu.SharedFramePool / render_frame_shared (the multi-GPU e2e path)
    with gloo at world size 3: every rank writes only its tiles into one
    POSIX-shared frame; rank 0 sees the whole frame, blocks still referenced
    by a returned frame are not reused, released ones are."""
    import multiprocessing as mp

    world, port = 3, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shared_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results, keys = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w, h = 70, 50
    owner = np.zeros((h, w))
    for r in range(world):
        px, py, ok = mg.compact_pixels(w, h, r, world)
        owner[py[ok], px[ok]] = r + 1.0
    for i, (rgb, op) in enumerate(results):
        np.testing.assert_array_equal(op, owner)
        np.testing.assert_array_equal(rgb[..., 0], owner)
        assert np.all(rgb[..., 1] == i)
    assert keys[1] != keys[0]  # frame 0 was still referenced
    assert keys[2] == keys[1]  # frame 1 was released and reused
