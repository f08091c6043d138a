"""multi_gpu.PeerFrame: one frame in rank 0's device memory that every rank
maps with CUDA IPC and stores its tile shard into (the fused compute +
frame-assembly path of bench.py at N > 1).  On a one-GPU box the two ranks
share cuda:0 -- CUDA IPC between processes on one device takes the same
open/close path -- and synchronise on the host (gloo), so nothing waits on
the device for another rank's kernel."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_06598_b200 import RenderSettings, front_camera
        from paper_2504_06598_b200.multi_gpu import PeerFrame
        from paper_2504_06598_b200.render import prepare
        from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles
        from paper_2504_06598_b200.synthetic import random_cloud

        w, h = 200, 120
        S2 = 8.0
        asset = random_cloud(5_000, seed=11, sh_degree=1)
        st = RenderSettings(width=w, height=h, spp=1)
        sc = prepare(asset, st, device=0)
        cam = make_camera(camera_tuple(front_camera(), w, h))
        stream = torch.cuda.current_stream().cuda_stream
        pf = PeerFrame(w * h * 16, rank, 0)
        if not pf.ok:
            q.put(("unavailable", pf.error))
            return
        acc = torch.empty(shard_tiles(w, h) * 256 * 4, device="cuda")
        prm = make_render_params(w, h, 1, 1, 0, S2, shard_index=rank, shard_count=world)
        sc.render_pass_frame_device(cam, prm, 0, acc.data_ptr(), True, True, pf.ptr, rank > 0, stream)
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:

            class _View:  # the IPC frame (this process's device memory) seen by torch
                __cuda_array_interface__ = {"shape": (w * h * 4,), "typestr": "<f4", "data": (pf.ptr, False),
                                            "version": 3}

            frame = torch.as_tensor(_View(), device="cuda")
            full = torch.zeros(w * h * 4, device="cuda")
            sc.render_pass_device(cam, make_render_params(w, h, 1, 1, 0, S2), 0, acc.data_ptr(), True, True,
                                  full.data_ptr(), stream)
            torch.cuda.synchronize()
            q.put(("ok", bool(torch.equal(frame, full)), float(full[3::4].mean())))
        dist.barrier()
        pf.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_store_into_one_ipc_frame():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    if res[0] == "unavailable":
        pytest.skip(f"CUDA IPC unavailable on this box: {res[1]}")
    assert all(p.exitcode == 0 for p in procs)
    assert res[1], "frame assembled from two ranks differs from the single-GPU frame"
    assert res[2] > 0.0
