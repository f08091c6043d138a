"""Multi-GPU frame driver: one process per GPU, scene replicated, work sharded,
one NCCL collective per frame.

Two shardings, both with no exchange during tracing:

* ``"tiles"``   16x16 tiles interleaved over ranks (tile t -> rank t % G).
  Interleaving balances the dense centre of the cloud against the empty
  border.  Each rank writes its tiles into a tile-compact buffer
  ``(max_tiles * 256, 4)``; rank 0 gathers the G buffers with one
  ``torch.distributed.gather`` (NCCL over NVLink) and scatters them into the
  frame (``srt_unpack_tiles_device`` on the GPU).
* ``"samples"`` passes split into contiguous ranges (rank r traces passes
  [P r / G, P (r + 1) / G)).  The counter RNG is keyed on the GLOBAL pass
  index, so every sample is the one the single-GPU render draws.  Rank 0
  gathers the per-rank partial means and combines them in rank order (a
  fixed-order sum, so the result does not depend on NCCL's reduction order).

The host-side bookkeeping (tile ownership, pixel order of the compact layout,
pass ranges, assembly) is plain numpy here so it can be exercised with the
gloo backend on CPU; the GPU path swaps in libsrt kernels for the per-rank
trace and the unpack.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

TILE = 16


# ---------------------------------------------------------------------------
# host-side bookkeeping (mirrors tile_pixel in csrc/trace.cu / shade.cu)
# ---------------------------------------------------------------------------

def tiles_xy(width: int, height: int) -> tuple[int, int]:
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


def shard_tile_ids(width: int, height: int, rank: int, world: int) -> np.ndarray:
    """Global 16x16 tile ids owned by `rank` (t % world == rank), in local order."""
    tx, ty = tiles_xy(width, height)
    return np.arange(rank, tx * ty, world, dtype=np.int64)


def max_shard_tiles(width: int, height: int, world: int) -> int:
    return len(shard_tile_ids(width, height, 0, world))


def compact_pixels(width: int, height: int, rank: int, world: int):
    """(px, py, valid) of each entry of the rank's tile-compact buffer: local
    tile j covers entries [256 j, 256 j + 256); inside a tile, warp w holds an
    8x4 block at ((w & 1) * 8, (w >> 1) * 4) and lane l its pixel (l & 7, l >> 3)."""
    tx, _ = tiles_xy(width, height)
    tiles = shard_tile_ids(width, height, rank, world)
    tid = np.arange(256)
    w, lane = tid >> 5, tid & 31
    ox = (w & 1) * 8 + (lane & 7)
    oy = (w >> 1) * 4 + (lane >> 3)
    px = ((tiles % tx) * TILE)[:, None] + ox[None, :]
    py = ((tiles // tx) * TILE)[:, None] + oy[None, :]
    px, py = px.reshape(-1), py.reshape(-1)
    return px, py, (px < width) & (py < height)


def assemble_tiles(gathered: list, width: int, height: int) -> np.ndarray:
    """Scatter G tile-compact (n, 4) buffers into a (H, W, 4) frame (CPU
    statement of srt_unpack_tiles_device)."""
    world = len(gathered)
    frame = np.zeros((height, width, 4), np.float32)
    for r, buf in enumerate(gathered):
        px, py, ok = compact_pixels(width, height, r, world)
        b = np.asarray(buf, np.float32).reshape(-1, 4)[: px.shape[0]]
        frame[py[ok], px[ok]] = b[ok]
    return frame


def pass_range(passes: int, rank: int, world: int) -> tuple[int, int]:
    """[first, last) global pass indices of `rank` under sample sharding."""
    return passes * rank // world, passes * (rank + 1) // world


def combine_samples(gathered_means: list, pass_counts: list) -> np.ndarray:
    """Fixed-order combination of per-rank partial means (weights = passes)."""
    total = float(sum(pass_counts))
    acc = np.zeros_like(np.asarray(gathered_means[0], np.float64))
    for m, c in zip(gathered_means, pass_counts):
        if c:
            acc += np.asarray(m, np.float64) * c
    return acc / total


# ---------------------------------------------------------------------------
# the driver
# ---------------------------------------------------------------------------

@dataclass
class ShardPlan:
    mode: str
    rank: int
    world: int
    width: int
    height: int
    passes: int

    @property
    def pass0(self) -> int:
        return pass_range(self.passes, self.rank, self.world)[0] if self.mode == "samples" else 0

    @property
    def local_passes(self) -> int:
        if self.mode == "samples":
            a, b = pass_range(self.passes, self.rank, self.world)
            return b - a
        return self.passes

    @property
    def buffer_pixels(self) -> int:
        if self.mode == "samples":
            return self.width * self.height
        return max_shard_tiles(self.width, self.height, self.world) * 256


def plan(mode: str, rank: int, world: int, width: int, height: int, passes: int) -> ShardPlan:
    if mode not in ("tiles", "samples"):
        raise ValueError(f"unknown sharding {mode!r}")
    return ShardPlan(mode, rank, world, width, height, passes)


def render_frame(p: ShardPlan, shard_render: Callable, group=None, device=None):
    """Run one sharded frame.

    ``shard_render(plan) -> torch.Tensor (buffer_pixels, 4) float32`` renders
    the rank's share (tile-compact means for "tiles", row-major when there is
    a single rank; a full frame of partial means over its pass range for
    "samples").  Returns the (H, W, 4) float32
    frame on rank 0 and None elsewhere.  One ``gather`` per frame.
    """
    import torch
    import torch.distributed as dist

    local = shard_render(p)
    if p.world == 1:
        # a single rank renders the whole frame row-major (no compact layout)
        return local.reshape(-1)[: p.height * p.width * 4].reshape(p.height, p.width, 4)
    else:
        gathered = [torch.empty_like(local) for _ in range(p.world)] if p.rank == 0 else None
        dist.gather(local, gathered, dst=0, group=group)
    if p.rank != 0:
        return None
    if p.mode == "tiles":
        if local.is_cuda:
            from .scene import unpack_tiles_device

            packed = torch.cat([g.reshape(-1) for g in gathered])
            frame = torch.zeros(p.height * p.width * 4, dtype=torch.float32, device=local.device)
            unpack_tiles_device(packed.data_ptr(), p.width, p.height, p.world,
                                max_shard_tiles(p.width, p.height, p.world), frame.data_ptr(),
                                torch.cuda.current_stream(local.device).cuda_stream)
            return frame.reshape(p.height, p.width, 4)
        return torch.from_numpy(assemble_tiles([g.numpy() for g in gathered], p.width, p.height))
    counts = [pass_range(p.passes, r, p.world)[1] - pass_range(p.passes, r, p.world)[0] for r in range(p.world)]
    if local.is_cuda:
        acc = torch.zeros_like(local, dtype=torch.float64)
        for g, c in zip(gathered, counts):  # fixed rank order
            if c:
                acc += g.double() * c
        return (acc / float(sum(counts))).float().reshape(p.height, p.width, 4)
    return torch.from_numpy(combine_samples([g.numpy() for g in gathered], counts).astype(np.float32)).reshape(
        p.height, p.width, 4)


FIXED_ONE = float(1 << 32)  # 2^32: fixed-point unit of the frame sums (csrc/trace.cu CameraSource)


def resolve_sums(sums: np.ndarray, width: int, height: int, rank: int, world: int, passes: int, nslots: int,
                 frame: np.ndarray) -> None:
    """CPU statement of srt_resolve_frame_device: a shard's tile-compact
    fixed-point sums (n, 4) int64 -> f64 means written into its pixels of
    the (H, W, 4) frame."""
    px, py, ok = compact_pixels(width, height, rank, world)
    s = np.asarray(sums, np.int64).reshape(-1, 4)[: px.shape[0]][ok]
    inv = 1.0 / (float(passes) * float(nslots))
    frame[py[ok], px[ok], :3] = s[:, :3].astype(np.uint64).astype(np.float64) * (inv / FIXED_ONE)
    frame[py[ok], px[ok], 3] = (s[:, 3].astype(np.uint64) >> np.uint64(32)).astype(np.float64) * inv


def render_frame_sums(p: ShardPlan, shard_sums: Callable, nslots: int, group=None):
    """Run one sharded frame on exact fixed-point sums (every pass of the
    rank's share in one launch, srt_render_frame_device).

    ``shard_sums(plan) -> int64 tensor (n, 4)``: tile-compact 2^-32 sums of
    the rank's tiles ("tiles", n = max shard tiles * 256) or of the whole
    frame over its pass range ("samples", the one-shard layout).  "tiles"
    gathers the sums to rank 0, which resolves each shard into its own pixels;
    "samples" adds them with one integer ``reduce`` -- exact, so the order
    NCCL sums in does not matter.  Either way the f64 frame on rank 0 is bit
    for bit the single-GPU frame, for any world size.  Returns (H, W, 4) f64
    on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    local = shard_sums(p)
    if p.world > 1:
        if p.mode == "tiles":
            gathered = [torch.empty_like(local) for _ in range(p.world)] if p.rank == 0 else None
            dist.gather(local, gathered, dst=0, group=group)
        else:
            dist.reduce(local, dst=0, op=dist.ReduceOp.SUM, group=group)
            gathered = [local]
        if p.rank != 0:
            return None
    else:
        gathered = [local]
    shards = [(r, p.world, g) for r, g in enumerate(gathered)] if p.mode == "tiles" else [(0, 1, gathered[0])]
    if local.is_cuda:
        from .scene import make_render_params, resolve_frame_device

        rgb = torch.zeros((p.height, p.width, 3), dtype=torch.float64, device=local.device)
        op = torch.zeros((p.height, p.width), dtype=torch.float64, device=local.device)
        for r, g_world, buf in shards:
            prm = make_render_params(p.width, p.height, p.passes, nslots, 0, 1.0, True, 0, (0.0, 0.0, 0.0), 0, r,
                                     g_world)
            resolve_frame_device(prm, buf.data_ptr(), rgb.data_ptr(), op.data_ptr(),
                                 torch.cuda.current_stream(local.device).cuda_stream)
        return torch.cat([rgb, op[..., None]], dim=2)
    frame = np.zeros((p.height, p.width, 4))
    for r, g_world, buf in shards:
        resolve_sums(buf.numpy(), p.width, p.height, r, g_world, p.passes, nslots, frame)
    return torch.from_numpy(frame)


def gpu_shard_sums(scene, camera_tuple, settings, device):
    """shard_sums callback: the rank's share of every pass in one libsrt launch."""
    import torch

    from .scene import make_camera, make_render_params, shard_tiles

    cam = make_camera(camera_tuple)
    mode = 0 if settings.depth_mode == "mean" else 1

    def run(p: ShardPlan):
        dev = torch.device("cuda", device)
        if p.mode == "tiles":
            prm = make_render_params(p.width, p.height, p.passes, settings.multisample, mode, settings.cutoff_s ** 2,
                                     True, settings.seed, settings.background, 0, p.rank, p.world)
            n = max_shard_tiles(p.width, p.height, p.world) * 256
        else:
            prm = make_render_params(p.width, p.height, max(p.local_passes, 1), settings.multisample, mode,
                                     settings.cutoff_s ** 2, True, settings.seed, settings.background, p.pass0)
            n = shard_tiles(p.width, p.height) * 256
        acc = torch.zeros((n, 4), dtype=torch.int64, device=dev)
        if p.mode == "samples" and p.local_passes == 0:
            return acc
        scene.render_frame_device(cam, prm, acc.data_ptr(), 0, torch.cuda.current_stream(dev).cuda_stream)
        return acc

    return run


def gpu_shard_renderer(scene, camera_tuple, settings, device):
    """shard_render callback tracing the rank's share with libsrt on `device`."""
    import torch

    from .scene import make_camera, make_render_params

    cam = make_camera(camera_tuple)
    mode = 0 if settings.depth_mode == "mean" else 1

    def run(p: ShardPlan):
        dev = torch.device("cuda", device)
        if p.mode == "tiles":
            prm = make_render_params(p.width, p.height, p.passes, settings.multisample, mode,
                                     settings.cutoff_s ** 2, True, settings.seed, settings.background,
                                     0, p.rank, p.world)
        else:
            prm = make_render_params(p.width, p.height, max(p.local_passes, 1), settings.multisample, mode,
                                     settings.cutoff_s ** 2, True, settings.seed, settings.background, p.pass0)
        from .scene import shard_tiles

        n = max(p.buffer_pixels, p.width * p.height if p.world == 1 else 0)
        out = torch.zeros((n, 4), dtype=torch.float32, device=dev)
        if p.mode == "samples" and p.local_passes == 0:
            return out
        # trace scratch in the tile-compact layout of the traced tiles
        tiles = shard_tiles(p.width, p.height, p.rank, p.world) if p.mode == "tiles" else shard_tiles(p.width, p.height)
        # every pass in one launch, fixed-point sums (bitwise the render() frame)
        acc = torch.empty((max(tiles, 1) * 256, 4), dtype=torch.int64, device=dev)
        scene.render_frame_device(cam, prm, acc.data_ptr(), out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
        return out

    return run


# ---------------------------------------------------------------------------
# one device frame every rank stores into (multi-GPU frames on rank 0's GPU)
# ---------------------------------------------------------------------------

class PeerFrame:
    """A row-major (H*W) float4 frame in rank 0's HBM that every rank maps
    with CUDA IPC (srt_ipc_alloc / srt_ipc_open): each rank's fused walk
    stores its own tiles' pixels straight into it over NVLink
    (srt_render_pass_frame_device), so the frame gather of the NCCL path
    and its unpack kernel disappear -- the transfer overlaps the walk, tile
    by tile.  Collective construction; ``ok`` is False on every rank when
    any rank could not map the buffer (callers then fall back to the NCCL
    gather).  ``ptr`` is the device address valid on this rank."""

    def __init__(self, nbytes: int, rank: int, device: int, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib

        L = _lib.load()
        self.rank, self.device, self.ptr, self._owned = rank, device, 0, False
        p = ctypes.c_void_p()
        err = ""
        box = [None]
        if rank == 0:
            h = (ctypes.c_uint8 * 64)()
            if L.srt_ipc_alloc(device, int(nbytes), ctypes.byref(p), h) == 0:
                self.ptr, self._owned = p.value, True
                box = [bytes(h)]
            else:
                err = L.srt_last_error().decode(errors="replace")
        dist.broadcast_object_list(box, src=0, group=group)
        if rank != 0 and box[0] is not None:
            h = (ctypes.c_uint8 * 64).from_buffer_copy(box[0])
            if L.srt_ipc_open(device, h, ctypes.byref(p)) == 0:
                self.ptr = p.value
            else:
                err = L.srt_last_error().decode(errors="replace")
        dev = torch.device("cuda", device) if dist.get_backend(group) == "nccl" else "cpu"
        flag = torch.tensor([1 if self.ptr else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        self.ok = bool(flag.item())
        self.error = err
        if not self.ok:
            self.close()

    def close(self) -> None:
        import ctypes

        from . import _lib

        if self.ptr:
            L = _lib.load()
            (L.srt_ipc_free if self._owned else L.srt_ipc_close)(self.device, ctypes.c_void_p(self.ptr))
        self.ptr = 0


# ---------------------------------------------------------------------------
# one host frame shared by every rank (multi-GPU e2e)
# ---------------------------------------------------------------------------

def _bcast_ints(values, group=None, src: int = 0) -> list:
    """Broadcast a few ints from `src` (a device tensor under NCCL)."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(values), dtype=torch.int64, device=dev)
    dist.broadcast(t, src, group=group)
    return [int(v) for v in t.tolist()]


class _SharedBlock:
    """Numpy-visible view of one pooled shared frame; returns the frame to the
    pool when the last array viewing it is collected (rank 0)."""

    def __init__(self, pool, key: int, base: np.ndarray):
        self._pool, self._key, self._base = pool, key, base
        self.__array_interface__ = {"shape": base.shape, "typestr": "|u1",
                                    "data": (base.__array_interface__["data"][0], False), "version": 3}

    def __del__(self):
        try:
            self._pool._release(self._key)
        except Exception:
            pass


class SharedFramePool:
    """Host frames in POSIX shared memory (/dev/shm), mapped by every rank of
    the group and page-locked + device-mapped on each (srt_host_register):
    each GPU writes its own 16x16 tiles of the f64 frame straight into the one
    buffer over its own PCIe link, so the frame is assembled on the host
    without a gather through rank 0's GPU and link.

    Rank 0 owns the pool: per frame it picks a free block (or creates one) and
    broadcasts its index; blocks return to the pool when rank 0's AccumBuffer
    arrays are collected.  ``register=False`` skips the CUDA registration
    (CPU tests of the protocol)."""

    SHM_DIR = "/dev/shm"

    def __init__(self, register: bool = True):
        self.register = register
        self._prefix = None
        self._attached: dict = {}  # key -> (mmap, uint8 array, nbytes)
        self._free: dict = {}      # nbytes -> [key]   (rank 0)
        self._next = 0
        self._owner = False

    def _path(self, key: int) -> str:
        return f"{self.SHM_DIR}/{self._prefix}_{key}"

    def _attach(self, key: int, nbytes: int, create: bool):
        import mmap
        import os

        flags = os.O_RDWR | (os.O_CREAT | os.O_EXCL if create else 0)
        fd = os.open(self._path(key), flags, 0o600)
        try:
            if create:
                os.ftruncate(fd, nbytes)
            mm = mmap.mmap(fd, nbytes)
        finally:
            os.close(fd)
        arr = np.frombuffer(mm, dtype=np.uint8)
        if self.register:
            import ctypes

            from . import _lib

            _lib.check(_lib.load().srt_host_register(ctypes.c_void_p(arr.__array_interface__["data"][0]), nbytes))
        self._attached[key] = (mm, arr, nbytes)

    def acquire(self, nbytes: int, rank: int, group=None):
        """(key, writable uint8 view of the block) on every rank; collective."""
        import os
        import uuid

        import torch.distributed as dist

        if self._prefix is None:
            box = [f"srt{os.getpid()}_{uuid.uuid4().hex[:8]}" if rank == 0 else None]
            dist.broadcast_object_list(box, src=0, group=group)
            self._prefix = box[0]
            if rank == 0:
                import atexit

                self._owner = True
                atexit.register(self.close)
        key = -1
        if rank == 0:
            free = self._free.setdefault(nbytes, [])
            if free:
                key = free.pop()
            else:
                key = self._next
                self._next += 1
                self._attach(key, nbytes, create=True)
        key = _bcast_ints([key], group)[0]
        if key not in self._attached:
            self._attach(key, nbytes, create=False)
        _, arr, _ = self._attached[key]
        if rank == 0:
            return key, np.asarray(_SharedBlock(self, key, arr))
        return key, arr

    def _release(self, key: int) -> None:
        if key in self._attached:
            self._free.setdefault(self._attached[key][2], []).append(key)

    def close(self) -> None:
        import os

        for key, (mm, arr, nb) in self._attached.items():
            if self.register:
                try:
                    import ctypes

                    from . import _lib

                    _lib.load().srt_host_unregister(ctypes.c_void_p(arr.__array_interface__["data"][0]))
                except Exception:
                    pass
            if self._owner:
                try:
                    os.unlink(self._path(key))
                except OSError:
                    pass
        self._attached.clear()  # the mappings go with the last array that views them


_SHARED = None


def shared_frame_pool() -> SharedFramePool:
    global _SHARED
    if _SHARED is None:
        _SHARED = SharedFramePool()
    return _SHARED


def render_frame_shared(p: ShardPlan, shard_write: Callable, pool: SharedFramePool, group=None):
    """One tile-sharded frame assembled in host shared memory: every rank
    calls ``shard_write(plan, rgb (H,W,3) f64 view, opacity (H,W) f64 view)``,
    which writes exactly its own tiles; one barrier; rank 0 returns the
    (rgb, opacity) arrays (pooled), the others None."""
    import torch.distributed as dist

    H, W = p.height, p.width
    nbytes = H * W * 4 * 8
    _, raw = pool.acquire(nbytes, p.rank, group)
    f = raw.view(np.float64)
    rgb, op = f[: H * W * 3].reshape(H, W, 3), f[H * W * 3:].reshape(H, W)
    shard_write(p, rgb, op)
    dist.barrier(group=group)
    return (rgb, op) if p.rank == 0 else None


def render_distributed(asset, camera, settings, mode: str = "tiles", group=None, device: int | None = None,
                       transport: str | None = None):
    """Drop-in multi-GPU render: call on every rank of an initialised process
    group (NCCL).  Returns the AccumBuffer on rank 0, None on the others.

    ``transport`` (tiles mode): ``"host"`` (default at world size > 1) -- every
    rank writes its tiles of the f64 frame into one shared, mapped host buffer
    (SharedFramePool); ``"nccl"`` -- tile buffers gathered to rank 0's GPU with
    one NCCL gather, then one device->host copy."""
    import torch
    import torch.distributed as dist

    from .render import AccumBuffer, prepare
    from .scene import camera_tuple

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if device is None:
        device = torch.cuda.current_device()
    sc = prepare(asset, settings, device=device)
    ct = camera_tuple(camera, settings.width, settings.height)
    p = plan(mode, rank, world, settings.width, settings.height, settings.passes)
    if transport is None:
        transport = "host" if (mode == "tiles" and world > 1) else "nccl"
    if transport not in ("host", "nccl"):
        raise ValueError(f"unknown transport {transport!r}")
    if transport == "host" and mode == "tiles" and world > 1:
        m = 0 if settings.depth_mode == "mean" else 1

        def write(plan_, rgb, op):
            sc.render(ct, plan_.width, plan_.height, settings.passes, settings.multisample, m,
                      settings.cutoff_s ** 2, True, settings.seed, settings.background, out_rgb=rgb, out_op=op,
                      shard_index=plan_.rank, shard_count=plan_.world)

        got = render_frame_shared(p, write, shared_frame_pool(), group)
        return None if got is None else AccumBuffer(got[0], got[1], settings.samples_per_pixel)
    if settings.passes > 1 or mode == "samples":
        # exact fixed-point sums: bitwise the single-GPU render() frame
        frame = render_frame_sums(p, gpu_shard_sums(sc, ct, settings, device), settings.multisample, group)
    else:
        frame = render_frame(p, gpu_shard_renderer(sc, ct, settings, device), group)
    torch.cuda.current_stream(torch.device("cuda", device)).synchronize()
    sc.check_status()  # a stack overflow in this rank's launch raises here, not silently
    if frame is None:
        return None
    if frame.is_cuda:
        # f64 on the device, then one device->host copy into page-locked memory
        f64 = frame.double()
        host = torch.empty(f64.shape, dtype=torch.float64, pin_memory=True)
        host.copy_(f64, non_blocking=True)
        torch.cuda.current_stream(f64.device).synchronize()
        f = host.numpy()
    else:
        f = frame.double().numpy()
    return AccumBuffer(f[..., :3], f[..., 3], settings.samples_per_pixel)


def render_devices(asset, camera, settings, devices, rng: str = "counter"):
    """Single-process multi-GPU render (SURVEY.md 8(b) "plus optional devices";
    8(e) tile sharding): one host thread drives every device -- shard i of G
    traces the interleaved tiles t % G == i on ``devices[i]`` in one launch
    (every pass, fixed-point sums, async on per-device streams); the sums are
    copied to ``devices[0]`` (peer copies over NVLink) and resolved there into
    one f64 frame, each shard writing its own pixels.  The counter stream is
    keyed per pixel and the sums are exact, so the frame equals the
    single-GPU render bit for bit.  A device may appear more than once (its
    shards then run back to back on one stream).  Single-pass frames and
    rng="trig64" take the per-pass path with float means, as render() does."""
    import torch

    from .render import AccumBuffer, prepare
    from .scene import camera_tuple, make_camera, make_render_params, resolve_frame_device, shard_tiles

    devices = [int(d) for d in devices]
    G = len(devices)
    if G == 0:
        raise ValueError("devices must name at least one GPU")
    W, H = settings.width, settings.height
    cam = make_camera(camera_tuple(camera, W, H))
    mode = 0 if settings.depth_mode == "mean" else 1
    d0 = torch.device("cuda", devices[0])
    fixed = rng == "counter" and settings.passes > 1  # srt_render's multi-pass path
    prms, bufs, scenes = [], [], []
    for i, d in enumerate(devices):
        sc = prepare(asset, settings, device=d)
        scenes.append(sc)
        dev = torch.device("cuda", d)
        prm = make_render_params(W, H, settings.passes, settings.multisample, mode, settings.cutoff_s ** 2, True,
                                 settings.seed, settings.background, 0, i, G, rng=rng)
        tiles = max(shard_tiles(W, H, i, G), 1)
        stream = torch.cuda.current_stream(dev).cuda_stream
        if fixed:
            acc = torch.empty((tiles * 256, 4), dtype=torch.int64, device=dev)
            sc.render_frame_device(cam, prm, acc.data_ptr(), 0, stream)
            bufs.append(acc)
        else:
            hits = torch.empty(tiles * 256 * settings.multisample, dtype=torch.int32, device=dev)
            acc = torch.empty((tiles * 256, 4), dtype=torch.float32, device=dev)
            out = torch.zeros((max_shard_tiles(W, H, G) * 256, 4), dtype=torch.float32, device=dev)
            sc.render_device(cam, prm, hits.data_ptr(), acc.data_ptr(), out.data_ptr(), stream)
            bufs.append(out)
        prms.append(prm)
    for d in set(devices):
        torch.cuda.current_stream(torch.device("cuda", d)).synchronize()
    for sc in scenes:
        sc.check_status()
    s0 = torch.cuda.current_stream(d0).cuda_stream
    if fixed:
        rgb = torch.zeros((H, W, 3), dtype=torch.float64, device=d0)
        op = torch.zeros((H, W), dtype=torch.float64, device=d0)
        with torch.cuda.device(d0):
            for prm, acc in zip(prms, bufs):
                a0 = acc.to(d0)
                resolve_frame_device(prm, a0.data_ptr(), rgb.data_ptr(), op.data_ptr(), s0)
            torch.cuda.current_stream(d0).synchronize()
        return AccumBuffer(rgb.cpu().numpy(), op.cpu().numpy(), settings.samples_per_pixel)
    from .scene import unpack_tiles_device

    packed = torch.cat([o.to(d0).reshape(-1) for o in bufs])
    frame = torch.zeros(H * W * 4, dtype=torch.float32, device=d0)
    unpack_tiles_device(packed.data_ptr(), W, H, G, max_shard_tiles(W, H, G), frame.data_ptr(), s0)
    f = frame.reshape(H, W, 4).double().cpu().numpy()
    return AccumBuffer(f[..., :3], f[..., 3], settings.samples_per_pixel)
