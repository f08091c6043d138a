"""Device-resident scene handle: the host side of the libsrt C ABI.

A ``DeviceScene`` owns one ``SrtScene*``: the packed float64 scene uploaded
once and converted to fp32 records in HBM, plus its BVH (GPU LBVH by
default, or an uploaded reference-layout BVH).  It is the object the
reference's ``render``/``kernels`` boundary maps onto.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from ._lib import SrtCamera, SrtRenderParams, SrtSceneDesc, SrtTraceParams, check

TMAX = float(np.finfo(np.float64).max)
RNG = {"counter": _lib.SRT_RNG_COUNTER, "table": _lib.SRT_RNG_TABLE, "trig64": _lib.SRT_RNG_TRIG64}


def _ptr(a) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if a is None else a.__array_interface__["data"][0])


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ci64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _rays(origins, dirs):
    """(R,3) f64 origin and direction arrays with matching row counts (the
    C ABI copies 24 R bytes from each)."""
    o = _c64(origins)
    d = _c64(dirs)
    if o.ndim != 2 or o.shape[1] != 3 or d.shape != o.shape:
        raise ValueError(f"origins and directions must both be (R, 3); got {o.shape} and {d.shape}")
    return o, d


_STRUCT_CACHE: dict = {}


def _cached(key, make):
    """ctypes argument structs memoised on their values (a render loop passes
    the same camera and settings every frame; building them costs ~5 us each)."""
    hit = _STRUCT_CACHE.get(key)
    if hit is None:
        if len(_STRUCT_CACHE) > 4096:
            _STRUCT_CACHE.clear()
        hit = _STRUCT_CACHE[key] = make()
    return hit


def make_camera(cam) -> SrtCamera:
    """SrtCamera from the 14 scalars (ex..ez, rx..rz, ux..uz, fx..fz, half_w, half_h)
    of render.py:144-150."""
    return _cached(("cam", tuple(cam)), lambda: _make_camera(cam))


def _make_camera(cam) -> SrtCamera:
    c = SrtCamera()
    v = [float(x) for x in cam]
    for k in range(3):
        c.position[k] = v[k]
        c.right[k] = v[3 + k]
        c.up[k] = v[6 + k]
        c.forward[k] = v[9 + k]
    c.half_w, c.half_h = v[12], v[13]
    return c


def make_render_params(width, height, passes, nslots, mode, s2, clip=True, seed=0, background=(0.0, 0.0, 0.0),
                       pass0=0, shard_index=0, shard_count=1, rng="counter") -> SrtRenderParams:
    key = ("prm", width, height, passes, nslots, mode, s2, clip, seed, tuple(float(b) for b in background), pass0,
           shard_index, shard_count, rng)
    return _cached(key, lambda: _make_render_params(width, height, passes, nslots, mode, s2, clip, seed, background,
                                                    pass0, shard_index, shard_count, rng))


def _make_render_params(width, height, passes, nslots, mode, s2, clip, seed, background, pass0, shard_index,
                        shard_count, rng) -> SrtRenderParams:
    p = SrtRenderParams()
    p.width, p.height, p.passes, p.nslots = int(width), int(height), int(passes), int(nslots)
    p.mode, p.clip, p.s2 = int(mode), int(bool(clip)), float(s2)
    p.seed = int(seed) & 0xFFFFFFFF
    p.pass0 = int(pass0)
    for k in range(3):
        p.background[k] = float(background[k])
    p.shard_index, p.shard_count = int(shard_index), int(shard_count)
    if rng not in ("counter", "trig64"):
        raise ValueError(f"render rng must be 'counter' or 'trig64', got {rng!r}")
    p.rng = RNG[rng]
    return p


class DeviceScene:
    """One packed scene on one GPU (libsrt ``SrtScene``)."""

    def __init__(self, means, cov_inv6, opacities, sh=None, sh_degree: int = 0, device: int = 0):
        L = _lib.load()
        _lib.require_device()
        means, cov6, opac = _c64(means).reshape(-1, 3), _c64(cov_inv6).reshape(-1, 6), _c64(opacities).reshape(-1)
        n = means.shape[0]
        if cov6.shape[0] != n or opac.shape[0] != n:
            raise ValueError("mismatched scene array shapes")
        if sh is not None:
            sh = _c64(sh)
            if sh.shape[0] != n or sh.size != n * 3 * (sh_degree + 1) ** 2:
                raise ValueError("sh array does not match n and sh_degree")
        desc = SrtSceneDesc(n, means.ctypes.data, cov6.ctypes.data, opac.ctypes.data,
                            None if sh is None else sh.ctypes.data, int(sh_degree))
        h = ctypes.c_void_p()
        check(L.srt_scene_create(ctypes.byref(desc), int(device), ctypes.byref(h)))
        self._h = h
        self.n = n
        self.sh_degree = int(sh_degree)
        self.device = int(device)
        self.bvh_key = None

    @classmethod
    def from_packed(cls, pack, device: int = 0) -> "DeviceScene":
        return cls(pack.means, pack.cov_inv6, pack.opacities, pack.sh, pack.sh_degree, device)

    @classmethod
    def from_splats(cls, asset, device: int = 0) -> "DeviceScene":
        """Upload a SplatAsset's raw fields and pack the inverse covariances on
        the GPU (srt_scene_create_from_splats) instead of via asset.packed."""
        from ._lib import SrtSplatDesc

        L = _lib.load()
        _lib.require_device()
        means, rot, sc = _c64(asset.means), _c64(asset.rotations), _c64(asset.scales)
        opac, sh = _c64(asset.opacities), _c64(asset.sh)
        desc = SrtSplatDesc(means.shape[0], means.ctypes.data, rot.ctypes.data, sc.ctypes.data, opac.ctypes.data,
                            sh.ctypes.data, int(asset.sh_degree))
        h = ctypes.c_void_p()
        check(L.srt_scene_create_from_splats(ctypes.byref(desc), int(device), ctypes.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self.n = means.shape[0]
        self.sh_degree = int(asset.sh_degree)
        self.device = int(device)
        self.bvh_key = None
        return self

    # -- lifetime ----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().srt_scene_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._h.value:
            raise ValueError("scene is closed")
        return self._h

    # -- BVH -----------------------------------------------------------------
    def build_bvh(self, cutoff_s: float, method: str = "ploc") -> None:
        """GPU BVH over the cutoff-ellipsoid boxes (srt_bvh_build_ex): "ploc"
        (agglomerative clustering, default) or "lbvh" (Karras radix tree)."""
        methods = {"lbvh": 0, "ploc": 1}
        if method not in methods:
            raise ValueError(f"unknown BVH build method {method!r}")
        check(_lib.load().srt_bvh_build_ex(self.handle, float(cutoff_s), methods[method]))
        self.bvh_key = ("lbvh", float(cutoff_s))

    def upload_bvh(self, bvh) -> None:
        """Upload a reference-layout BVH (bvh.py:29-47) (srt_bvh_upload)."""
        arrs = [_c64(bvh.node_lo), _c64(bvh.node_hi), _ci64(bvh.node_left), _ci64(bvh.node_right),
                _ci64(bvh.node_count), _ci64(bvh.prim_order), _c64(bvh.prim_lo), _c64(bvh.prim_hi)]
        M = arrs[0].reshape(-1, 3).shape[0]
        if arrs[5].shape[0] != self.n and M > 0:
            raise ValueError("BVH prim_order does not match the scene size")
        check(_lib.load().srt_bvh_upload(self.handle, M, *[_ptr(a) for a in arrs]))
        self.bvh_key = ("upload", id(bvh))
        self._bvh_ref = bvh  # keep id() meaningful

    def bvh_info(self) -> dict:
        nn, d, npr, nb = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        check(_lib.load().srt_bvh_info(self.handle, ctypes.byref(nn), ctypes.byref(d), ctypes.byref(npr),
                                       ctypes.byref(nb)))
        return {"num_nodes": nn.value, "depth": d.value, "num_prims": npr.value, "device_bytes": nb.value}

    def split_info(self) -> dict:
        """The packet walk's spatially split tree (srt_bvh_split_info): leaf
        references, 4-wide nodes, grid cells per axis (all 0 without one)."""
        nr, n4, c = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        check(_lib.load().srt_bvh_split_info(self.handle, ctypes.byref(nr), ctypes.byref(n4), ctypes.byref(c)))
        return {"num_refs": nr.value, "num_nodes4": n4.value, "cells": c.value}

    def download_bvh(self) -> dict:
        """Device BVH in the reference layout: inner nodes 0..M-1, then one
        single-primitive leaf node per slot (fp32 boxes)."""
        info = self.bvh_info()
        mi, n = info["num_nodes"], self.n
        tot = mi + n
        out = {
            "node_lo": np.zeros((tot, 3), np.float32), "node_hi": np.zeros((tot, 3), np.float32),
            "node_left": np.full(tot, -1, np.int64), "node_right": np.full(tot, -1, np.int64),
            "node_count": np.zeros(tot, np.int64), "prim_order": np.zeros(n, np.int64),
            "prim_lo": np.zeros((n, 3), np.float32), "prim_hi": np.zeros((n, 3), np.float32),
        }
        check(_lib.load().srt_bvh_download(self.handle, *[_ptr(out[k]) for k in (
            "node_lo", "node_hi", "node_left", "node_right", "node_count", "prim_order", "prim_lo", "prim_hi")]))
        out["num_inner"] = mi
        return out

    # -- explicit rays ---------------------------------------------------------
    def trace_rays(self, origins, dirs, t_min=0.0, t_max=TMAX, mode=0, s2=8.0, clip=True, nslots=1,
                   rng="counter", seed=0, ray_id0=0, sample0=0, table=None):
        """kernels.trace_batch semantics (kernels.py:527-540) on the GPU.
        rng: "counter" (default), "table" (explicit uniforms) or "trig64" (the
        reference's own fp64 trig-hash draw, parity mode).
        Returns (out_t (R,N) f64, +inf on miss; out_id (R,N) i64, -1 on miss)."""
        o, d = _rays(origins, dirs)
        R = o.shape[0]
        p = SrtTraceParams()
        p.t_min, p.t_max, p.mode, p.clip, p.s2 = float(t_min), float(t_max), int(mode), int(bool(clip)), float(s2)
        p.rng = RNG[rng]
        p.seed, p.ray_id0, p.sample0 = seed & 0xFFFFFFFF, ray_id0 & 0xFFFFFFFF, sample0 & 0xFFFFFFFF
        tab = None
        if rng == "table":
            tab = _c64(table)
            if tab.ndim != 2 or tab.shape[0] != self.n:
                raise ValueError("table must be (n, slots)")
            p.table, p.table_slots = tab.ctypes.data, tab.shape[1]
        out_t = np.empty((R, nslots))
        out_id = np.empty((R, nslots), np.int64)
        check(_lib.load().srt_trace_rays(self.handle, ctypes.byref(p), _ptr(o), _ptr(d), R, int(nslots),
                                         _ptr(out_t), _ptr(out_id)))
        return out_t, out_id

    def trace_rays_device(self, d_rays: int, num_rays: int, nslots: int, d_t: int, d_id: int, stream: int,
                          t_min=0.0, t_max=TMAX, mode=0, s2=8.0, clip=True, seed=0, ray_id0=0, sample0=0) -> None:
        """srt_trace_rays_device: counter-RNG walks of device-resident rays
        (d_rays: (R, 6) f64 origin+direction) into device outputs d_t (R, N)
        f32 and d_id (R, N) i32, asynchronously on `stream`."""
        p = SrtTraceParams()
        p.t_min, p.t_max, p.mode, p.clip, p.s2 = float(t_min), float(t_max), int(mode), int(bool(clip)), float(s2)
        p.rng = RNG["counter"]
        p.seed, p.ray_id0, p.sample0 = seed & 0xFFFFFFFF, ray_id0 & 0xFFFFFFFF, sample0 & 0xFFFFFFFF
        check(_lib.load().srt_trace_rays_device(self.handle, ctypes.byref(p), ctypes.c_void_p(d_rays), int(num_rays),
                                                int(nslots), ctypes.c_void_p(d_t), ctypes.c_void_p(d_id),
                                                ctypes.c_void_p(stream)))

    def transmittance(self, origins, dirs, t_min=0.0, t_max=TMAX, mode=0, s2=8.0) -> np.ndarray:
        o, d = _rays(origins, dirs)
        out = np.empty(o.shape[0])
        check(_lib.load().srt_transmittance_rays(self.handle, _ptr(o), _ptr(d), o.shape[0], float(t_min),
                                                 float(t_max), int(mode), float(s2), _ptr(out)))
        return out

    def exact_rays(self, origins, dirs, t_min=0.0, t_max=TMAX, mode=0, s2=8.0, background=(0.0, 0.0, 0.0)):
        """kernels.exact_batch semantics (kernels.py:584-604): sorted compositing
        of every valid candidate.  Returns (rgb (R,3) f64, opacity (R,) f64)."""
        o, d = _rays(origins, dirs)
        bg = _c64(background).reshape(3)
        rgb = np.empty((o.shape[0], 3))
        op = np.empty(o.shape[0])
        check(_lib.load().srt_exact_rays(self.handle, _ptr(o), _ptr(d), o.shape[0], float(t_min), float(t_max),
                                         int(mode), float(s2), _ptr(bg), _ptr(rgb), _ptr(op)))
        return rgb, op

    def biased_rays(self, origins, dirs, kk, t_min=0.0, t_max=TMAX, mode=0, s2=8.0, background=(0.0, 0.0, 0.0),
                    rng="counter", seed=0, ray_id0=0, sample0=0, table=None):
        """kernels.biased_batch semantics (kernels.py:479-518, 561-580): one
        acceptance draw per candidate (slot 0 of the ray's stream), the kk
        nearest accepted composited with their own alphas.  Returns rgb (R,3)."""
        if int(kk) < 1:
            raise ValueError(f"k must be >= 1, got {kk}")
        o, d = _rays(origins, dirs)
        bg = _c64(background).reshape(3)
        p = SrtTraceParams()
        p.t_min, p.t_max, p.mode, p.clip, p.s2 = float(t_min), float(t_max), int(mode), 0, float(s2)
        p.rng = RNG[rng]
        p.seed, p.ray_id0, p.sample0 = seed & 0xFFFFFFFF, ray_id0 & 0xFFFFFFFF, sample0 & 0xFFFFFFFF
        tab = None
        if rng == "table":
            tab = _c64(table)
            if tab.ndim == 1:
                tab = tab.reshape(-1, 1)
            if tab.ndim != 2 or tab.shape[0] != self.n:
                raise ValueError("table must be (n,) or (n, slots)")
            p.table, p.table_slots = tab.ctypes.data, tab.shape[1]
        rgb = np.empty((o.shape[0], 3))
        check(_lib.load().srt_biased_rays(self.handle, ctypes.byref(p), _ptr(o), _ptr(d), o.shape[0], int(kk),
                                          _ptr(bg), _ptr(rgb)))
        return rgb

    def render_biased(self, cam, width, height, kk, passes=1, mode=0, s2=8.0, seed=0, background=(0.0, 0.0, 0.0),
                      pass0=0, rng="counter", out_rgb=None):
        """cli._biased_frame semantics (cli.py:164-203): per-pixel mean over
        `passes` jittered rays of the biased k-nearest composite."""
        if int(kk) < 1:
            raise ValueError(f"k must be >= 1, got {kk}")
        camera = make_camera(cam)
        prm = make_render_params(width, height, passes, 1, mode, s2, False, seed, background, pass0, rng=rng)
        rgb = np.empty((height, width, 3)) if out_rgb is None else out_rgb
        check(_lib.load().srt_render_biased(self.handle, ctypes.byref(camera), ctypes.byref(prm), int(kk), _ptr(rgb)))
        return rgb

    def render_exact(self, cam, width, height, frames=1, mode=0, s2=8.0, seed=0, background=(0.0, 0.0, 0.0),
                     out_rgb=None, out_op=None):
        """kernels.render_exact semantics (kernels.py:677-723)."""
        camera = make_camera(cam)
        prm = make_render_params(width, height, frames, 1, mode, s2, True, seed, background)
        rgb = np.empty((height, width, 3)) if out_rgb is None else out_rgb
        op = np.empty((height, width)) if out_op is None else out_op
        check(_lib.load().srt_render_exact(self.handle, ctypes.byref(camera), ctypes.byref(prm), _ptr(rgb), _ptr(op)))
        return rgb, op

    # -- frames ----------------------------------------------------------------
    def render(self, cam, width, height, passes=1, nslots=1, mode=0, s2=8.0, clip=True, seed=0,
               background=(0.0, 0.0, 0.0), pass0=0, want_ids=False, out_rgb=None, out_op=None, rng="counter",
               shard_index=0, shard_count=1):
        """kernels.render_stochastic semantics (kernels.py:622-673) on the GPU.
        Returns (rgb (H,W,3) f64, opacity (H,W) f64, ids (H,W,N) i64 of pass pass0 or None).
        shard_count > 1 renders only the 16x16 tiles t with t % shard_count ==
        shard_index, into mapped host outputs (multi_gpu.SharedFramePool)."""
        camera = make_camera(cam)
        prm = make_render_params(width, height, passes, nslots, mode, s2, clip, seed, background, pass0,
                                 shard_index=shard_index, shard_count=shard_count, rng=rng)
        rgb = np.empty((height, width, 3)) if out_rgb is None else out_rgb
        op = np.empty((height, width)) if out_op is None else out_op
        ids = np.full((height, width, nslots), -1, np.int64) if want_ids else None
        check(_lib.load().srt_render(self.handle, ctypes.byref(camera), ctypes.byref(prm), _ptr(rgb), _ptr(op),
                                     _ptr(ids)))
        return rgb, op, ids

    def check_status(self, reset: bool = True) -> None:
        """Raise if any launch on this scene overflowed its traversal stack
        since the last reset (srt_scene_check; the *_device entry points do
        not report it themselves)."""
        check(_lib.load().srt_scene_check(self.handle, int(bool(reset))))

    def trace_stats(self, reset: bool = True) -> dict:
        """Traversal counters (collected only when SRT_TRACE_STATS=1 was set)."""
        out = np.zeros(16, np.uint64)
        check(_lib.load().srt_trace_counters(self.handle, _ptr(out), 16, int(bool(reset))))
        names = ("node_visits", "leaf_visits", "screen_pass", "exact_evals", "accepts", "pops", "culled_pops",
                 "walks", "visits_with_leaf_hit", "leaf_children_hit", "inner_children_hit", "lanes_hitting",
                 "lanes_without_hit", "job_rounds", "empty_visits", "unused")
        return dict(zip(names, (int(v) for v in out)))

    # device-pointer variants (bench.py, multi_gpu.py); pointers are ints
    def trace_pass_device(self, camera, prm, pass_index, d_hits, stream) -> None:
        check(_lib.load().srt_trace_pass_device(self.handle, ctypes.byref(camera), ctypes.byref(prm),
                                                int(pass_index), ctypes.c_void_p(d_hits), ctypes.c_void_p(stream)))

    def shade_pass_device(self, camera, prm, pass_index, d_hits, d_accum, first, last, d_out, stream) -> None:
        check(_lib.load().srt_shade_pass_device(self.handle, ctypes.byref(camera), ctypes.byref(prm),
                                                int(pass_index), ctypes.c_void_p(d_hits), ctypes.c_void_p(d_accum),
                                                int(bool(first)), int(bool(last)), ctypes.c_void_p(d_out),
                                                ctypes.c_void_p(stream)))

    def render_pass_device(self, camera, prm, pass_index, d_accum, first, last, d_out, stream) -> None:
        """One pass traced and shaded by a single kernel (srt_render_pass_device)."""
        check(_lib.load().srt_render_pass_device(self.handle, ctypes.byref(camera), ctypes.byref(prm),
                                                 int(pass_index), ctypes.c_void_p(d_accum), int(bool(first)),
                                                 int(bool(last)), ctypes.c_void_p(d_out), ctypes.c_void_p(stream)))

    def render_pass_frame_device(self, camera, prm, pass_index, d_accum, first, last, d_frame, peer, stream) -> None:
        """srt_render_pass_frame_device: the fused pass writing the row-major
        full frame (a shard writes only its pixels; d_frame may be a peer
        GPU's IPC-mapped buffer when peer is set)."""
        check(_lib.load().srt_render_pass_frame_device(self.handle, ctypes.byref(camera), ctypes.byref(prm),
                                                       int(pass_index), ctypes.c_void_p(d_accum), int(bool(first)),
                                                       int(bool(last)), ctypes.c_void_p(d_frame), int(bool(peer)),
                                                       ctypes.c_void_p(stream)))

    def render_frame_device(self, camera, prm, d_acc, d_out, stream) -> None:
        """srt_render_frame_device: every pass of the frame in one launch;
        d_acc: (local tiles * 256, 4) uint64 scratch, d_out: float4 means."""
        check(_lib.load().srt_render_frame_device(self.handle, ctypes.byref(camera), ctypes.byref(prm),
                                                  ctypes.c_void_p(d_acc), ctypes.c_void_p(d_out),
                                                  ctypes.c_void_p(stream)))

    def render_device(self, camera, prm, d_hits, d_accum, d_out, stream) -> None:
        check(_lib.load().srt_render_device(self.handle, ctypes.byref(camera), ctypes.byref(prm),
                                            ctypes.c_void_p(d_hits), ctypes.c_void_p(d_accum),
                                            ctypes.c_void_p(d_out), ctypes.c_void_p(stream)))


def resolve_frame_device(prm, d_acc: int, d_rgb: int, d_op: int, stream: int) -> None:
    """srt_resolve_frame_device: a shard's fixed-point sums -> f64 means in the
    row-major full-frame buffers (current device)."""
    check(_lib.load().srt_resolve_frame_device(ctypes.byref(prm), ctypes.c_void_p(d_acc), ctypes.c_void_p(d_rgb),
                                               ctypes.c_void_p(d_op), ctypes.c_void_p(stream)))


def shard_tiles(width: int, height: int, shard_index: int = 0, shard_count: int = 1) -> int:
    return int(_lib.load().srt_shard_tiles(int(width), int(height), int(shard_index), int(shard_count)))


def unpack_tiles_device(d_gathered: int, width: int, height: int, shard_count: int, max_tiles: int, d_frame: int,
                        stream: int) -> None:
    check(_lib.load().srt_unpack_tiles_device(ctypes.c_void_p(d_gathered), int(width), int(height),
                                              int(shard_count), int(max_tiles), ctypes.c_void_p(d_frame),
                                              ctypes.c_void_p(stream)))


_CAMERA_CACHE: dict = {}


def camera_tuple(camera, width: int, height: int) -> tuple:
    """The 14 camera scalars of render.py:140-150 from a CameraConfig
    (memoised on the camera's values: the numpy basis costs ~90 us a frame)."""
    key = (camera.position.tobytes(), camera.look_at.tobytes(), camera.up.tobytes(), float(camera.fov_deg),
           int(width), int(height))
    hit = _CAMERA_CACHE.get(key)
    if hit is None:
        if len(_CAMERA_CACHE) > 1024:
            _CAMERA_CACHE.clear()
        hit = _CAMERA_CACHE[key] = _camera_tuple(camera, width, height)
    return hit


def _camera_tuple(camera, width: int, height: int) -> tuple:
    fwd = camera.look_at - camera.position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, camera.up)
    nr = np.linalg.norm(right)
    if nr < 1e-12:
        raise ValueError("camera up vector is parallel to the view direction")
    right = right / nr
    up = np.cross(right, fwd)
    half_h = math.tan(math.radians(camera.fov_deg) / 2.0)
    half_w = half_h * (width / height)
    return (float(camera.position[0]), float(camera.position[1]), float(camera.position[2]),
            float(right[0]), float(right[1]), float(right[2]), float(up[0]), float(up[1]), float(up[2]),
            float(fwd[0]), float(fwd[1]), float(fwd[2]), half_w, half_h)
