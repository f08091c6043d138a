"""Operator-boundary shim: the reference's compiled-kernel entry points, on the GPU.

``render_stochastic``, ``trace_batch``, ``transmittance_batch``,
``exact_batch``, ``render_exact``, ``biased_batch``, ``hash_position_batch``
and ``pixel_jitter_batch`` -- every public entry point of
/root/reference/pkg/src/splatray/kernels.py -- take the SAME positional
arguments (lines 622-628, 527-532, 544-549, 584-588, 677-681, 561-565,
119-122, 125-135): flat float64/int64
numpy arrays in, outputs written in place, None returned.  Pointing the reference's callers
(``render.py:166-173``, ``validate.py:106,177``, its acceptance tests) at
this module swaps its numba CPU loops for libsrt.  Keyword-only extras
select the counter stream (seed / ray_id0 / sample0), a scripted ``table``
of uniforms, ``rng="trig64"`` (the reference's own trig-hash draw in fp64,
for direct comparison with the unmodified reference), and the device.

Differences from the reference, by construction:
* the default acceptance draw is the counter RNG (or a table), not the trig
  hash of the fp64 hit position; ``rng="trig64"`` restores
  the reference's own draw;
* depths are traced in fp32 (``out_t`` agrees to ~1e-6 relative);
* multi-primitive reference leaves keep their per-primitive box tests.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import numpy as np

from . import _lib
from .scene import DeviceScene


class _Bvh:
    def __init__(self, node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi):
        self.node_lo, self.node_hi = node_lo, node_hi
        self.node_left, self.node_right, self.node_count = node_left, node_right, node_count
        self.prim_order, self.prim_lo, self.prim_hi = prim_order, prim_lo, prim_hi


def _fingerprint(a) -> tuple:
    """Identity of an input array as the reference's callers pass them: object
    id, buffer address, shape, dtype, plus a 64-element strided sample of its
    values (catches in-place rewrites of a reused buffer without hashing the
    whole scene every call)."""
    if a is None:
        return (None,)
    if not isinstance(a, np.ndarray):
        return ("value", repr(a))
    flat = a.reshape(-1)
    step = max(1, flat.shape[0] // 64)
    return (id(a), a.__array_interface__["data"][0], a.shape, a.dtype.str, flat[::step][:64].tobytes())


class _SceneCache:
    """Device scenes of recent (scene arrays, BVH arrays) inputs, so repeated
    calls through the shim -- a render loop, validate.py's checks -- upload
    and convert the scene once, as the reference caches ``asset.packed``
    (assets.py:144) and ``render(bvh=...)`` reuses a prebuilt tree
    (render.py:164-165).  The cache holds references to the keyed arrays, so
    their ids stay unique while cached.  Small LRU (multi-GB scenes)."""

    def __init__(self, capacity: int = 4):
        self.capacity = capacity
        self._d: OrderedDict = OrderedDict()
        self._lock = threading.Lock()

    def get(self, arrays: tuple, make):
        key = tuple(_fingerprint(a) for a in arrays)
        with self._lock:
            hit = self._d.get(key)
            if hit is not None:
                self._d.move_to_end(key)
                return hit[0]
        sc = make()
        with self._lock:
            self._d[key] = (sc, arrays)
            while len(self._d) > self.capacity:
                old, _ = self._d.popitem(last=False)[1]
                old.close()
        return sc

    def clear(self) -> None:
        with self._lock:
            for sc, _ in self._d.values():
                sc.close()
            self._d.clear()


_CACHE = _SceneCache()


def _scene(bvh_arrays, means, cov6, opac, sh=None, deg=0, device=0) -> DeviceScene:
    def make():
        sc = DeviceScene(means, cov6, opac, sh, deg, device)
        sc.upload_bvh(_Bvh(*bvh_arrays))
        return sc

    return _CACHE.get((*bvh_arrays, means, cov6, opac, sh, int(deg), int(device)), make)


def trace_batch(node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi,
                means, cov6, opac, origins, directions, t_min, t_max, mode, s2, clip, out_t, out_id,
                *, seed=0, ray_id0=0, sample0=0, rng="counter", table=None, device=0):
    """kernels.py:527-540.  N = out_t.shape[1]; ray i draws with ray_id0 + i,
    slot k with sample0 + k."""
    sc = _scene((node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi),
                means, cov6, opac, device=device)
    t, ids = sc.trace_rays(origins, directions, t_min, t_max, mode, s2, clip, out_t.shape[1], rng, seed,
                           ray_id0, sample0, table)
    out_t[...] = t
    out_id[...] = ids


def transmittance_batch(node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi,
                        means, cov6, opac, origins, directions, t_min, t_max, mode, s2, out, *, device=0):
    """kernels.py:544-557: prod(1 - alpha) over every valid candidate."""
    sc = _scene((node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi),
                means, cov6, opac, device=device)
    out[...] = sc.transmittance(origins, directions, t_min, t_max, mode, s2)


def render_stochastic(node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi,
                      means, cov6, opac, sh, deg,
                      ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h,
                      width, height, passes, nslots, mode, s2, clip, seed,
                      bgr, bgg, bgb, out_rgb, out_op, *, device=0, rng="counter"):
    """kernels.py:622-673: per-pixel means over passes x nslots samples."""
    sc = _scene((node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi),
                means, cov6, opac, sh, int(deg), device)
    # results straight into the caller's arrays when they are C-contiguous f64
    direct = _is_f64c(out_rgb) and _is_f64c(out_op)
    rgb, op, _ = sc.render((ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h), int(width),
                           int(height), int(passes), int(nslots), int(mode), float(s2), bool(clip), int(seed),
                           (bgr, bgg, bgb), rng=rng, out_rgb=out_rgb if direct else None,
                           out_op=out_op if direct else None)
    if not direct:
        out_rgb[...] = rgb
        out_op[...] = op


def _is_f64c(a) -> bool:
    return isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous


def _lbvh_scene(means, cov6, opac, sh, deg, s2, device) -> DeviceScene:
    def make():
        sc = DeviceScene(means, cov6, opac, sh, deg, device)
        sc.build_bvh(float(np.sqrt(s2)))  # boxes at the cutoff radius the validity test uses
        return sc

    return _CACHE.get(("lbvh", means, cov6, opac, sh, int(deg), float(s2), int(device)), make)


def exact_batch(means, cov6, opac, sh, deg, origins, directions, t_min, t_max, mode, s2, bgr, bgg, bgb,
                out_rgb, out_op, *, device=0):
    """kernels.py:584-604: exact sorted compositing per explicit ray (the
    reference brute-forces all primitives; here a GPU LBVH collects them)."""
    sc = _lbvh_scene(means, cov6, opac, sh, int(deg), s2, device)
    rgb, op = sc.exact_rays(origins, directions, t_min, t_max, int(mode), float(s2), (bgr, bgg, bgb))
    out_rgb[...] = rgb
    out_op[...] = op


def biased_batch(means, cov6, opac, sh, deg, origins, directions, t_min, t_max, mode, s2, kk, bgr, bgg, bgb,
                 out_rgb, *, seed=0, ray_id0=0, sample0=0, rng="counter", table=None, device=0):
    """kernels.py:561-580 (the `--compare-biased` baseline, cli.py:164-203):
    per ray, one acceptance draw per valid candidate, then the kk nearest
    accepted composited front to back with their original alphas."""
    if int(kk) < 1:
        raise ValueError(f"k must be >= 1, got {kk}")  # tracer.py:325-326
    sc = _lbvh_scene(means, cov6, opac, sh, int(deg), s2, device)
    rgb = sc.biased_rays(origins, directions, int(kk), t_min, t_max, int(mode), float(s2), (bgr, bgg, bgb), rng,
                         seed, ray_id0, sample0, table)
    out_rgb[...] = rgb


def render_exact(means, cov6, opac, sh, deg, ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h,
                 width, height, frames, mode, s2, seed, bgr, bgg, bgb, out_rgb, out_op, *, device=0):
    """kernels.py:677-723: per-pixel exact composite averaged over `frames` jittered rays."""
    sc = _lbvh_scene(means, cov6, opac, sh, int(deg), s2, device)
    rgb, op = sc.render_exact((ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h), int(width),
                              int(height), int(frames), int(mode), float(s2), int(seed), (bgr, bgg, bgb))
    out_rgb[...] = rgb
    out_op[...] = op


def hash_position_batch(points, slot, out, *, device=0):
    """kernels.py:119-122: out[i] = the reference's trig hash of points[i] for
    `slot` (fp64 on the GPU; device sin agrees with the CPU's to ~1e-5)."""
    p = np.ascontiguousarray(points, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 3:
        raise ValueError(f"points must be (n, 3), got {p.shape}")
    res = np.empty(p.shape[0])
    _lib.check(_lib.load().srt_hash_positions(ctypes.c_void_p(p.ctypes.data), p.shape[0], int(slot),
                                              ctypes.c_void_p(res.ctypes.data), int(device)))
    out[...] = res


def pixel_jitter_batch(px, py, frames, seed, out, *, device=0):
    """kernels.py:125-135: out[i] = the scrambled Sobol jitter (jx, jy) of pixel
    (px, py) for frames[i] (integer exact on the GPU)."""
    f = np.ascontiguousarray(frames, dtype=np.int64).reshape(-1)
    res = np.empty((f.shape[0], 2))
    _lib.check(_lib.load().srt_pixel_jitter(int(px), int(py), ctypes.c_void_p(f.ctypes.data), f.shape[0],
                                            int(seed) & 0xFFFFFFFF, ctypes.c_void_p(res.ctypes.data), int(device)))
    out[...] = res


__all__ = ["biased_batch", "exact_batch", "hash_position_batch", "pixel_jitter_batch", "render_exact",
           "render_stochastic", "trace_batch", "transmittance_batch", "np"]
