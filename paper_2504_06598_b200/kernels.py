"""Operator-boundary shim: the reference's compiled-kernel entry points, on the GPU.

``render_stochastic``, ``trace_batch``, ``transmittance_batch``,
``exact_batch``, ``render_exact`` and ``biased_batch`` take the SAME
positional arguments as /root/reference/pkg/src/splatray/kernels.py (lines
622-628, 527-532, 544-549, 584-588, 677-681, 561-565): flat float64/int64
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

import numpy as np

from .scene import DeviceScene


class _Bvh:
    def __init__(self, node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi):
        self.node_lo, self.node_hi = node_lo, node_hi
        self.node_left, self.node_right, self.node_count = node_left, node_right, node_count
        self.prim_order, self.prim_lo, self.prim_hi = prim_order, prim_lo, prim_hi


def _scene(bvh_arrays, means, cov6, opac, sh=None, deg=0, device=0) -> DeviceScene:
    sc = DeviceScene(means, cov6, opac, sh, deg, device)
    sc.upload_bvh(_Bvh(*bvh_arrays))
    return sc


def trace_batch(node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi,
                means, cov6, opac, origins, directions, t_min, t_max, mode, s2, clip, out_t, out_id,
                *, seed=0, ray_id0=0, sample0=0, rng="counter", table=None, device=0):
    """kernels.py:527-540.  N = out_t.shape[1]; ray i draws with ray_id0 + i,
    slot k with sample0 + k."""
    sc = _scene((node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi),
                means, cov6, opac, device=device)
    try:
        t, ids = sc.trace_rays(origins, directions, t_min, t_max, mode, s2, clip, out_t.shape[1], rng, seed,
                               ray_id0, sample0, table)
    finally:
        sc.close()
    out_t[...] = t
    out_id[...] = ids


def transmittance_batch(node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi,
                        means, cov6, opac, origins, directions, t_min, t_max, mode, s2, out, *, device=0):
    """kernels.py:544-557: prod(1 - alpha) over every valid candidate."""
    sc = _scene((node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi),
                means, cov6, opac, device=device)
    try:
        out[...] = sc.transmittance(origins, directions, t_min, t_max, mode, s2)
    finally:
        sc.close()


def render_stochastic(node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi,
                      means, cov6, opac, sh, deg,
                      ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h,
                      width, height, passes, nslots, mode, s2, clip, seed,
                      bgr, bgg, bgb, out_rgb, out_op, *, device=0, rng="counter"):
    """kernels.py:622-673: per-pixel means over passes x nslots samples."""
    sc = _scene((node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi),
                means, cov6, opac, sh, int(deg), device)
    try:
        rgb, op, _ = sc.render((ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h), int(width),
                               int(height), int(passes), int(nslots), int(mode), float(s2), bool(clip), int(seed),
                               (bgr, bgg, bgb), rng=rng)
    finally:
        sc.close()
    out_rgb[...] = rgb
    out_op[...] = op


def _lbvh_scene(means, cov6, opac, sh, deg, s2, device) -> DeviceScene:
    sc = DeviceScene(means, cov6, opac, sh, deg, device)
    sc.build_bvh(float(np.sqrt(s2)))  # boxes at the cutoff radius the validity test uses
    return sc


def exact_batch(means, cov6, opac, sh, deg, origins, directions, t_min, t_max, mode, s2, bgr, bgg, bgb,
                out_rgb, out_op, *, device=0):
    """kernels.py:584-604: exact sorted compositing per explicit ray (the
    reference brute-forces all primitives; here a GPU LBVH collects them)."""
    sc = _lbvh_scene(means, cov6, opac, sh, int(deg), s2, device)
    try:
        rgb, op = sc.exact_rays(origins, directions, t_min, t_max, int(mode), float(s2), (bgr, bgg, bgb))
    finally:
        sc.close()
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
    try:
        rgb = sc.biased_rays(origins, directions, int(kk), t_min, t_max, int(mode), float(s2), (bgr, bgg, bgb), rng,
                             seed, ray_id0, sample0, table)
    finally:
        sc.close()
    out_rgb[...] = rgb


def render_exact(means, cov6, opac, sh, deg, ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h,
                 width, height, frames, mode, s2, seed, bgr, bgg, bgb, out_rgb, out_op, *, device=0):
    """kernels.py:677-723: per-pixel exact composite averaged over `frames` jittered rays."""
    sc = _lbvh_scene(means, cov6, opac, sh, int(deg), s2, device)
    try:
        rgb, op = sc.render_exact((ex, ey, ez, rx, ry, rz, ux, uy, uz, fx, fy, fz, half_w, half_h), int(width),
                                  int(height), int(frames), int(mode), float(s2), int(seed), (bgr, bgg, bgb))
    finally:
        sc.close()
    out_rgb[...] = rgb
    out_op[...] = op


__all__ = ["biased_batch", "exact_batch", "render_exact", "render_stochastic", "trace_batch", "transmittance_batch", "np"]
