"""ctypes front of the C restatement in ``srt_oracle.c``.

TEST INFRASTRUCTURE.  This module is the parity checker for the sm_100a
product path and the CPU baseline of ``bench.py``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / ``--impl
reference``) may import it.  The product (``paper_2504_06598_b200``) never
does, and fails loudly when its CUDA library is missing.

Parity pinning: in ``rng="trig"`` mode every function here is bitwise equal
to the reference (``/root/reference/pkg/src/splatray/kernels.py``), checked by
``tests/test_oracle_golden.py`` against fixtures generated from the reference
by ``oracle/gen_golden.py``.  ``rng="counter"`` swaps only the acceptance draw
(``kernels.py:354``) for the counter hash the GPU reproduces bit for bit.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"

RNG_MODES = {"trig": 0, "counter": 1, "table": 2}
TMAX = float(np.finfo(np.float64).max)

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_int = ctypes.c_int
_dbl = ctypes.c_double


def build(force: bool = False) -> Path:
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    src = _HERE / "srt_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE), "liboracle.so"], check=True)
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.srt_oracle_hash_position.restype = _dbl
        L.srt_oracle_hash_position.argtypes = [_dbl, _dbl, _dbl, _i64]
        L.srt_oracle_walk_key.restype = _u32
        L.srt_oracle_walk_key.argtypes = [_u32, _u32, _u32]
        L.srt_oracle_counter_u.restype = _dbl
        L.srt_oracle_counter_u.argtypes = [_u32, _u32]
        L.srt_oracle_pixel_jitter.restype = None
        L.srt_oracle_pixel_jitter.argtypes = [_i64, _i64, _i64, _i64, _f64p, _f64p]
        L.srt_oracle_sh_color.restype = None
        L.srt_oracle_sh_color.argtypes = [_f64p, _i64, _i64, _dbl, _dbl, _dbl, _f64p]
        L.srt_oracle_max_threads.restype = _int
        L.srt_oracle_sah_build.restype = _i64
        L.srt_oracle_sah_build.argtypes = [_f64p, _f64p, _i64, _i64, _f64p, _f64p, _i64p, _i64p, _i64p, _i64p]
        bvh_args = [_f64p, _f64p, _i64p, _i64p, _i64p, _i64, _i64p, _f64p, _f64p]
        L.srt_oracle_trace_batch.restype = None
        L.srt_oracle_trace_batch.argtypes = bvh_args + [
            _f64p, _f64p, _f64p, _i64,  # means cov6 opac n
            _f64p, _f64p, _i64, _dbl, _dbl,  # origins dirs R tmin tmax
            _int, _dbl, _int, _int, _u32, _u32, _u32,  # mode s2 clip rng seed ray_id0 sample0
            _f64p, _i64, _i64,  # table table_slots nslots
            _f64p, _i64p, _i64p, _int,  # out_t out_id counters threads
        ]
        L.srt_oracle_render.restype = None
        L.srt_oracle_render.argtypes = bvh_args + [
            _f64p, _f64p, _f64p, _f64p, _i64, _i64,  # means cov6 opac sh n deg
            _f64p, _i64, _i64, _i64, _i64, _i64,  # cam W H passes pass0 nslots
            _int, _dbl, _int, _i64, _int, _f64p,  # mode s2 clip seed rng bg
            _i64, _i64, _f64p, _f64p, _i64p, _i64p, _int,  # strides out_rgb out_op out_ids counters threads
        ]
        L.srt_oracle_transmittance.restype = None
        L.srt_oracle_transmittance.argtypes = bvh_args + [
            _f64p, _f64p, _f64p, _i64, _f64p, _f64p, _i64, _dbl, _dbl, _int, _dbl, _f64p, _int,
        ]
        L.srt_oracle_exact_batch.restype = None
        L.srt_oracle_exact_batch.argtypes = [_f64p, _f64p, _f64p, _f64p, _i64, _i64, _f64p, _f64p, _i64, _dbl, _dbl,
                                             _int, _dbl, _f64p, _f64p, _f64p, _int]
        L.srt_oracle_biased_batch.restype = None
        L.srt_oracle_biased_batch.argtypes = [_f64p, _f64p, _f64p, _f64p, _i64, _i64, _f64p, _f64p, _i64, _dbl, _dbl,
                                              _int, _dbl, _i64, _f64p, _int, ctypes.c_uint32, ctypes.c_uint32,
                                              ctypes.c_uint32, _f64p, _i64, _f64p, _int]
        L.srt_oracle_render_exact.restype = None
        L.srt_oracle_render_exact.argtypes = [_f64p, _f64p, _f64p, _f64p, _i64, _i64, _f64p, _i64, _i64, _i64, _int,
                                              _dbl, _i64, _f64p, _f64p, _f64p, _int]
        _lib = L
    return _lib


def _p(a, ptype=_f64p):
    if a is None:
        return ctypes.cast(None, ptype)
    return a.ctypes.data_as(ptype)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def max_threads() -> int:
    return int(lib().srt_oracle_max_threads())


# ---------------------------------------------------------------------------
# BVH: binned SAH, bit-identical to bvh.build (bvh.py:87-193)
# ---------------------------------------------------------------------------


@dataclass
class OracleBvh:
    """Flat arrays with the reference layout (bvh.py:29-47)."""

    node_lo: np.ndarray
    node_hi: np.ndarray
    node_left: np.ndarray
    node_right: np.ndarray
    node_count: np.ndarray
    prim_order: np.ndarray
    prim_lo: np.ndarray
    prim_hi: np.ndarray
    leaf_size: int = 4

    @property
    def num_nodes(self) -> int:
        return int(self.node_lo.shape[0])

    def args(self):
        return (_p(self.node_lo), _p(self.node_hi), _p(self.node_left, _i64p), _p(self.node_right, _i64p),
                _p(self.node_count, _i64p), _i64(self.num_nodes), _p(self.prim_order, _i64p),
                _p(self.prim_lo), _p(self.prim_hi))


def as_oracle_bvh(b) -> OracleBvh:
    """Wrap any object with the reference Bvh attributes."""
    return OracleBvh(
        _c(b.node_lo, np.float64).reshape(-1, 3), _c(b.node_hi, np.float64).reshape(-1, 3),
        _c(b.node_left, np.int64), _c(b.node_right, np.int64), _c(b.node_count, np.int64),
        _c(b.prim_order, np.int64), _c(b.prim_lo, np.float64).reshape(-1, 3),
        _c(b.prim_hi, np.float64).reshape(-1, 3), int(getattr(b, "leaf_size", 4)),
    )


def sah_build(lo, hi, leaf_size: int = 4) -> OracleBvh:
    lo = _c(lo, np.float64).reshape(-1, 3)
    hi = _c(hi, np.float64).reshape(-1, 3)
    n = lo.shape[0]
    cap = max(2 * n, 1)
    node_lo = np.zeros((cap, 3))
    node_hi = np.zeros((cap, 3))
    node_left = np.zeros(cap, np.int64)
    node_right = np.zeros(cap, np.int64)
    node_count = np.zeros(cap, np.int64)
    prim_order = np.zeros(n, np.int64)
    m = lib().srt_oracle_sah_build(_p(lo), _p(hi), n, leaf_size, _p(node_lo), _p(node_hi), _p(node_left, _i64p),
                                   _p(node_right, _i64p), _p(node_count, _i64p), _p(prim_order, _i64p))
    return OracleBvh(node_lo[:m].copy(), node_hi[:m].copy(), node_left[:m].copy(), node_right[:m].copy(),
                     node_count[:m].copy(), prim_order, lo.copy(), hi.copy(), leaf_size)


# ---------------------------------------------------------------------------
# randomness
# ---------------------------------------------------------------------------


def hash_position(p, slot: int = 0) -> float:
    return float(lib().srt_oracle_hash_position(float(p[0]), float(p[1]), float(p[2]), int(slot)))


def pixel_jitter(px: int, py: int, frame: int, seed: int = 0) -> tuple[float, float]:
    jx, jy = _dbl(), _dbl()
    lib().srt_oracle_pixel_jitter(px, py, frame, seed, ctypes.byref(jx), ctypes.byref(jy))
    return jx.value, jy.value


def walk_key(seed: int, ray_id: int, sample: int) -> int:
    return int(lib().srt_oracle_walk_key(seed & 0xFFFFFFFF, ray_id & 0xFFFFFFFF, sample & 0xFFFFFFFF))


def counter_u(key: int, prim: int) -> float:
    return float(lib().srt_oracle_counter_u(key & 0xFFFFFFFF, prim & 0xFFFFFFFF))


# vectorised numpy restatement of the same counter hash (spec check)
def _mix32_np(x):
    x = np.asarray(x, dtype=np.uint32).copy()
    x ^= x >> np.uint32(16)
    x *= np.uint32(0x7FEB352D)
    x ^= x >> np.uint32(15)
    x *= np.uint32(0x846CA68B)
    x ^= x >> np.uint32(16)
    return x


def counter_u_np(seed, ray_id, sample, prim):
    with np.errstate(over="ignore"):
        k = _mix32_np(_mix32_np(_mix32_np(np.uint32(seed) ^ np.uint32(0x9E3779B9)) ^ np.uint32(ray_id))
                      ^ np.asarray(sample, np.uint32))
        h = _mix32_np(_mix32_np(k ^ np.asarray(prim, np.uint32)) ^ np.uint32(0x68E31DA4))
    return (h >> np.uint32(8)).astype(np.float64) * (1.0 / 16777216.0)


def sh_color(sh, deg: int, pid: int, d) -> np.ndarray:
    sh = _c(sh, np.float64)
    out = np.empty(3)
    lib().srt_oracle_sh_color(_p(sh), deg, pid, float(d[0]), float(d[1]), float(d[2]), _p(out))
    return out


# ---------------------------------------------------------------------------
# traversal
# ---------------------------------------------------------------------------

COUNTER_NAMES = ("inner", "prim_tests", "candidates", "draws", "hits", "max_depth")


def trace_batch(bvh: OracleBvh, means, cov6, opac, origins, dirs, t_min=0.0, t_max=TMAX, mode=0,
                s2=8.0, clip=True, nslots=1, rng="trig", seed=0, ray_id0=0, sample0=0, table=None,
                counters=False, threads=0):
    """kernels.trace_batch (kernels.py:527-540) with a switchable draw.

    Returns (out_t (R,nslots) f64, out_id (R,nslots) i64[, counters dict])."""
    means = _c(means, np.float64)
    cov6 = _c(cov6, np.float64)
    opac = _c(opac, np.float64)
    origins = _c(origins, np.float64).reshape(-1, 3)
    dirs = _c(dirs, np.float64).reshape(-1, 3)
    R = origins.shape[0]
    out_t = np.empty((R, nslots))
    out_id = np.empty((R, nslots), np.int64)
    tab = None if table is None else _c(table, np.float64)
    cnt = np.zeros(6, np.int64) if counters else None
    lib().srt_oracle_trace_batch(*bvh.args(), _p(means), _p(cov6), _p(opac), means.shape[0], _p(origins), _p(dirs),
                                 R, float(t_min), float(t_max), int(mode), float(s2), int(bool(clip)),
                                 RNG_MODES[rng], seed & 0xFFFFFFFF, ray_id0 & 0xFFFFFFFF, sample0 & 0xFFFFFFFF,
                                 _p(tab), 0 if tab is None else tab.shape[1], nslots, _p(out_t),
                                 _p(out_id, _i64p), _p(cnt, _i64p), int(threads))
    if counters:
        return out_t, out_id, dict(zip(COUNTER_NAMES, (int(v) for v in cnt)))
    return out_t, out_id


def transmittance(bvh: OracleBvh, means, cov6, opac, origins, dirs, t_min=0.0, t_max=TMAX, mode=0, s2=8.0,
                  threads=0):
    means = _c(means, np.float64)
    cov6 = _c(cov6, np.float64)
    opac = _c(opac, np.float64)
    origins = _c(origins, np.float64).reshape(-1, 3)
    dirs = _c(dirs, np.float64).reshape(-1, 3)
    out = np.empty(origins.shape[0])
    lib().srt_oracle_transmittance(*bvh.args(), _p(means), _p(cov6), _p(opac), means.shape[0], _p(origins),
                                   _p(dirs), origins.shape[0], float(t_min), float(t_max), int(mode), float(s2),
                                   _p(out), int(threads))
    return out


def camera_tuple(position, look_at, up, fov_deg, width, height):
    """The 14 camera scalars of render.py:140-150 (camera_basis render.py:58-68)."""
    position = np.asarray(position, np.float64)
    fwd = np.asarray(look_at, np.float64) - position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right = right / np.linalg.norm(right)
    upv = np.cross(right, fwd)
    half_h = math.tan(math.radians(fov_deg) / 2.0)
    half_w = half_h * (width / height)
    return np.array([*position, *right, *upv, *fwd, half_w, half_h], dtype=np.float64)


def render(bvh: OracleBvh, means, cov6, opac, sh, deg, cam, width, height, passes=1, nslots=1, mode=0,
           s2=8.0, clip=True, seed=0, rng="trig", background=(0.0, 0.0, 0.0), stride=(1, 1), pass0=0,
           want_ids=False, counters=False, threads=0):
    """kernels.render_stochastic (kernels.py:622-673) with a switchable draw.

    Returns dict(rgb (H,W,3), opacity (H,W)[, ids (H,W,nslots) of pass pass0][, counters])."""
    means = _c(means, np.float64)
    cov6 = _c(cov6, np.float64)
    opac = _c(opac, np.float64)
    sh = _c(sh, np.float64)
    cam = _c(cam, np.float64)
    bg = _c(background, np.float64)
    rgb = np.zeros((height, width, 3))
    op = np.zeros((height, width))
    ids = np.full((height, width, nslots), -2, np.int64) if want_ids else None
    cnt = np.zeros(6, np.int64) if counters else None
    lib().srt_oracle_render(*bvh.args(), _p(means), _p(cov6), _p(opac), _p(sh), means.shape[0], int(deg), _p(cam),
                            int(width), int(height), int(passes), int(pass0), int(nslots), int(mode), float(s2),
                            int(bool(clip)), int(seed), RNG_MODES[rng], _p(bg), int(stride[0]), int(stride[1]),
                            _p(rgb), _p(op), _p(ids, _i64p), _p(cnt, _i64p), int(threads))
    out = {"rgb": rgb, "opacity": op}
    if want_ids:
        out["ids"] = ids
    if counters:
        out["counters"] = dict(zip(COUNTER_NAMES, (int(v) for v in cnt)))
    return out


def exact_batch(means, cov6, opac, sh, deg, origins, dirs, t_min=0.0, t_max=TMAX, mode=0, s2=8.0,
                background=(0.0, 0.0, 0.0), threads=0):
    """kernels.exact_batch (kernels.py:584-604): brute-force sorted compositing."""
    means, cov6, opac, sh = (_c(x, np.float64) for x in (means, cov6, opac, sh))
    origins = _c(origins, np.float64).reshape(-1, 3)
    dirs = _c(dirs, np.float64).reshape(-1, 3)
    bg = _c(background, np.float64)
    rgb = np.empty((origins.shape[0], 3))
    op = np.empty(origins.shape[0])
    lib().srt_oracle_exact_batch(_p(means), _p(cov6), _p(opac), _p(sh), means.shape[0], int(deg), _p(origins),
                                 _p(dirs), origins.shape[0], float(t_min), float(t_max), int(mode), float(s2), _p(bg),
                                 _p(rgb), _p(op), int(threads))
    return rgb, op


def biased_batch(means, cov6, opac, sh, deg, origins, dirs, kk, t_min=0.0, t_max=TMAX, mode=0, s2=8.0,
                 background=(0.0, 0.0, 0.0), rng="trig", seed=0, ray_id0=0, sample0=0, table=None, threads=0):
    """kernels.biased_batch (kernels.py:561-580): brute force, one draw per
    candidate, kk nearest accepted composited.  rng "trig" is the reference."""
    means, cov6, opac, sh = (_c(x, np.float64) for x in (means, cov6, opac, sh))
    origins = _c(origins, np.float64).reshape(-1, 3)
    dirs = _c(dirs, np.float64).reshape(-1, 3)
    bg = _c(background, np.float64)
    tab = _c(table if table is not None else np.zeros((1, 1)), np.float64)
    if tab.ndim == 1:
        tab = tab.reshape(-1, 1)
    rgb = np.empty((origins.shape[0], 3))
    lib().srt_oracle_biased_batch(_p(means), _p(cov6), _p(opac), _p(sh), means.shape[0], int(deg), _p(origins),
                                  _p(dirs), origins.shape[0], float(t_min), float(t_max), int(mode), float(s2),
                                  int(kk), _p(bg), RNG_MODES[rng], seed & 0xFFFFFFFF, ray_id0 & 0xFFFFFFFF,
                                  sample0 & 0xFFFFFFFF, _p(tab), tab.shape[1], _p(rgb), int(threads))
    return rgb


def render_exact(means, cov6, opac, sh, deg, cam, width, height, frames=1, mode=0, s2=8.0, seed=0,
                 background=(0.0, 0.0, 0.0), threads=0):
    """kernels.render_exact (kernels.py:677-723)."""
    means, cov6, opac, sh = (_c(x, np.float64) for x in (means, cov6, opac, sh))
    cam = _c(cam, np.float64)
    bg = _c(background, np.float64)
    rgb = np.zeros((height, width, 3))
    op = np.zeros((height, width))
    lib().srt_oracle_render_exact(_p(means), _p(cov6), _p(opac), _p(sh), means.shape[0], int(deg), _p(cam),
                                  int(width), int(height), int(frames), int(mode), float(s2), int(seed), _p(bg),
                                  _p(rgb), _p(op), int(threads))
    return rgb, op


def library_path() -> str:
    return os.fspath(_LIB_PATH)
