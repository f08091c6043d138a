"""ctypes binding of libsrt.so (the C ABI declared in include/srt.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises.  Build with ``python -c "import
__graft_entry__ as g; g.build()"`` or ``make -C paper_2504_06598_b200/csrc``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# SRT_LIBSRT_PATH overrides the in-tree library (A/B timing of two builds)
LIB_PATH = Path(os.environ.get("SRT_LIBSRT_PATH", _HERE / "libsrt.so"))

SRT_OK = 0
SRT_RNG_COUNTER = 1
SRT_RNG_TABLE = 2
SRT_RNG_TRIG64 = 3
_STATUS_NAMES = {1: "invalid argument", 2: "CUDA error", 3: "out of device memory", 4: "no BVH",
                 5: "stack overflow", 6: "unsupported"}


class SrtError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"libsrt {_STATUS_NAMES.get(status, status)}: {message}")
        self.status = status


class SrtSceneDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("means", ctypes.c_void_p), ("cov_inv6", ctypes.c_void_p),
                ("opacities", ctypes.c_void_p), ("sh", ctypes.c_void_p), ("sh_degree", ctypes.c_int32)]


class SrtSplatDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("means", ctypes.c_void_p), ("rotations", ctypes.c_void_p),
                ("scales", ctypes.c_void_p), ("opacities", ctypes.c_void_p), ("sh", ctypes.c_void_p),
                ("sh_degree", ctypes.c_int32)]


class SrtCamera(ctypes.Structure):
    _fields_ = [("position", ctypes.c_double * 3), ("right", ctypes.c_double * 3), ("up", ctypes.c_double * 3),
                ("forward", ctypes.c_double * 3), ("half_w", ctypes.c_double), ("half_h", ctypes.c_double)]


class SrtRenderParams(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("passes", ctypes.c_int32),
                ("nslots", ctypes.c_int32), ("mode", ctypes.c_int32), ("clip", ctypes.c_int32),
                ("s2", ctypes.c_double), ("seed", ctypes.c_uint32), ("pass0", ctypes.c_int32),
                ("background", ctypes.c_double * 3), ("shard_index", ctypes.c_int32),
                ("shard_count", ctypes.c_int32), ("rng", ctypes.c_int32)]


class SrtTraceParams(ctypes.Structure):
    _fields_ = [("t_min", ctypes.c_double), ("t_max", ctypes.c_double), ("mode", ctypes.c_int32),
                ("clip", ctypes.c_int32), ("s2", ctypes.c_double), ("rng", ctypes.c_int32),
                ("seed", ctypes.c_uint32), ("ray_id0", ctypes.c_uint32), ("sample0", ctypes.c_uint32),
                ("table", ctypes.c_void_p), ("table_slots", ctypes.c_int64)]


# (name, restype, argtypes): every symbol include/srt.h declares
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
SYMBOLS = [
    ("srt_last_error", ctypes.c_char_p, []),
    ("srt_version", ctypes.c_char_p, []),
    ("srt_build_id", ctypes.c_char_p, []),
    ("srt_probe_l2_bandwidth", _i32, [_i32, _i64, _i32, ctypes.POINTER(_f64)]),
    ("srt_device_count", _i32, []),
    ("srt_host_alloc", _i32, [_i64, ctypes.POINTER(_vp)]),
    ("srt_host_free", _i32, [_vp]),
    ("srt_host_register", _i32, [_vp, _i64]),
    ("srt_host_unregister", _i32, [_vp]),
    ("srt_scene_create", _i32, [ctypes.POINTER(SrtSceneDesc), _i32, ctypes.POINTER(_vp)]),
    ("srt_scene_destroy", _i32, [_vp]),
    ("srt_scene_create_from_splats", _i32, [ctypes.POINTER(SrtSplatDesc), _i32, ctypes.POINTER(_vp)]),
    ("srt_bvh_build", _i32, [_vp, _f64]),
    ("srt_bvh_build_ex", _i32, [_vp, _f64, _i32]),
    ("srt_bvh_upload", _i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("srt_bvh_split_info", _i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    ("srt_bvh_info", _i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i64),
                            ctypes.POINTER(_i64)]),
    ("srt_bvh_download", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("srt_trace_rays", _i32, [_vp, ctypes.POINTER(SrtTraceParams), _vp, _vp, _i64, _i32, _vp, _vp]),
    ("srt_trace_rays_device", _i32, [_vp, ctypes.POINTER(SrtTraceParams), _vp, _i64, _i32, _vp, _vp, _vp]),
    ("srt_transmittance_rays", _i32, [_vp, _vp, _vp, _i64, _f64, _f64, _i32, _f64, _vp]),
    ("srt_exact_rays", _i32, [_vp, _vp, _vp, _i64, _f64, _f64, _i32, _f64, _vp, _vp, _vp]),
    ("srt_biased_rays", _i32, [_vp, ctypes.POINTER(SrtTraceParams), _vp, _vp, _i64, _i32, _vp, _vp]),
    ("srt_render_biased", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _i32, _vp]),
    ("srt_render_exact", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _vp, _vp]),
    ("srt_render", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _vp, _vp, _vp]),
    ("srt_trace_pass_device", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _i32, _vp,
                                     _vp]),
    ("srt_shade_pass_device", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _i32, _vp,
                                     _vp, _i32, _i32, _vp, _vp]),
    ("srt_render_pass_device", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _i32, _vp,
                                      _i32, _i32, _vp, _vp]),
    ("srt_render_frame_device", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _vp, _vp,
                                       _vp]),
    ("srt_resolve_frame_device", _i32, [ctypes.POINTER(SrtRenderParams), _vp, _vp, _vp, _vp]),
    ("srt_render_pass_frame_device", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _i32,
                                            _vp, _i32, _i32, _vp, _i32, _vp]),
    ("srt_ipc_alloc", _i32, [_i32, _i64, ctypes.POINTER(_vp), _vp]),
    ("srt_ipc_open", _i32, [_i32, _vp, ctypes.POINTER(_vp)]),
    ("srt_ipc_close", _i32, [_i32, _vp]),
    ("srt_ipc_free", _i32, [_i32, _vp]),
    ("srt_render_device", _i32, [_vp, ctypes.POINTER(SrtCamera), ctypes.POINTER(SrtRenderParams), _vp, _vp, _vp,
                                 _vp]),
    ("srt_scene_check", _i32, [_vp, _i32]),
    ("srt_hash_positions", _i32, [_vp, _i64, _i64, _vp, _i32]),
    ("srt_pixel_jitter", _i32, [_i64, _i64, _vp, _i64, ctypes.c_uint32, _vp, _i32]),
    ("srt_trace_stats", _i32, [_vp, _vp, _i32]),
    ("srt_trace_counters", _i32, [_vp, _vp, _i32, _i32]),
    ("srt_shard_tiles", _i64, [_i32, _i32, _i32, _i32]),
    ("srt_unpack_tiles_device", _i32, [_vp, _i32, _i32, _i32, _i64, _vp, _vp]),
]

_lib = None


def load() -> ctypes.CDLL:
    """Load libsrt.so and bind every exported symbol (raises if absent)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                              f"(there is no CPU fallback for the GPU renderer)")
        lib = ctypes.CDLL(os.fspath(LIB_PATH))
        override = "SRT_LIBSRT_PATH" in os.environ
        for name, res, args in SYMBOLS:
            if override and not hasattr(lib, name):
                continue  # an older build under A/B comparison
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != SRT_OK:
        msg = load().srt_last_error().decode(errors="replace")
        if status == 1:
            raise ValueError(f"libsrt: {msg}")
        raise SrtError(status, msg)


def require_device() -> int:
    """Number of visible CUDA devices; raises when there is none."""
    n = load().srt_device_count()
    if n < 1:
        raise SrtError(2, "no CUDA device visible (the renderer has no CPU fallback)")
    return n
