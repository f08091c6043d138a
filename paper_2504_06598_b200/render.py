"""The drop-in render API: ``render(asset, camera, settings, bvh=None, threads=None)``.

Same signature, inputs and output type as the reference
(/root/reference/pkg/src/splatray/render.py:125-174): a per-pixel mean image
and opacity in an ``AccumBuffer`` with ``spp = passes * multisample``.  The
frame is traced and shaded on a B200 by libsrt; the acceptance draw is the
counter RNG u(seed, ray = py*W+px, sample = pass*N+slot, prim) instead of the
reference's position hash (the fp64 trig hash cannot be
reproduced by an fp32 tracer).  The device scene (fp32 records + LBVH) is
cached on the asset, keyed by device and cutoff, like the reference caches
``asset.packed``.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib

from .config import CameraConfig, RenderSettings
from .sampling import pixel_jitter
from .scene import DeviceScene, camera_tuple


@dataclass
class AccumBuffer:
    """Per-pixel mean radiance, mean opacity and per-pixel sample count (render.py:32-55)."""

    rgb: np.ndarray
    opacity: np.ndarray
    spp: int

    def __post_init__(self):
        self.rgb = np.asarray(self.rgb, dtype=np.float64)
        self.opacity = np.asarray(self.opacity, dtype=np.float64)
        if self.rgb.ndim != 3 or self.rgb.shape[2] != 3 or self.rgb.shape[:2] != self.opacity.shape:
            raise ValueError("AccumBuffer shapes disagree")
        self.spp = int(self.spp)
        if self.spp < 1:
            raise ValueError("sample count must be positive")

    @property
    def width(self) -> int:
        return int(self.rgb.shape[1])

    @property
    def height(self) -> int:
        return int(self.rgb.shape[0])


class _PinnedBlock:
    """Page-locked host block exposed to numpy as an array of `shape` and
    `dtype`; returned to the pool when the last array viewing it is collected."""

    def __init__(self, pool, ptr: int, nbytes: int, shape, typestr: str):
        self._pool, self._ptr, self._nbytes = pool, ptr, nbytes
        self.__array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3}

    def __del__(self):
        try:
            self._pool.release(self._ptr, self._nbytes)
        except Exception:
            pass


class PinnedPool:
    """Reuses cudaHostAlloc blocks (srt_host_alloc) for render() outputs, so the
    device->host copy of the AccumBuffer runs at link speed."""

    def __init__(self):
        self._free: dict[int, list[int]] = {}
        self._lock = threading.Lock()

    def array(self, shape, dtype=np.float64) -> np.ndarray:
        dt = np.dtype(dtype)
        nbytes = math.prod(shape) * dt.itemsize
        with self._lock:
            lst = self._free.get(nbytes)
            ptr = lst.pop() if lst else None
        if ptr is None:
            p = ctypes.c_void_p()
            _lib.check(_lib.load().srt_host_alloc(nbytes, ctypes.byref(p)))
            ptr = p.value
        return np.asarray(_PinnedBlock(self, ptr, nbytes, tuple(shape), dt.str))

    def release(self, ptr: int, nbytes: int) -> None:
        with self._lock:
            self._free.setdefault(nbytes, []).append(ptr)


_PINNED = PinnedPool()


def camera_basis(camera: CameraConfig):
    """Orthonormal (forward, right, up) of a look-at camera (render.py:58-68)."""
    fwd = camera.look_at - camera.position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, camera.up)
    n = np.linalg.norm(right)
    if n < 1e-12:
        raise ValueError("camera up vector is parallel to the view direction")
    right = right / n
    up = np.cross(right, fwd)
    return fwd, right, up


def generate_camera_ray(camera: CameraConfig, settings: RenderSettings, pixel, frame: int):
    """(origin, unit direction) of the jittered primary ray (render.py:71-94)."""
    fwd, right, up = camera_basis(camera)
    jx, jy = pixel_jitter(pixel, frame, settings.seed)
    px, py = int(pixel[0]), int(pixel[1])
    if not (0 <= px < settings.width and 0 <= py < settings.height):
        raise ValueError(f"pixel {pixel} outside {settings.width}x{settings.height}")
    half_h = math.tan(math.radians(camera.fov_deg) / 2.0)
    half_w = half_h * (settings.width / settings.height)
    u = 2.0 * (px + jx) / settings.width - 1.0
    v = 1.0 - 2.0 * (py + jy) / settings.height
    d = fwd + u * half_w * right + v * half_h * up
    return camera.position.copy(), d / np.linalg.norm(d)


def device_scene(asset, device: int = 0) -> DeviceScene:
    """The asset's cached DeviceScene on `device` (uploaded on first use)."""
    cache = asset.__dict__.setdefault("_srt_device_scenes", {})
    sc = cache.get(device)
    if sc is None:
        sc = DeviceScene.from_packed(asset.packed, device)
        cache[device] = sc
    return sc


def prepare(asset, settings: RenderSettings, bvh=None, device: int = 0) -> DeviceScene:
    """Scene + BVH ready for `settings` (LBVH keyed by cutoff_s, or the given reference BVH)."""
    sc = device_scene(asset, device)
    if bvh is not None:
        if sc.bvh_key != ("upload", id(bvh)):
            sc.upload_bvh(bvh)
    elif sc.bvh_key != ("lbvh", float(settings.cutoff_s)):
        sc.build_bvh(settings.cutoff_s)
    return sc


def render(asset, camera: CameraConfig, settings: RenderSettings, bvh=None, threads: int | None = None,
           device: int = 0, rng: str = "counter", devices=None) -> AccumBuffer:
    """Render a frame on the GPU (render.py:125-174).

    ``threads`` is accepted for signature compatibility (the reference's CPU
    thread count); it has no effect on the GPU.  ``rng="trig64"`` draws the
    reference's own trig-hash stream in fp64 (parity mode, slower).
    ``settings.reference_mode`` renders exact sorted compositing instead
    (render_exact, kernels.py:677-723), with ``spp = passes``.
    ``devices=[d0, d1, ...]`` shards 16x16 tiles over several GPUs from this
    one process (``multi_gpu.render_devices``); same frame, bit for bit.
    """
    del threads
    if devices is not None and len(devices) > 1 and not settings.reference_mode and bvh is None:
        from .multi_gpu import render_devices

        return render_devices(asset, camera, settings, devices, rng=rng)
    sc = prepare(asset, settings, bvh, device)
    cam = camera_tuple(camera, settings.width, settings.height)
    mode = 0 if settings.depth_mode == "mean" else 1
    h, w = settings.height, settings.width
    if settings.reference_mode:
        # exact sorted compositing averaged over the same jittered rays (render.py:156-163)
        rgb, op = sc.render_exact(cam, w, h, settings.passes, mode, settings.cutoff_s * settings.cutoff_s,
                                  settings.seed, settings.background, out_rgb=_PINNED.array((h, w, 3)),
                                  out_op=_PINNED.array((h, w)))
        return AccumBuffer(rgb, op, settings.passes)
    rgb, op, _ = sc.render(cam, w, h, settings.passes, settings.multisample, mode,
                           settings.cutoff_s * settings.cutoff_s, True, settings.seed, settings.background,
                           out_rgb=_PINNED.array((h, w, 3)), out_op=_PINNED.array((h, w)), rng=rng)
    return AccumBuffer(rgb, op, settings.samples_per_pixel)


def render_biased(asset, camera: CameraConfig, settings: RenderSettings, k: int, bvh=None, device: int = 0,
                  rng: str = "counter") -> np.ndarray:
    """The bench's ``--compare-biased K`` frame (cli.py:164-203) on the GPU:
    per pixel, the mean over ``settings.passes`` jittered rays of the biased
    k-nearest composite (kernels.py:479-518).  Returns (H, W, 3) f64."""
    if int(k) < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    sc = prepare(asset, settings, bvh, device)
    cam = camera_tuple(camera, settings.width, settings.height)
    mode = 0 if settings.depth_mode == "mean" else 1
    # pooled mapped page-locked output, as render(): 8.8 -> 5.6 ms for the 1080p
    # k=4 frame against a fresh pageable array (profiles/r02m_resolve/)
    return sc.render_biased(cam, settings.width, settings.height, int(k), settings.passes, mode,
                            settings.cutoff_s * settings.cutoff_s, settings.seed, settings.background, rng=rng,
                            out_rgb=_PINNED.array((settings.height, settings.width, 3)))


def image_metrics(image: AccumBuffer, reference: AccumBuffer) -> dict:
    """MSE / PSNR (peak = max(1, reference max)) and mean |opacity error| (render.py:177-195)."""
    if image.rgb.shape != reference.rgb.shape:
        raise ValueError(f"image shapes disagree: {image.rgb.shape} vs {reference.rgb.shape}")
    diff = image.rgb - reference.rgb
    mse = float(np.mean(diff * diff))
    peak = max(1.0, float(reference.rgb.max()))
    psnr = math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)
    return {"mse": mse, "psnr": psnr,
            "mean_abs_opacity_error": float(np.mean(np.abs(image.opacity - reference.opacity)))}
