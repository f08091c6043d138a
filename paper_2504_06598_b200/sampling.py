"""Host-side statement of the two random streams the GPU consumes.

* ``pixel_jitter``: the reference's scrambled Sobol (0,2) jitter
  (/root/reference/pkg/src/splatray/sampling.py:84-156), integer exact; the
  device copy is ``pixel_jitter`` in csrc/srt_device.cuh.
* ``counter_uniform``: the acceptance draw u(seed, ray, sample, prim) that
  replaces the reference's position hash (kernels.py:354);
  the device copy is ``counter_u`` in csrc/srt_device.cuh.
"""

from __future__ import annotations

import numpy as np

_MASK32 = 0xFFFFFFFF
_INV32 = 1.0 / 4294967296.0


def _wang32(x: int) -> int:
    x &= _MASK32
    x = (x ^ 61) ^ (x >> 16)
    x = (x * 9) & _MASK32
    x ^= x >> 4
    x = (x * 0x27D4EB2D) & _MASK32
    x ^= x >> 15
    return x


def _sobol_bits(index: int) -> tuple[int, int]:
    """Dimension 0 (bit reversal) and dimension 1 (x^2+x+1) of Sobol point index."""
    i = index & _MASK32
    x = int(f"{i:032b}"[::-1], 2)
    y, m, k = 0, 1, 0
    while i:
        if i & 1:
            y ^= m << (31 - k)
        m = (m ^ (m << 1)) & ((1 << (k + 2)) - 1)
        i >>= 1
        k += 1
    return x, y & _MASK32


def pixel_jitter(pixel, frame: int, seed: int = 0) -> np.ndarray:
    """Sub-pixel offset in [0,1)^2 of a pixel at a pass index (sampling.py:134-147)."""
    px, py = int(pixel[0]), int(pixel[1])
    frame = int(frame)
    if frame < 0:
        raise ValueError("frame index must be nonnegative")
    base = _wang32(((px & _MASK32) * 0x9E3779B1) & _MASK32 ^ ((py & _MASK32) * 0x85EBCA77) & _MASK32
                   ^ ((int(seed) & _MASK32) * 0xC2B2AE3D) & _MASK32)
    sx, sy = _wang32(base ^ 0x68E31DA4), _wang32(base ^ 0xB5297A4D)
    bx, by = _sobol_bits(frame)
    return np.array([(bx ^ sx) * _INV32, (by ^ sy) * _INV32])


def _mix32(x):
    x = np.asarray(x, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x7FEB352D)
        x ^= x >> np.uint32(15)
        x *= np.uint32(0x846CA68B)
        x ^= x >> np.uint32(16)
    return x


def counter_uniform(seed, ray_id, sample, prim) -> np.ndarray:
    """u = U24(mix(mix(K ^ prim) ^ 0x68E31DA4)), K = mix(mix(mix(seed ^ 0x9E3779B9) ^ ray) ^ sample).

    Camera rays use ray_id = py * width + px and sample = pass * N + slot.
    Broadcasts over array arguments; exact (24-bit) so CPU and GPU agree bit for bit.
    """
    k = _mix32(_mix32(_mix32(np.uint32(seed & _MASK32) ^ np.uint32(0x9E3779B9))
                      ^ np.asarray(ray_id, np.int64).astype(np.uint32))
               ^ np.asarray(sample, np.int64).astype(np.uint32))
    h = _mix32(_mix32(k ^ np.asarray(prim, np.int64).astype(np.uint32)) ^ np.uint32(0x68E31DA4))
    return (h >> np.uint32(8)).astype(np.float64) * (1.0 / 16777216.0)
