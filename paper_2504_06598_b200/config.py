"""Render settings and camera description -- the drop-in surface's input types.

Same fields, defaults, validation and error types as the reference's
``splatray.config`` (/root/reference/pkg/src/splatray/config.py:26-94), so
code written against the reference constructs them unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Mahalanobis cutoff radius (gaussians.py:22): exp(-0.5 * 8) ~ 2% of the peak.
DEFAULT_CUTOFF = 2.0 * math.sqrt(2.0)
DEPTH_MODES = ("mean", "center")
MULTISAMPLE_MAX = 256


class ConfigError(ValueError):
    """Invalid setting values (config.py:21-22)."""


def _vec3(v) -> np.ndarray:
    return np.asarray(v, dtype=np.float64).reshape(3)


@dataclass
class CameraConfig:
    """Pinhole camera (config.py:26-47): position, target, up hint, vertical fov."""

    position: np.ndarray
    look_at: np.ndarray = field(default_factory=lambda: np.zeros(3))
    up: np.ndarray = field(default_factory=lambda: np.array([0.0, 1.0, 0.0]))
    fov_deg: float = 60.0

    def __post_init__(self):
        self.position = _vec3(self.position)
        self.look_at = _vec3(self.look_at)
        self.up = _vec3(self.up)
        self.fov_deg = float(self.fov_deg)
        for name in ("position", "look_at", "up"):
            if not np.isfinite(getattr(self, name)).all():
                raise ConfigError(f"camera {name} must be finite")
        if np.allclose(self.position, self.look_at):
            raise ConfigError("camera position and look_at coincide")
        if np.linalg.norm(self.up) < 1e-12:
            raise ConfigError("camera up vector is zero")
        if not 0.0 < self.fov_deg < 180.0:
            raise ConfigError(f"fov_deg must lie in (0, 180), got {self.fov_deg}")


@dataclass
class RenderSettings:
    """Everything about a render that is not the camera or the asset (config.py:51-94)."""

    width: int = 640
    height: int = 480
    spp: int = 64
    depth_mode: str = "mean"
    cutoff_s: float = DEFAULT_CUTOFF
    multisample: int = 1
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    seed: int = 0
    reference_mode: bool = False

    def __post_init__(self):
        self.width = int(self.width)
        self.height = int(self.height)
        self.spp = int(self.spp)
        self.multisample = int(self.multisample)
        self.seed = int(self.seed)
        self.cutoff_s = float(self.cutoff_s)
        self.background = _vec3(self.background)
        self.reference_mode = bool(self.reference_mode)
        if self.width < 1 or self.height < 1:
            raise ConfigError(f"image size must be positive, got {self.width}x{self.height}")
        if self.spp < 1:
            raise ConfigError(f"spp must be >= 1, got {self.spp}")
        if self.depth_mode not in DEPTH_MODES:
            raise ConfigError(f"depth_mode must be one of {DEPTH_MODES}, got {self.depth_mode!r}")
        if not 1 <= self.multisample <= MULTISAMPLE_MAX:
            raise ConfigError(f"multisample must lie in [1, {MULTISAMPLE_MAX}], got {self.multisample}")
        if self.cutoff_s <= 0.0 or not np.isfinite(self.cutoff_s):
            raise ConfigError(f"cutoff_s must be positive and finite, got {self.cutoff_s}")
        if not np.isfinite(self.background).all() or np.any(self.background < 0.0):
            raise ConfigError("background must be finite and nonnegative")

    @property
    def passes(self) -> int:
        """Traversals per pixel: ceil(spp / multisample) (config.py:87-89)."""
        return -(-self.spp // self.multisample)

    @property
    def samples_per_pixel(self) -> int:
        """passes * multisample >= spp (config.py:91-94)."""
        return self.passes * self.multisample
