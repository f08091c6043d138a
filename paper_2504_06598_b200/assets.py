"""Splat asset container and its packed (kernel-boundary) form.

``SplatAsset`` keeps the reference's structure-of-arrays contract and
validation (/root/reference/pkg/src/splatray/assets.py:60-102).  ``packed``
produces the exact arrays the reference hands its kernels (assets.py:145-171):
the same rotation-matrix formula, the same ``einsum`` for Sigma = R S^2 R^T,
the same batched ``np.linalg.inv`` and symmetrisation, so the float64 inputs
the GPU scene is built from are bitwise those of the reference.  The
per-primitive Python loop of the reference (assets.py:148-150) is vectorised.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np


class EmptyAssetError(ValueError):
    """Raised when an asset contains no primitives."""


def rotation_matrices(q: np.ndarray) -> np.ndarray:
    """(n,3,3) rotation matrices of unit quaternions (w, x, y, z) (gaussians.py:166-176)."""
    w, x, y, z = (q[:, i] for i in range(4))
    r = np.empty((q.shape[0], 3, 3))
    r[:, 0, 0] = 1.0 - 2.0 * (y * y + z * z)
    r[:, 0, 1] = 2.0 * (x * y - w * z)
    r[:, 0, 2] = 2.0 * (x * z + w * y)
    r[:, 1, 0] = 2.0 * (x * y + w * z)
    r[:, 1, 1] = 1.0 - 2.0 * (x * x + z * z)
    r[:, 1, 2] = 2.0 * (y * z - w * x)
    r[:, 2, 0] = 2.0 * (x * z - w * y)
    r[:, 2, 1] = 2.0 * (y * z + w * x)
    r[:, 2, 2] = 1.0 - 2.0 * (x * x + y * y)
    return r


@dataclass
class PackedScene:
    """Flat float64 arrays at the kernel boundary (assets.py:188-195)."""

    means: np.ndarray
    cov_inv: np.ndarray
    cov_inv6: np.ndarray
    opacities: np.ndarray
    sh: np.ndarray
    sh_degree: int
    rot: np.ndarray


@dataclass(eq=False)
class SplatAsset:
    """means (n,3), rotations (n,4) unit quaternions (w,x,y,z), scales (n,3) > 0,
    opacities (n,) in [0,1], sh (n,3,K) with K in {1,4,9,16} (assets.py:60-102)."""

    means: np.ndarray
    rotations: np.ndarray
    scales: np.ndarray
    opacities: np.ndarray
    sh: np.ndarray
    source_path: str = ""

    def __post_init__(self):
        self.means = np.ascontiguousarray(self.means, dtype=np.float64)
        self.rotations = np.ascontiguousarray(self.rotations, dtype=np.float64)
        self.scales = np.ascontiguousarray(self.scales, dtype=np.float64)
        self.opacities = np.ascontiguousarray(self.opacities, dtype=np.float64)
        self.sh = np.ascontiguousarray(self.sh, dtype=np.float64)
        n = self.means.shape[0]
        if n == 0:
            raise EmptyAssetError("asset has no primitives")
        if self.means.shape != (n, 3) or self.rotations.shape != (n, 4) or self.scales.shape != (n, 3):
            raise ValueError("mismatched asset array shapes")
        if self.opacities.shape != (n,) or self.sh.ndim != 3 or self.sh.shape[:2] != (n, 3):
            raise ValueError("mismatched asset array shapes")
        if self.sh.shape[2] not in (1, 4, 9, 16):
            raise ValueError(f"unsupported SH band count {self.sh.shape[2]}")
        for name in ("means", "rotations", "scales", "opacities", "sh"):
            if not np.isfinite(getattr(self, name)).all():
                raise ValueError(f"asset field {name} contains non-finite values")
        norms = np.linalg.norm(self.rotations, axis=1)
        if np.any(norms < 1e-12):
            raise ValueError("asset contains zero-norm rotation quaternions")
        self.rotations = self.rotations / norms[:, None]
        if np.any(self.scales <= 0.0):
            raise ValueError("asset scales must be positive")
        if np.any(self.opacities < 0.0) or np.any(self.opacities > 1.0):
            raise ValueError("asset opacities must lie in [0, 1]")

    def __len__(self) -> int:
        return int(self.means.shape[0])

    @property
    def sh_degree(self) -> int:
        return {1: 0, 4: 1, 9: 2, 16: 3}[self.sh.shape[2]]

    @cached_property
    def packed(self) -> PackedScene:
        rot = rotation_matrices(self.rotations)
        cov = np.einsum("nij,nj,nkj->nik", rot, self.scales**2, rot)
        cov_inv = np.linalg.inv(cov)
        cov_inv = 0.5 * (cov_inv + np.transpose(cov_inv, (0, 2, 1)))
        if not np.isfinite(cov_inv).all():
            raise ValueError("asset contains singular covariances")
        cov_inv6 = np.stack(
            [cov_inv[:, 0, 0], cov_inv[:, 0, 1], cov_inv[:, 0, 2],
             cov_inv[:, 1, 1], cov_inv[:, 1, 2], cov_inv[:, 2, 2]],
            axis=1,
        )
        return PackedScene(
            means=self.means,
            cov_inv=cov_inv,
            cov_inv6=np.ascontiguousarray(cov_inv6),
            opacities=self.opacities,
            sh=self.sh,
            sh_degree=self.sh_degree,
            rot=rot,
        )

    def aabb_arrays(self, s: float) -> tuple[np.ndarray, np.ndarray]:
        """Per-primitive AABB of the s-sigma rotated box (assets.py:173-184)."""
        if s <= 0.0:
            raise ValueError(f"cutoff radius must be positive, got {s}")
        rot = self.packed.rot
        half = s * self.scales
        signs = np.array([[sx, sy, sz] for sx in (-1.0, 1.0) for sy in (-1.0, 1.0) for sz in (-1.0, 1.0)])
        corners = np.einsum("nij,knj->nki", rot, signs[:, None, :] * half[None, :, :])
        return self.means + corners.min(axis=1), self.means + corners.max(axis=1)
