"""paper_2504_06598_b200: B200-native stochastic ray tracing of transparent 3D Gaussians.

Drop-in for the hot path of the reference package ``splatray``
(arXiv 2504.06598): ``render(asset, camera, settings)`` and the kernel-level
entry points of ``kernels`` run on hand-written sm_100a CUDA (``csrc/``, C
ABI in ``include/srt.h``): a GPU PLOC/LBVH build, a warp-packet stochastic
N-slot traversal driven by a counter RNG with SH shading fused into the
walk, exact and biased compositing, the reference's trig-hash stream in
fp64 (``rng="trig64"``), PLY ingest and multi-GPU frame drivers.  There is
no CPU fallback.
"""

from .assets import EmptyAssetError, PackedScene, SplatAsset
from .config import DEFAULT_CUTOFF, CameraConfig, ConfigError, RenderSettings
from .ply import PlyFormatError, load_ply, save_ply
from .render import AccumBuffer, camera_basis, generate_camera_ray, image_metrics, render, render_biased
from .sampling import counter_uniform, pixel_jitter
from .scene import DeviceScene
from .synthetic import (anisotropic_sheets, density_cloud, front_camera, pancake_stack, random_cloud,
                        two_layer_scene)

__version__ = "0.1.0"

__all__ = [
    "AccumBuffer", "CameraConfig", "ConfigError", "DEFAULT_CUTOFF", "DeviceScene", "EmptyAssetError",
    "PackedScene", "PlyFormatError", "RenderSettings", "SplatAsset", "anisotropic_sheets", "camera_basis",
    "counter_uniform", "density_cloud", "front_camera", "generate_camera_ray", "image_metrics", "load_ply",
    "pancake_stack", "pixel_jitter", "random_cloud", "render", "render_biased", "save_ply", "two_layer_scene",
]
