"""Generate the at-scale convergence fixture tests/golden/c5_converged_grid.npz
(TEST INFRASTRUCTURE; run here, on CPU, in a few minutes):

    python oracle/gen_scale_fixtures.py

BASELINE.json configs[4] (C5): 6M density-preserving SH-3 Gaussians
(``density_cloud(6_000_000, seed=0)``), 1920x1080, 1024 spp, front camera,
mean depth, cutoff 2*sqrt(2), background 0, seed 0.  The oracle renders a
16x16-strided pixel grid (120 x 68 = 8,160 pixels x 1024 passes) twice:

* ``rng="counter"`` -- the reference algorithm (kernels.py:622-673) with the
  counter draw the GPU reproduces: the converged mean the GPU must match at
  >= 45 dB (same stream, SURVEY.md 8(c) chain step iv);
* ``rng="trig"`` -- bitwise the unmodified reference (tests/test_oracle_golden.py
  pins the oracle's trig mode to splatray's numba kernels): the reference's own
  converged output, reported beside it (an independent stream, so it only
  agrees to the Monte-Carlo noise of 1024 samples).

The walk's result does not depend on the BVH, so the oracle's SAH tree and the
GPU's PLOC tree give the same samples.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[0] = str(ROOT)  # not oracle/ itself: `oracle` must resolve to the package

N, W, H, SPP, STRIDE = 6_000_000, 1920, 1080, 1024, 16
OUT = ROOT / "tests" / "golden" / "c5_converged_grid.npz"


def main() -> None:
    from oracle import oracle as O
    from paper_2504_06598_b200.scene import camera_tuple
    from paper_2504_06598_b200.synthetic import density_cloud, front_camera

    t0 = time.time()
    asset = density_cloud(N, seed=0, sh_degree=3)
    pk = asset.packed
    lo, hi = asset.aabb_arrays(2.0 * np.sqrt(2.0))
    bvh = O.sah_build(lo, hi)
    print(f"scene + SAH build: {time.time() - t0:.1f} s", flush=True)
    ct = np.array(camera_tuple(front_camera(), W, H))
    sub = (slice(None, None, STRIDE), slice(None, None, STRIDE))
    out = {}
    for rng in ("counter", "trig"):
        t0 = time.time()
        r = O.render(bvh, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 3, ct, W, H, passes=SPP, nslots=1, s2=8.0,
                     seed=0, rng=rng, stride=(STRIDE, STRIDE))
        out[f"{rng}_rgb"] = r["rgb"][sub].copy()
        out[f"{rng}_opacity"] = r["opacity"][sub].copy()
        print(f"{rng}: {time.time() - t0:.1f} s", flush=True)
    d = out["counter_rgb"] - out["trig_rgb"]
    mse = float(np.mean(d * d))
    peak = max(1.0, float(out["trig_rgb"].max()))
    print(f"counter vs trig (independent streams) PSNR {10 * np.log10(peak * peak / mse):.2f} dB")
    np.savez_compressed(OUT, n=N, width=W, height=H, spp=SPP, stride=STRIDE, **out)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
