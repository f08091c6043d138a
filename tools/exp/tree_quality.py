"""Cost metrics of the PLOC binary tree for (seed, radius) pairs, to set
against the frame times of tools/exp/radius_seeds.sh (same deterministic
trees): SAH = sum of inner-node surface areas / root area; SAHz = the same
with the area projected on the image plane (x*y, the front camera looks
along +z) -- what coherent primary rays pay per node."""
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

from paper_2504_06598_b200.scene import DeviceScene
from paper_2504_06598_b200.synthetic import density_cloud

CUT = 2.0 * np.sqrt(2.0)
for seed in (0, 1, 2):
    a = density_cloud(1_000_000, seed=seed)
    sc = DeviceScene.from_packed(a.packed)
    for r in (8, 12, 16, 20, 24, 32):
        os.environ["SRT_PLOC_RADIUS"] = str(r)
        sc.build_bvh(CUT)
        b = sc.download_bvh()
        mi = b["num_inner"]
        e = (b["node_hi"][:mi] - b["node_lo"][:mi]).astype(np.float64)
        sa = e[:, 0] * e[:, 1] + e[:, 1] * e[:, 2] + e[:, 2] * e[:, 0]
        az = e[:, 0] * e[:, 1]
        print(f"seed {seed} radius {r}: SAH {sa.sum() / sa[0]:.2f} SAHz {az.sum() / az[0]:.2f} "
              f"depth {sc.bvh_info()['depth']}", flush=True)
    sc.close()
