"""Tree-quality probe: front-camera C3-target frame time and a view-independent
probe (14 views -- 6 axis + 8 diagonal cameras around the scene, 480x270,
1 spp) for the current build (SRT_PLOC_RADIUS selects the PLOC radius in
the experiments build):
    make -C paper_2504_06598_b200/csrc experiments
    SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so SRT_PLOC_RADIUS=r python tools/tree_probe.py seed"""
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06598_b200 import CameraConfig, RenderSettings, front_camera  # noqa: E402
from paper_2504_06598_b200.render import prepare  # noqa: E402
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sc = prepare(density_cloud(1_000_000, seed=seed), RenderSettings(width=1920, height=1080, spp=1))
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def frame_ms(camera, W, H, reps):
    cam = make_camera(camera_tuple(camera, W, H))
    prm = make_render_params(W, H, 1, 1, 0, 8.0)
    acc = torch.empty(shard_tiles(W, H) * 256 * 4, device="cuda")
    out = torch.empty(W * H * 4, device="cuda")
    for _ in range(2):
        sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


front = frame_ms(front_camera(), 1920, 1080, 15)
views = [np.array(v, float) for v in [(6, 0, 0), (-6, 0, 0), (0, 6, 0.01), (0, -6, 0.01), (0, 0, 6), (0, 0, -6)]]
views += [np.array(v, float) * 6 / np.sqrt(3) for v in [(sx, sy, sz) for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]]
probe = sum(frame_ms(CameraConfig(position=v, fov_deg=45.0), 480, 270, 5) for v in views)
print(f"seed {seed} radius {os.environ.get('SRT_PLOC_RADIUS', 'default')}: front {front:.3f} ms, probe {probe:.3f} ms, "
      f"bvh {sc.bvh_info()}", flush=True)
