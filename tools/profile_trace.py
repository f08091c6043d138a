"""Minimal ncu driver: the bench's timed call (srt_render_pass_device, fused
walk + SH shade, C3-target 1080p) for a few frames, no oracle, no L2 flush.

    python tools/profile_trace.py [n_prims] [frames] [seed]

Writes gpurun_out/build_id.txt (srt_build_id of the library that ran), which
tools/ncu_summary.py stamps into profiles/ncu_summary.json so bench.py can tell
whether the committed profile belongs to the build it times.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2504_06598_b200 import RenderSettings, _lib, front_camera  # noqa: E402
from paper_2504_06598_b200.render import prepare  # noqa: E402
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
W, H = 1920, 1080
asset = density_cloud(n, seed=seed)
st = RenderSettings(width=W, height=H, spp=1)
sc = prepare(asset, st)
cam = make_camera(camera_tuple(front_camera(), W, H))
prm = make_render_params(W, H, 1, 1, 0, st.cutoff_s ** 2)
acc = torch.empty(shard_tiles(W, H) * 256 * 4, device="cuda")
out = torch.empty(W * H * 4, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for f in range(frames):
    sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
torch.cuda.synchronize()
bid = _lib.load().srt_build_id().decode()
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "build_id.txt").write_text(bid + "\n")
print("ok", bid, sc.bvh_info())
