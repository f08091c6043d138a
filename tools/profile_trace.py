"""Minimal driver for ncu: C3-target scene, a few trace+shade passes (no oracle)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2504_06598_b200 import RenderSettings, front_camera
from paper_2504_06598_b200.render import prepare
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles
from paper_2504_06598_b200.synthetic import density_cloud

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
W, H = 1920, 1080
asset = density_cloud(n)
st = RenderSettings(width=W, height=H, spp=1)
sc = prepare(asset, st)
cam = make_camera(camera_tuple(front_camera(), W, H))
prm = make_render_params(W, H, 1, 1, 0, st.cutoff_s ** 2)
t = shard_tiles(W, H)
hits = torch.empty(t * 256, dtype=torch.int32, device="cuda")
acc = torch.empty(t * 256 * 4, device="cuda")
out = torch.empty(W * H * 4, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for f in range(frames):
    sc.render_device(cam, prm, hits.data_ptr(), acc.data_ptr(), out.data_ptr(), s)
torch.cuda.synchronize()
print("ok", sc.bvh_info())
