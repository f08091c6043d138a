"""Per-rank walk time of tile-sharded C3-target frames, measured on one GPU:
rank r of G renders the 16x16 tiles t with t % G == r (srt_render_pass_device
with shard_index / shard_count), exactly the work of one rank of a G-GPU
frame.  The slowest rank bounds the G-GPU frame; ideal = 1-GPU time / G.
    python tools/shard_times.py [seed] [n] [W] [H]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2504_06598_b200 import RenderSettings, front_camera  # noqa: E402
from paper_2504_06598_b200.render import prepare  # noqa: E402
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
W = int(sys.argv[3]) if len(sys.argv) > 3 else 1920
H = int(sys.argv[4]) if len(sys.argv) > 4 else 1080
sc = prepare(density_cloud(n, seed=seed), RenderSettings(width=W, height=H, spp=1))
cam = make_camera(camera_tuple(front_camera(), W, H))
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
acc = torch.empty(shard_tiles(W, H) * 256 * 4, device="cuda")
out = torch.empty(W * H * 4, device="cuda")


def ms(prm, reps=15):
    for _ in range(3):
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


one = ms(make_render_params(W, H, 1, 1, 0, 8.0))
print(f"seed {seed}, {n} Gaussians, {W}x{H}: 1 GPU {one:.3f} ms")
for G in (2, 4, 8):
    per = [ms(make_render_params(W, H, 1, 1, 0, 8.0, shard_index=r, shard_count=G)) for r in range(G)]
    worst = max(per)
    print(f"  G={G}: per-rank {' '.join(f'{x:.3f}' for x in per)} ms; slowest {worst:.3f} ms, ideal {one / G:.3f} ms, "
          f"scaling bound {one / worst:.2f}x", flush=True)
