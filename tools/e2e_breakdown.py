"""Where the end-to-end render() time goes at C3-target: wall time of
render() (mapped f64 outputs), of a 16x16 render() (host overhead), and the
device time of the same fused pass writing device memory / mapped host memory.
    python tools/e2e_breakdown.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06598_b200 import RenderSettings, front_camera, render  # noqa: E402
from paper_2504_06598_b200.render import _PINNED, prepare  # noqa: E402
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

W, H = 1920, 1080
a = density_cloud(1_000_000)
st = RenderSettings(width=W, height=H, spp=1)
sc = prepare(a, st)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def wall(f, reps=15):
    f()
    t = []
    for _ in range(reps):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        t.append(time.perf_counter() - t0)
    return statistics.median(t) * 1e3


print(f"render() 1080p mapped f64 out      {wall(lambda: render(a, front_camera(), st)):8.3f} ms")
small = RenderSettings(width=16, height=16, spp=1)
print(f"render() 16x16 (host overhead)     {wall(lambda: render(a, front_camera(), small)):8.3f} ms")
ct = camera_tuple(front_camera(), W, H)
print(f"sc.render pageable f64 out         {wall(lambda: sc.render(ct, W, H, 1, 1, 0, 8.0, True, 0, (0, 0, 0))):8.3f} ms")
rgb, op = _PINNED.array((H, W, 3)), _PINNED.array((H, W))
print(f"sc.render mapped f64 out           "
      f"{wall(lambda: sc.render(ct, W, H, 1, 1, 0, 8.0, True, 0, (0, 0, 0), out_rgb=rgb, out_op=op)):8.3f} ms")
cam = make_camera(ct)
prm = make_render_params(W, H, 1, 1, 0, 8.0)
acc = torch.empty(shard_tiles(W, H) * 256 * 4, device="cuda")
out = torch.empty(W * H * 4, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def dev():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


dev()
ts = []
for _ in range(15):
    flush.fill_(1)
    ts.append(dev())
print(f"fused pass, device float4 out      {statistics.median(ts):8.3f} ms (device time)")

# small frames: where does the fixed cost go
ct16 = camera_tuple(front_camera(), 16, 16)
print(f"sc.render 16x16 pageable           {wall(lambda: sc.render(ct16, 16, 16, 1, 1, 0, 8.0, True, 0, (0, 0, 0))):8.3f} ms")
prm16 = make_render_params(16, 16, 1, 1, 0, 8.0)
cam16 = make_camera(ct16)


def dev16():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sc.render_pass_device(cam16, prm16, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


dev16()
ts = []
for _ in range(15):
    flush.fill_(1)
    ts.append(dev16())
print(f"fused pass 16x16 device             {statistics.median(ts):8.3f} ms (device time)")
ts = []
for _ in range(15):
    ts.append(dev16())
print(f"fused pass 16x16 device, warm L2    {statistics.median(ts):8.3f} ms (device time)")
