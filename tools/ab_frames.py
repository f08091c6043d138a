"""Device-timed C3-target frames (fused walk + shade, srt_render_pass_device,
L2 flushed between frames) on several scene seeds, for A/B of builds:

    SRT_LIBSRT_PATH=build/ab/libsrt_X.so python tools/ab_frames.py [reps] [seed ...]

Prints one line per seed (median / min ms) and the mean over seeds.
SRT_TRACE_STATS=1 adds the per-walk traversal counters.
"""
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2504_06598_b200 import RenderSettings, _lib, front_camera  # noqa: E402
from paper_2504_06598_b200.render import prepare  # noqa: E402
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
seeds = [int(x) for x in sys.argv[2:]] or [0, 1, 2]
n = int(os.environ.get("SRT_N", "1000000"))
W, H = int(os.environ.get("SRT_W", "1920")), int(os.environ.get("SRT_H", "1080"))
st = RenderSettings(width=W, height=H, spp=1)
cam = make_camera(camera_tuple(front_camera(), W, H))
prm = make_render_params(W, H, 1, 1, 0, st.cutoff_s ** 2)
acc = torch.empty(shard_tiles(W, H) * 256 * 4, device="cuda")
out = torch.empty(W * H * 4, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
lib = os.environ.get("SRT_LIBSRT_PATH", "libsrt.so").split("/")[-1]
means = []
for seed in seeds:
    sc = prepare(density_cloud(n, seed=seed), st)
    if hasattr(sc, "split_info"):
        print(f"seed {seed}: split tree {sc.split_info()}", flush=True)
    for _ in range(3):
        sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
    if os.environ.get("SRT_TRACE_STATS") == "1":
        sc.trace_stats(reset=True)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    sc.check_status()
    med = statistics.median(ts)
    means.append(med)
    extra = ""
    if os.environ.get("SRT_TRACE_STATS") == "1":
        d = sc.trace_stats()
        w = max(d["walks"], 1)
        extra = " " + str({k: round(v / w, 2) for k, v in d.items()})
    print(f"{lib} seed {seed}: median {med:.3f} ms min {min(ts):.3f} ms ({W * H / med / 1e3:.0f} Mrays/s){extra}",
          flush=True)
    sc.close()
print(f"{lib} mean over seeds {seeds}: {statistics.mean(means):.3f} ms "
      f"({W * H / statistics.mean(means) / 1e3:.0f} Mrays/s)")
