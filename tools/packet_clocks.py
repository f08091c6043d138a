"""Per-packet durations of the C3-target frame kernel and what dispatch
order would do to the frame's tail (experiments build with per-packet
timers):

    bash tools/build_variant.sh clk -DSRT_PACKET_CLOCKS
    SRT_LIBSRT_PATH=build/ab/libsrt_clk.so python tools/packet_clocks.py [seed] [out.npz]

Prints the measured span, the ideal span (total packet time / resident
warps) and list-scheduling makespans of the measured durations under other
dispatch orders (row-major tiles = the kernel's order)."""
import ctypes
import heapq
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06598_b200 import CameraConfig, RenderSettings, _lib, front_camera  # noqa: E402
from paper_2504_06598_b200.render import prepare  # noqa: E402
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
out_npz = sys.argv[2] if len(sys.argv) > 2 else None
W, H = 1920, 1080
st = RenderSettings(width=W, height=H, spp=1)
camera = front_camera()
if os.environ.get("SRT_CAM_SHIFT"):  # translate the camera (and its target) by (dx, dy)
    dx, dy = (float(v) for v in os.environ["SRT_CAM_SHIFT"].split(","))
    camera = CameraConfig(position=camera.position + [dx, dy, 0.0], look_at=camera.look_at + [dx, dy, 0.0],
                          fov_deg=camera.fov_deg)
cam = make_camera(camera_tuple(camera, W, H))
prm = make_render_params(W, H, 1, 1, 0, st.cutoff_s ** 2)
acc = torch.empty(shard_tiles(W, H) * 256 * 4, device="cuda")
out = torch.empty(W * H * 4, device="cuda")
s = torch.cuda.current_stream().cuda_stream
sc = prepare(density_cloud(1_000_000, seed=seed), st)
for _ in range(5):
    sc.render_pass_device(cam, prm, 0, acc.data_ptr(), True, True, out.data_ptr(), s)
torch.cuda.synchronize()
lib = _lib.load()
fn = lib.srt_exp_packet_clocks
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
tiles_x, tiles_y = (W + 15) // 16, (H + 15) // 16
npk = tiles_x * tiles_y * 8
buf = np.zeros(2 * npk, dtype=np.uint64)
assert fn(buf.ctypes.data, npk) == 0
start = buf[0::2].astype(np.int64)
dur = (buf[1::2] & ((1 << 48) - 1)).astype(np.int64)
smid = (buf[1::2] >> 48).astype(np.int64)
ok = dur > 0
t0 = start[ok].min()
span = (start + dur)[ok].max() - t0
warps = 148 * 8 * 4
ideal = dur[ok].sum() / warps
print(f"seed {seed}: packets {ok.sum()} of {npk}; measured span {span / 1e3:.1f} us; "
      f"ideal (sum / {warps} warps) {ideal / 1e3:.1f} us; mean packet {dur[ok].mean() / 1e3:.1f} us, "
      f"max {dur.max() / 1e3:.1f} us")
# activity over time: fraction of warps busy in 20 bins
edges = np.linspace(0, span, 21)
busy = []
for a, b in zip(edges[:-1], edges[1:]):
    s0 = np.clip(start[ok] - t0, a, b)
    s1 = np.clip(start[ok] - t0 + dur[ok], a, b)
    busy.append((s1 - s0).sum() / ((b - a) * warps))
print("busy fraction per 5% of the span:", " ".join(f"{x:.2f}" for x in busy))


def makespan(order):
    h = [0] * warps
    heapq.heapify(h)
    for i in order:
        t = heapq.heappop(h)
        heapq.heappush(h, t + dur[i])
    return max(h)


# packet index p -> (tile, warp-in-tile): tile = p // 8, 16x16 tiles row-major
p = np.arange(npk)
tile = p // 8
w = p % 8
px = (tile % tiles_x) * 16 + (w & 1) * 8 + 4
py = (tile // tiles_x) * 16 + (w >> 1) * 4 + 2
cx, cy = W / 2, H / 2
orders = {
    "row-major (kernel)": p,
    "reversed": p[::-1],
    "centre-out": np.argsort(np.hypot(px - cx, py - cy), kind="stable"),
    "edges-first": np.argsort(-np.hypot(px - cx, py - cy), kind="stable"),
    "LPT (measured durations)": np.argsort(-dur, kind="stable"),
    "random": np.random.default_rng(0).permutation(npk),
}
for name, o in orders.items():
    print(f"  {name:28s} makespan {makespan(o) / 1e3:8.1f} us")
cnt = np.zeros(4 * npk, dtype=np.uint32)
fc = lib.srt_exp_packet_counts
fc.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert fc(cnt.ctypes.data, npk) == 0
visits, jobs, pops, flags = (cnt[k::4].astype(np.int64) for k in range(4))
mixed, lanes_hit = flags & 1, flags >> 1
print(f"mean per packet: visits {visits.mean():.1f} jobs {jobs.mean():.1f} pops {pops.mean():.1f} "
      f"mixed {mixed.mean():.4f} lanes hit {lanes_hit.mean():.1f}")
cc = np.corrcoef(np.stack([dur, visits, jobs, pops]))[0, 1:]
print(f"corr(duration, visits / jobs / pops) = {cc[0]:.3f} / {cc[1]:.3f} / {cc[2]:.3f}")
top = np.argsort(-dur)[:12]
for i in top:
    print(f"  packet {i}: {dur[i] / 1e3:6.1f} us visits {visits[i]} jobs {jobs[i]} pops {pops[i]} "
          f"mixed {mixed[i]} lanes hit {lanes_hit[i]} at block ({px[i] // 8}, {py[i] // 4})")
col = np.bincount(px // 8, weights=visits, minlength=W // 8) / np.maximum(np.bincount(px // 8, minlength=W // 8), 1)
row = np.bincount(py // 4, weights=visits, minlength=H // 4) / np.maximum(np.bincount(py // 4, minlength=H // 4), 1)
print("visits per packet by block column (every 4th):", " ".join(f"{v:.0f}" for v in col[::4]))
print("visits per packet by block row (every 4th):", " ".join(f"{v:.0f}" for v in row[::4]))
if out_npz:
    np.savez_compressed(out_npz, start=start, dur=dur, smid=smid, visits=visits, jobs=jobs, pops=pops, flags=flags)
