"""Wall time of trace_batch through the host C ABI (srt_trace_rays: host f64
rays in, host f64/i64 outputs) vs the device-resident walk, 1080p camera rays
in the 1M cloud: python tools/time_trace_e2e.py [kind] [N] [op]   (kind camera|random, op trace|trans)"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

from paper_2504_06598_b200 import RenderSettings, front_camera
from paper_2504_06598_b200.render import camera_basis, prepare
from paper_2504_06598_b200.synthetic import density_cloud

kind = sys.argv[1] if len(sys.argv) > 1 else "camera"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1
op = sys.argv[3] if len(sys.argv) > 3 else "trace"
st = RenderSettings(width=1920, height=1080, spp=1)
sc = prepare(density_cloud(1_000_000), st)
W, H = 1920, 1080
if kind == "camera":
    cam = front_camera()
    ys, xs = np.mgrid[0:H, 0:W]
    fwd, right, up = camera_basis(cam)
    hh = np.tan(np.radians(cam.fov_deg) / 2)
    u = 2 * (xs.ravel() + 0.5) / W - 1
    v = 1 - 2 * (ys.ravel() + 0.5) / H
    d = fwd[None] + u[:, None] * hh * W / H * right[None] + v[:, None] * hh * up[None]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.tile(np.asarray(cam.position, dtype=np.float64), (d.shape[0], 1))
else:
    rng = np.random.default_rng(0)
    o = rng.uniform(-2, 2, (W * H, 3))
    d = rng.normal(size=(W * H, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
o, d = np.ascontiguousarray(o), np.ascontiguousarray(d)
ts = []
for i in range(8):
    t0 = time.perf_counter()
    if op == "trans":
        t = sc.transmittance(o, d, 0.0, np.finfo(np.float64).max, 0, st.cutoff_s ** 2)
        ids = np.zeros((o.shape[0], 1), np.int64)
    else:
        t, ids = sc.trace_rays(o, d, 0.0, np.finfo(np.float64).max, 0, st.cutoff_s ** 2, True, N, "counter")
    ts.append(time.perf_counter() - t0)
ms = sorted(ts[2:])[len(ts[2:]) // 2] * 1e3
print(f"{op} e2e {kind} N={N}: {ms:.2f} ms  {o.shape[0] / ms / 1e3:.1f} Mrays/s  "
      f"(in {o.nbytes + d.nbytes} B, out {t.nbytes + ids.nbytes} B, hit {float((ids[:, 0] >= 0).mean()):.3f})")
