"""Throughput of explicit-ray walks (trace_batch semantics, srt_trace_rays_device)
on device-resident rays: python tools/time_rays.py [n_prims] [n_rays] [kind] [N]
kind: "random" (origins in the cloud, isotropic directions: incoherent
secondary rays), "camera" (the C3-target primary rays, row-major) or
"parallel" (validate.py:36-43-style jittered origins on z = -6, all along +z).
SRT_PACKET_RAYS=0/1 pins the route (default: packets for one-hemisphere batches)."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch

from paper_2504_06598_b200 import RenderSettings, front_camera
from paper_2504_06598_b200.render import generate_camera_ray, prepare
from paper_2504_06598_b200.synthetic import density_cloud

a = sys.argv[1:]
n = int(a[0]) if a else 1_000_000
R = int(a[1]) if len(a) > 1 else 1 << 21
kind = a[2] if len(a) > 2 else "random"
N = int(a[3]) if len(a) > 3 else 1
asset = density_cloud(n)
st = RenderSettings(width=1920, height=1080, spp=1)
sc = prepare(asset, st)
rng = np.random.default_rng(0)
if kind == "random":
    o = rng.uniform(-2, 2, (R, 3))
    d = rng.normal(size=(R, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
elif kind == "parallel":
    o = np.stack([rng.uniform(-2, 2, R), rng.uniform(-2, 2, R), np.full(R, -6.0)], axis=1)
    d = np.tile([0.0, 0.0, 1.0], (R, 1))
else:
    W, H = 1920, 1080
    cam = front_camera()
    # same directions as the camera pass 0, row-major (vectorised pinhole, no jitter)
    ys, xs = np.mgrid[0:H, 0:W]
    from paper_2504_06598_b200.render import camera_basis
    fwd, right, up = camera_basis(cam)
    hh = np.tan(np.radians(cam.fov_deg) / 2)
    hw = hh * W / H
    u = 2 * (xs.ravel() + 0.5) / W - 1
    v = 1 - 2 * (ys.ravel() + 0.5) / H
    d = fwd[None] + u[:, None] * hw * right[None] + v[:, None] * hh * up[None]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.tile(cam.position, (d.shape[0], 1))
    R = d.shape[0]
rays = torch.from_numpy(np.concatenate([o, d], axis=1)).cuda()
t = torch.empty((R, N), dtype=torch.float32, device="cuda")
ids = torch.empty((R, N), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    sc.trace_rays_device(rays.data_ptr(), R, N, t.data_ptr(), ids.data_ptr(), s, s2=st.cutoff_s ** 2)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.fill_(1)
    ev[0].record()
    sc.trace_rays_device(rays.data_ptr(), R, N, t.data_ptr(), ids.data_ptr(), s, s2=st.cutoff_s ** 2)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ts.sort()
ms = ts[len(ts) // 2]
hit = float((ids[:, 0] >= 0).float().mean())
print(f"{kind} rays n={n} R={R} N={N}: {ms:.3f} ms  {R / ms / 1e3:.1f} Mrays/s  hit fraction {hit:.3f}")
