"""Time k_trace + k_shade for a config: python tools/time_frames.py [n] [W] [H] [spp] [N] [reps]"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2504_06598_b200 import RenderSettings, front_camera
from paper_2504_06598_b200.render import prepare
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles
from paper_2504_06598_b200.synthetic import density_cloud, random_cloud

a = sys.argv[1:]
n = int(a[0]) if a else 1_000_000
W = int(a[1]) if len(a) > 1 else 1920
H = int(a[2]) if len(a) > 2 else 1080
spp = int(a[3]) if len(a) > 3 else 1
N = int(a[4]) if len(a) > 4 else 1
reps = int(a[5]) if len(a) > 5 else 10
_seed = int(__import__("os").environ.get("SRT_SEED", "0"))  # scene seed (sweeps over scenes)
asset = density_cloud(n, seed=_seed) if n > 10_000 else random_cloud(n, seed=_seed, sh_degree=0)
st = RenderSettings(width=W, height=H, spp=spp, multisample=N)
sc = prepare(asset, st)
import os
if os.environ.get("SRT_BVH_METHOD"):
    sc.build_bvh(st.cutoff_s, method=os.environ["SRT_BVH_METHOD"])
if os.environ.get("SRT_SAH") == "1":
    from oracle import oracle as O
    lo, hi = asset.aabb_arrays(st.cutoff_s)
    if os.environ.get("SRT_SAH_TIGHT") == "1":  # ellipsoid AABBs, as the LBVH uses
        import numpy as np
        half = st.cutoff_s * np.sqrt(np.einsum("nii->ni", np.linalg.inv(asset.packed.cov_inv)))
        lo, hi = asset.means - half, asset.means + half
    import time as _t
    _t0 = _t.time()
    ob = O.sah_build(lo, hi, leaf_size=int(os.environ.get("SRT_SAH_LEAF", "1")))
    print("host SAH build", _t.time() - _t0)
    sc.upload_bvh(ob)
cam = make_camera(camera_tuple(front_camera(), W, H))
prm = make_render_params(W, H, st.passes, N, 0, st.cutoff_s ** 2)
t = shard_tiles(W, H)
hits = torch.empty(t * 256 * N, dtype=torch.int32, device="cuda")
acc = torch.empty(t * 256 * 4, device="cuda")
out = torch.empty(W * H * 4, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    sc.render_device(cam, prm, hits.data_ptr(), acc.data_ptr(), out.data_ptr(), s)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tt, ts = [], []
fused = os.environ.get("SRT_SPLIT") != "1"
onelaunch = os.environ.get("SRT_ONE_LAUNCH") == "1"
acc64 = torch.empty(t * 256 * 4, dtype=torch.int64, device="cuda") if onelaunch else None
for _ in range(reps):
    flush.fill_(1)
    ev[0].record()
    if onelaunch:
        sc.render_frame_device(cam, prm, acc64.data_ptr(), out.data_ptr(), s)
        ev[1].record()
    elif fused:
        for f in range(st.passes):
            sc.render_pass_device(cam, prm, f, acc.data_ptr(), f == 0, f == st.passes - 1, out.data_ptr(), s)
        ev[1].record()
    else:
        for f in range(st.passes):
            sc.trace_pass_device(cam, prm, f, hits.data_ptr(), s)
        ev[1].record()
        sc.shade_pass_device(cam, prm, 0, hits.data_ptr(), acc.data_ptr(), True, True, out.data_ptr(), s)
    ev[2].record()
    torch.cuda.synchronize()
    tt.append(ev[0].elapsed_time(ev[1]))
    ts.append(ev[1].elapsed_time(ev[2]))
tt.sort(); ts.sort()
if os.environ.get("SRT_TRACE_STATS") == "1":
    d = sc.trace_stats()
    w = max(d["walks"], 1)
    print("per walk:", {k: round(v / w, 2) for k, v in d.items()})
walks = W * H * st.passes
import time as _tt
_t0 = _tt.time(); sc.build_bvh(st.cutoff_s, method=os.environ.get("SRT_BVH_METHOD", "ploc")); _bt = _tt.time() - _t0
print(f"build {_bt*1e3:.1f} ms", end="  ")
print(f"n={n} {W}x{H} spp={spp} N={N}: trace {tt[len(tt)//2]:.3f} ms ({walks/tt[len(tt)//2]/1e3:.1f} Mwalks/s, "
      f"{walks*N/tt[len(tt)//2]/1e3:.1f} Msamples/s) shade {ts[len(ts)//2]:.3f} ms  bvh {sc.bvh_info()}")
