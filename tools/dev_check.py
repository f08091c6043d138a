"""Developer check on a GPU box: parity on small scenes + a rough timing of C3-target."""
import sys, time, math
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from oracle import oracle as O
from paper_2504_06598_b200 import RenderSettings, front_camera, random_cloud, density_cloud, two_layer_scene
from paper_2504_06598_b200.render import prepare, render
from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles

def parity(asset, w, h, spp=1, N=1, seed=0, label=""):
    cam = front_camera()
    st = RenderSettings(width=w, height=h, spp=spp, multisample=N, seed=seed)
    t0 = time.time(); sc = prepare(asset, st); t1 = time.time()
    ct = camera_tuple(cam, w, h)
    rgb, op, ids = sc.render(ct, w, h, st.passes, N, 0, st.cutoff_s**2, True, seed, st.background, want_ids=True)
    pk = asset.packed
    lo, hi = asset.aabb_arrays(st.cutoff_s)
    ob = O.sah_build(lo, hi)
    ref = O.render(ob, pk.means, pk.cov_inv6, pk.opacities, pk.sh, pk.sh_degree, np.array(ct), w, h, passes=st.passes,
                   nslots=N, s2=st.cutoff_s**2, seed=seed, rng="counter", want_ids=True)
    agree = np.mean(ids == ref["ids"])
    same = np.all(ids == ref["ids"], axis=2)
    rel = np.abs(rgb - ref["rgb"]) / np.maximum(np.abs(ref["rgb"]), 1e-6)
    print(f"{label}: n={len(asset)} {w}x{h} N={N} build {t1-t0:.3f}s info {sc.bvh_info()} agree {agree:.6f} "
          f"hit {np.mean(ids>=0):.3f} max rel colour err (agreeing) {rel[same].max() if st.passes==1 else float('nan'):.2e}")
    return sc

parity(two_layer_scene(), 16, 16, label="two-layer")
parity(random_cloud(10_000, seed=0, sh_degree=0), 64, 64, label="C1")
parity(random_cloud(10_000, seed=0, sh_degree=3), 64, 64, N=4, label="C1 N4")
parity(density_cloud(100_000), 128, 128, label="C2-ish")

# timing C3-target
asset = density_cloud(1_000_000)
st = RenderSettings(width=1920, height=1080, spp=1)
t0 = time.time(); sc = prepare(asset, st); torch.cuda.synchronize(); print("prepare 1M", time.time()-t0, sc.bvh_info())
t0 = time.time(); sc.build_bvh(st.cutoff_s); print("lbvh 1M", time.time()-t0)
cam = make_camera(camera_tuple(front_camera(), 1920, 1080))
prm = make_render_params(1920, 1080, 1, 1, 0, st.cutoff_s**2)
tiles = shard_tiles(1920, 1080)
hits = torch.empty(tiles*256, dtype=torch.int32, device="cuda")
acc = torch.empty(tiles*256*4, dtype=torch.float32, device="cuda")
out = torch.empty(1920*1080*4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    sc.render_device(cam, prm, hits.data_ptr(), acc.data_ptr(), out.data_ptr(), s)
torch.cuda.synchronize()
e0, e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(5):
    e0.record(); sc.trace_pass_device(cam, prm, 0, hits.data_ptr(), s); e1.record()
    sc.shade_pass_device(cam, prm, 0, hits.data_ptr(), acc.data_ptr(), True, True, out.data_ptr(), s); e2.record()
    torch.cuda.synchronize()
    tt, ts = e0.elapsed_time(e1), e1.elapsed_time(e2)
    print(f"C3-target trace {tt:.3f} ms shade {ts:.3f} ms -> {1920*1080/((tt+ts)*1e-3)/1e6:.1f} Mrays/s")
# parity sample at 1M: oracle on strided pixels
ct = camera_tuple(front_camera(), 1920, 1080)
rgb, op, ids = sc.render(ct, 1920, 1080, 1, 1, 0, st.cutoff_s**2, True, 0, st.background, want_ids=True)
pk = asset.packed
lo, hi = asset.aabb_arrays(st.cutoff_s)
t0=time.time(); ob = O.sah_build(lo, hi); print("oracle sah 1M", time.time()-t0)
t0=time.time()
ref = O.render(ob, pk.means, pk.cov_inv6, pk.opacities, pk.sh, 3, np.array(ct), 1920, 1080, rng="counter", stride=(8,8), want_ids=True, counters=True)
print("oracle strided render", time.time()-t0, ref["counters"])
m = ref["ids"][::8, ::8, 0]
g = ids[::8, ::8, 0]
print("1M agree", np.mean(m == g), "n", m.size, "hit", np.mean(g >= 0))
