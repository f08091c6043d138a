"""Wall time of the secondary paths at C3-target scale (1M SH-3, 1080p):
exact compositing (reference_mode), the biased k=4 frame, the trig64 bridge
frame, transmittance and explicit-ray walks.  python tools/time_paths.py"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

from paper_2504_06598_b200 import RenderSettings, front_camera, render, render_biased
from paper_2504_06598_b200.render import prepare
from paper_2504_06598_b200.synthetic import density_cloud

a = density_cloud(1_000_000)
cam = front_camera()
W, H = 1920, 1080
st = RenderSettings(width=W, height=H, spp=1)
sc = prepare(a, st)


def timed(name, f, rays, reps=3):
    f()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        t.append(time.perf_counter() - t0)
    ms = float(np.median(t)) * 1e3
    print(f"{name:42s} {ms:9.2f} ms  {rays / ms / 1e3:8.1f} Mrays/s")


timed("render() stochastic 1 spp", lambda: render(a, cam, st), W * H)
timed("render() reference_mode (exact) 1 spp", lambda: render(a, cam, RenderSettings(width=W, height=H, spp=1,
                                                                                     reference_mode=True)), W * H)
timed("render_biased k=4 (counter)", lambda: render_biased(a, cam, st, 4), W * H)
timed("render() rng=trig64 1 spp", lambda: render(a, cam, st, rng="trig64"), W * H)
timed("render() 16 spp, one launch", lambda: render(a, cam, RenderSettings(width=W, height=H, spp=16)), W * H * 16)
rng = np.random.default_rng(0)
o = rng.uniform(-2, 2, (1 << 20, 3))
d = rng.normal(size=(1 << 20, 3))
d /= np.linalg.norm(d, axis=1, keepdims=True)
timed("transmittance, 1M random rays (host I/O)", lambda: sc.transmittance(o, d, s2=st.cutoff_s ** 2), 1 << 20)
timed("trace_rays N=1, 1M random rays (host I/O)", lambda: sc.trace_rays(o, d, s2=st.cutoff_s ** 2), 1 << 20)
