import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2504_06598_b200 import RenderSettings, front_camera, render
from paper_2504_06598_b200.synthetic import random_cloud
import cProfile, pstats
a = random_cloud(2000, seed=1)
st = RenderSettings(width=16, height=16, spp=1)
cam = front_camera()
for _ in range(20):
    render(a, cam, st)
t = []
for _ in range(200):
    t0 = time.perf_counter(); render(a, cam, st); t.append(time.perf_counter() - t0)
print("render() 16x16 median us", np.median(t) * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    render(a, cam, st)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
