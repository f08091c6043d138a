import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2504_06598_b200 import RenderSettings, front_camera, render
from paper_2504_06598_b200.synthetic import density_cloud
a = density_cloud(1_000_000)
st = RenderSettings(width=1920, height=1080, spp=1, reference_mode=True)
render(a, front_camera(), st)
for _ in range(3):
    t0 = time.perf_counter(); b = render(a, front_camera(), st); t = time.perf_counter() - t0
    print(f"reference_mode 1080p 1M: {t*1e3:.1f} ms  mean op {b.opacity.mean():.4f}", flush=True)
