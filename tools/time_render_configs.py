"""render() wall time (f64 AccumBuffer in host memory) at the multi-pass
BASELINE configs: C2 (100k, 512^2, 16 spp), 1M 1080p 16 spp, C4 (3M, 4K,
4 spp).    python tools/time_render_configs.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_06598_b200 import RenderSettings, front_camera, render  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

for name, n, w, h, spp in [("C2 100k 512x512 16 spp", 100_000, 512, 512, 16),
                           ("1M 1080p 16 spp", 1_000_000, 1920, 1080, 16),
                           ("C4 3M 3840x2160 4 spp", 3_000_000, 3840, 2160, 4)]:
    a = density_cloud(n)
    st = RenderSettings(width=w, height=h, spp=spp)
    render(a, front_camera(), st)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        buf = render(a, front_camera(), st)
        ts.append(time.perf_counter() - t0)
        del buf
    ms = statistics.median(ts) * 1e3
    print(f"render() {name:26s} {ms:8.2f} ms  {w * h * spp / ms / 1e3:7.1f} Mrays/s", flush=True)
