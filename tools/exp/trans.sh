python -m pytest tests -m gpu -q -x -k "transmittance or a03" 2>&1 | tail -1
for v in 0 1; do SRT_RAY_SORT=$v python - <<'PY'
import sys, time; sys.path.insert(0, ".")
import numpy as np
from paper_2504_06598_b200 import RenderSettings
from paper_2504_06598_b200.render import prepare
from paper_2504_06598_b200.synthetic import density_cloud
import os
a = density_cloud(1_000_000); st = RenderSettings(width=1920, height=1080, spp=1); sc = prepare(a, st)
rng = np.random.default_rng(0); o = rng.uniform(-2, 2, (1 << 20, 3)); d = rng.normal(size=(1 << 20, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
sc.transmittance(o, d, s2=8.0)
t = []
for _ in range(3):
    t0 = time.perf_counter(); x = sc.transmittance(o, d, s2=8.0); t.append(time.perf_counter() - t0)
print("SRT_RAY_SORT", os.environ["SRT_RAY_SORT"], "transmittance 1M random rays ms", min(t) * 1e3, "mean T", x.mean())
PY
done
