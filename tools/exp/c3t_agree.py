import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2504_06598_b200 import RenderSettings, front_camera, render
from paper_2504_06598_b200.render import prepare
from paper_2504_06598_b200.synthetic import density_cloud
g = np.load("tests/golden/c3target_grid.npz")
a = density_cloud(1_000_000)
st = RenderSettings(width=1920, height=1080, spp=1)
sc = prepare(a, st)
t, ids = sc.trace_rays(g["origins"], g["dirs"], 0.0, float(np.finfo(np.float64).max), 0, 8.0, True, 1, rng="trig64")
agree = ids[:, 0] == g["id"][:, 0]
hit = agree & (g["id"][:, 0] >= 0)
print("trig64 id agreement", agree.mean(), "n", len(agree), "depth bitwise on agreeing hits", np.array_equal(t[hit, 0], g["t"][hit, 0]))
buf = render(a, front_camera(), st, rng="trig64")
got = buf.rgb[g["py"], g["px"]]
ok = np.all(np.abs(got - g["rgb"]) <= 1e-4 * np.abs(g["rgb"]) + 1e-6, axis=1)
print("rgb within 1e-4 rel", ok.mean(), "max abs diff on agreeing", np.abs(got - g["rgb"])[ok].max())
t2, ids2 = sc.trace_rays(g["origins"], g["dirs"], 0.0, float(np.finfo(np.float64).max), 0, 8.0, True, 1)
print("counter-stream hit fraction", (ids2 >= 0).mean(), "vs reference", (g["id"] >= 0).mean())
