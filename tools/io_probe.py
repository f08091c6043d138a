import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2504_06598_b200.scene import DeviceScene
from paper_2504_06598_b200.synthetic import random_cloud
a = random_cloud(100, seed=1)
sc = DeviceScene.from_packed(a.packed); sc.build_bvh(2.83)
R = 2073600
rng = np.random.default_rng(0)
o = np.tile([0.0, 0.0, -50.0], (R, 1)); d = rng.normal(size=(R, 3)); d[:, 2] = -abs(d[:, 2]); d /= np.linalg.norm(d, axis=1, keepdims=True)
for name, f in [("trace_rays (no hits, I/O bound)", lambda: sc.trace_rays(o, d)), ("transmittance", lambda: sc.transmittance(o, d))]:
    f(); ts = []
    for _ in range(5):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    print(f"{name}: {np.median(ts)*1e3:.2f} ms for {o.nbytes + d.nbytes} B in", flush=True)
x = np.empty(R * 6); y = np.random.rand(R * 6)
t0 = time.perf_counter(); x[:] = y; t1 = time.perf_counter()
print(f"numpy memcpy 100 MB single thread: {(t1-t0)*1e3:.2f} ms ({y.nbytes/(t1-t0)/1e9:.1f} GB/s)")
