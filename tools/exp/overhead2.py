import sys, time, ctypes
sys.path.insert(0, ".")
import numpy as np
from paper_2504_06598_b200 import RenderSettings, front_camera, render
from paper_2504_06598_b200.render import prepare, _PINNED
from paper_2504_06598_b200.scene import camera_tuple
from paper_2504_06598_b200.synthetic import random_cloud

def med(f, n=300):
    for _ in range(20): f()
    t = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); t.append(time.perf_counter() - t0)
    return np.median(t) * 1e6

a = random_cloud(2000, seed=1)
st = RenderSettings(width=16, height=16, spp=1)
cam = front_camera()
sc = prepare(a, st)
ct = camera_tuple(cam, 16, 16)
print("bvh_info us", med(lambda: sc.bvh_info()))
print("camera_tuple us", med(lambda: camera_tuple(cam, 16, 16)))
pr, po = _PINNED.array((16, 16, 3)), _PINNED.array((16, 16))
print("sc.render pinned us", med(lambda: sc.render(ct, 16, 16, 1, 1, 0, 8.0, True, 0, (0, 0, 0), out_rgb=pr, out_op=po)))
print("sc.render pageable us", med(lambda: sc.render(ct, 16, 16, 1, 1, 0, 8.0, True, 0, (0, 0, 0))))
print("render() us", med(lambda: render(a, cam, st)))
import torch
x = torch.zeros(1, device="cuda")
print("torch tiny op + sync us", med(lambda: (x.add_(1), torch.cuda.synchronize())))
