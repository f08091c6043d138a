import sys, faulthandler
faulthandler.enable()
sys.path.insert(0, "/root/repo")
print("start", flush=True)
import numpy as np
from paper_2504_06598_b200.scene import DeviceScene
from paper_2504_06598_b200.synthetic import random_cloud
a = random_cloud(2000, seed=1)
print("asset", flush=True)
sc = DeviceScene.from_packed(a.packed)
print("scene", flush=True)
sc.build_bvh(2.8284271247461903)
print("bvh", sc.bvh_info(), flush=True)
t, ids = sc.trace_rays([[0,0,-5]], [[0,0,1]])
print("trace", t, ids, flush=True)
