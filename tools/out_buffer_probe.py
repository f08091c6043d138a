import sys, time, statistics
sys.path.insert(0, "/root/repo")
from paper_2504_06598_b200 import RenderSettings, front_camera
from paper_2504_06598_b200.render import prepare, _PINNED
from paper_2504_06598_b200.scene import camera_tuple
from paper_2504_06598_b200.synthetic import density_cloud
a = density_cloud(1_000_000); W, H = 1920, 1080
st = RenderSettings(width=W, height=H, spp=1)
sc = prepare(a, st); ct = camera_tuple(front_camera(), W, H)
def t(f):
    f(); ts = []
    for _ in range(5):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3
print("biased pageable out", t(lambda: sc.render_biased(ct, W, H, 4, 1, 0, st.cutoff_s**2, 0, (0, 0, 0))))
print("biased pinned out  ", t(lambda: sc.render_biased(ct, W, H, 4, 1, 0, st.cutoff_s**2, 0, (0, 0, 0), out_rgb=_PINNED.array((H, W, 3)))))
print("exact pageable out ", t(lambda: sc.render_exact(ct, W, H, 1, 0, st.cutoff_s**2, 0, (0, 0, 0))))
print("exact pinned out   ", t(lambda: sc.render_exact(ct, W, H, 1, 0, st.cutoff_s**2, 0, (0, 0, 0), out_rgb=_PINNED.array((H, W, 3)), out_op=_PINNED.array((H, W)))))
