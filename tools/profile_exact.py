"""One 1080p exact-compositing frame (render(reference_mode=True)) at
C3-target scale, for an ncu launch list:
    ncu --metrics gpu__time_duration.sum --csv python tools/profile_exact.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_06598_b200 import RenderSettings, front_camera, render  # noqa: E402
from paper_2504_06598_b200.synthetic import density_cloud  # noqa: E402

a = density_cloud(1_000_000)
st = RenderSettings(width=1920, height=1080, spp=1, reference_mode=True)
render(a, front_camera(), st)
render(a, front_camera(), st)
