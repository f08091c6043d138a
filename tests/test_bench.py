"""bench.py's multi-rank plumbing on CPU: `bench.py --gpus N` re-launches
itself under torch.distributed.run (no torchrun needed by the caller), every
rank times its share, the max over ranks is reported, and the tile gather +
unpack and the shared host frame assemble every pixel (gloo stands in for
NCCL; a synthetic per-rank shard stands in for the kernel)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("gpus", [2, 3])
def test_bench_self_launches_ranks_gloo(gpus):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(gpus), "--selftest", "gloo",
                        "--steps", "3", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["selftest"] == "ok" and line["n_ranks"] == gpus and line["ms_per_step"] > 0


def test_bench_reference_config_matches_ours():
    """The reference arm reports the same config dict as ours (the driver's
    same_config check)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert b.CONFIG["width"] == 1920 and b.CONFIG["height"] == 1080 and b.CONFIG["n_gaussians"] == 1_000_000
    src = (ROOT / "bench.py").read_text()
    assert src.count('"config": dict(CONFIG)') == 2  # both arms
