"""The N > 1 path of bench.py run end to end on a one-GPU box: two ranks
both on cuda:0 (SRT_BENCH_SAME_GPU=1: gloo, host-side frame barrier) go
through the self-launch, the IPC peer frame (each rank's fused kernel stores
its tiles into rank 0's frame), per-rank timing and max over ranks, and the
multi-GPU e2e leg (render_distributed into the shared mapped host frame).
A functional check only: ranks share one GPU, so the timings mean nothing
(the line is marked functional_check_only)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, SRT_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = lines[0]
    assert line["n_gpus"] == 2 and "functional_check_only" in line
    assert "peer stores" in line["parallelism"], line["parallelism"]
    assert len(line["ranks"]) == 2 and all(x["walk_ms"] > 0 for x in line["ranks"])
    assert sum(x["tiles"] for x in line["ranks"]) == 8160  # every 16x16 tile of 1080p exactly once
    assert line["e2e"]["value"] > 0 and line["e2e"]["d2h_bytes_per_step"] == 1920 * 1080 * 32
