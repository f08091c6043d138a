"""Benchmark: Mrays/s and ms/frame of 1-spp camera rays through a 1M-Gaussian
SH-3 cloud at 1920x1080 (BASELINE.json metric; workload "C3-target",
BASELINE.md section 3), on N B200s, beside the reference CPU renderer.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun (one rank per GPU, NCCL): each rank traces the
16x16 tiles t with t % N == rank, and the tile-compact shards are gathered to
rank 0 with one NCCL gather per frame and unpacked there.

One JSON line on rank 0.  "value" = whole-job Mrays/s with the scene resident
in HBM, timed on the device with CUDA events (max over ranks).  "e2e" = the
same metric through the public render() API (libsrt host-pointer entry
point) with the fp64 AccumBuffer copied back to the host every step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WIDTH, HEIGHT, N_PRIMS, SH_DEG, SPP, NSLOTS = 1920, 1080, 1_000_000, 3, 1, 1
WORKLOAD = "C3-target: density_cloud(1M, SH3, seed 0), 1920x1080, 1 spp, N=1, front_camera, mean depth"
# Algorithmic bytes per walk: B = 64 I + 24 P + 48 C + S hits + 16/passes with the
# per-walk counts of the reference SAH BVH on this scene:
# I = 150.5, P = 167.3, C = 82.4, hits = 0.68, S = 192 B (SH degree 3).
YARD_I, YARD_P, YARD_C, YARD_HITS, SH_BYTES = 150.5, 167.3, 82.4, 0.68, 192
BYTES_PER_WALK = 64 * YARD_I + 24 * YARD_P + 48 * YARD_C + SH_BYTES * YARD_HITS + 16 / SPP
L2_FLUSH_BYTES = 256 << 20
PROFILE_SUMMARY = ROOT / "profiles" / "ncu_summary.json"


def _peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
        except Exception:
            pass
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def _traffic_per_launch():
    if PROFILE_SUMMARY.exists():
        try:
            d = json.loads(PROFILE_SUMMARY.read_text())
            return d.get("trace_dram_bytes_per_launch")
        except Exception:
            return None
    return None


def _issue_roofline(kernel_ms: float, clocks):
    """Issue-slot roofline of the dominant kernel: the walk is bound by SM
    instruction issue, not bytes.  achieved = warp instructions
    per launch (ncu, profiles/ncu_summary.json) / the live kernel time; peak =
    1 warp instruction per cycle per SM sub-partition (148 SMs x 4) at the SM
    clock sampled during the timed region."""
    try:
        d = json.loads(PROFILE_SUMMARY.read_text())
        inst = float(d["warp_inst_per_launch"])
    except Exception:
        return None
    import torch

    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    peak = sms * 4 * mhz * 1e6 / 1e9  # G warp-instructions / s
    achieved = inst / (kernel_ms * 1e-3) / 1e9
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "G warp-inst/s", "frac": achieved / peak,
            "warp_inst_per_launch": inst, "ncu_issue_active_pct": d.get("issue_active_pct"),
            "source": "warp instructions from profiles/ncu_summary.json, kernel time live"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"srt_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 5.0:  # wait for the first sample so the timed region is covered
                if self.path.exists() and self.path.stat().st_size > 0:
                    break
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        try:
            rows = [r.split(",") for r in self.path.read_text().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].strip().lower() == "active"})
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


_CPU_BVH = {}


def _cpu_baseline_sample(asset, threads: int, stride=(2, 2)) -> dict:
    """The reference algorithm (oracle C restatement, trig hash: bitwise equal to
    splatray.kernels.render_stochastic) on host cores, over every stride-th
    pixel of the same frame, prebuilt SAH BVH; returns rays, seconds."""
    from oracle import oracle as O
    from paper_2504_06598_b200.synthetic import front_camera
    from paper_2504_06598_b200.scene import camera_tuple

    O.build()
    pk = asset.packed
    if id(asset) not in _CPU_BVH:
        lo, hi = asset.aabb_arrays(2.0 * np.sqrt(2.0))
        t0 = time.perf_counter()
        _CPU_BVH[id(asset)] = (O.sah_build(lo, hi), time.perf_counter() - t0)
    b, build_s = _CPU_BVH[id(asset)]
    ct = np.array(camera_tuple(front_camera(), WIDTH, HEIGHT))
    t0 = time.perf_counter()
    O.render(b, pk.means, pk.cov_inv6, pk.opacities, pk.sh, SH_DEG, ct, WIDTH, HEIGHT, passes=SPP, nslots=NSLOTS,
             s2=8.0, seed=0, rng="trig", stride=stride, threads=threads)
    secs = time.perf_counter() - t0
    rays = len(range(0, WIDTH, stride[0])) * len(range(0, HEIGHT, stride[1])) * SPP
    return {"rays": rays, "seconds": secs, "bvh_build_s": build_s}


def run_reference(args) -> None:
    """--impl reference: the reference's CPU renderer on the box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2504_06598_b200.synthetic import density_cloud

    threads = os.cpu_count() or 1
    asset = density_cloud(N_PRIMS, seed=0, sh_degree=SH_DEG)
    stride = (4, 4)
    for _ in range(args.warmup):
        _cpu_baseline_sample(asset, threads, stride)
    times = []
    for _ in range(args.steps):
        r = _cpu_baseline_sample(asset, threads, stride)
        times.append(r["seconds"])
    rays = r["rays"]
    mrays = rays / statistics.mean(times) / 1e6
    frame_ms = WIDTH * HEIGHT * SPP / (mrays * 1e6) * 1e3
    sample = f"every 4th pixel in x and y of the 1920x1080 frame ({rays} rays/step), prebuilt SAH BVH"
    line = {
        "impl": "reference", "metric": "Mrays/s", "value": mrays, "unit": "Mrays/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": frame_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "width": WIDTH, "height": HEIGHT, "n_gaussians": N_PRIMS, "spp": SPP,
                   "sh_degree": SH_DEG, "ms_per_step_is": "extrapolated full-frame ms"},
        "cpu_baseline": {"value": mrays, "unit": "Mrays/s", "cores": threads, "kind": "port", "sample": sample,
                         "note": "oracle/srt_oracle.c in trig-hash mode, bitwise equal to the reference's numba "
                                 "render_stochastic (tests/test_oracle_golden.py); OpenMP over 16x16 tiles"},
        "e2e": {"value": mrays, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2504_06598_b200 import RenderSettings, front_camera, render
    from paper_2504_06598_b200.render import prepare
    from paper_2504_06598_b200.scene import camera_tuple, make_camera, make_render_params, shard_tiles, \
        unpack_tiles_device
    from paper_2504_06598_b200.synthetic import density_cloud

    asset = density_cloud(N_PRIMS, seed=0, sh_degree=SH_DEG)
    st = RenderSettings(width=WIDTH, height=HEIGHT, spp=SPP, multisample=NSLOTS)
    t0 = time.perf_counter()
    sc = prepare(asset, st, device=local)
    setup_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    sc.build_bvh(st.cutoff_s)
    lbvh_s = time.perf_counter() - t0
    cam = make_camera(camera_tuple(front_camera(), WIDTH, HEIGHT))
    prm = make_render_params(WIDTH, HEIGHT, st.passes, NSLOTS, 0, st.cutoff_s ** 2, shard_index=rank,
                             shard_count=world)
    dev = torch.device("cuda", local)
    tiles = shard_tiles(WIDTH, HEIGHT, rank, world)
    max_tiles = shard_tiles(WIDTH, HEIGHT, 0, world)
    hits = torch.empty(max_tiles * 256 * NSLOTS, dtype=torch.int32, device=dev)
    acc = torch.empty(max_tiles * 256 * 4, dtype=torch.float32, device=dev)
    out = torch.zeros(max_tiles * 256 * 4, dtype=torch.float32, device=dev)
    frame = torch.zeros(WIDTH * HEIGHT * 4, dtype=torch.float32, device=dev) if (world > 1 and rank == 0) else None
    gathered = [torch.empty_like(out) for _ in range(world)] if (world > 1 and rank == 0) else None
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        for f in range(st.passes):
            # one fused kernel per pass: packet walk + SH shade + accumulate
            sc.render_pass_device(cam, prm, f, acc.data_ptr(), f == 0, f == st.passes - 1, out.data_ptr(), sp)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:
            dist.gather(out, gathered if rank == 0 else None, dst=0)
            if rank == 0:
                packed = torch.cat(gathered)
                unpack_tiles_device(packed.data_ptr(), WIDTH, HEIGHT, world, max_tiles, frame.data_ptr(), sp)
        if ev is not None:
            ev[2].record(stream)

    events = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(max(args.warmup, 0)):
            step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # evict the scene from L2 between steps (outside the step events)
            step(events[i])
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - wall0
        time.sleep(0.25)  # let the sampler record the tail of the timed region
    if world > 1:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[2]) for e in events]
    trace_ms = [e[0].elapsed_time(e[1]) for e in events]
    local_ms = float(sum(step_ms))
    if world > 1:
        tt = torch.tensor([local_ms, float(sum(trace_ms))], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, trace_total = tt.tolist()
    else:
        total_ms, trace_total = local_ms, float(sum(trace_ms))
    ms_per_step = total_ms / args.steps
    rays_per_frame = WIDTH * HEIGHT * SPP
    value = rays_per_frame / (ms_per_step * 1e-3) / 1e6

    # roofline of the dominant kernel (k_trace_pass) on rank 0's stream
    trace_avg_ms = trace_total / (args.steps * st.passes)
    walks_per_launch = tiles * 256 if world > 1 else rays_per_frame / SPP
    walks_per_launch = min(walks_per_launch, WIDTH * HEIGHT)
    alg_bytes = BYTES_PER_WALK * walks_per_launch
    achieved = alg_bytes / (trace_avg_ms * 1e-3) / 1e9
    peak, peak_src = _peaks()

    # e2e: the public API with host buffers.  N > 1: render_distributed on
    # every rank (tile shards, one NCCL gather, f64 frame on rank 0's host),
    # wall clock on rank 0 between barriers
    e2e = None
    if world > 1:
        from paper_2504_06598_b200.multi_gpu import render_distributed

        render_distributed(asset, front_camera(), st, mode="tiles", device=local)  # warm
        e2e_t = []
        buf = None
        for _ in range(max(3, min(args.steps, 10))):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            dist.barrier()
            t0 = time.perf_counter()
            out_buf = render_distributed(asset, front_camera(), st, mode="tiles", device=local)
            dist.barrier()
            e2e_t.append(time.perf_counter() - t0)
            buf = out_buf if rank == 0 else buf
        if rank == 0:
            e2e = {"value": rays_per_frame / statistics.median(e2e_t) / 1e6, "unit": "Mrays/s",
                   "h2d_bytes_per_step": 192 * world, "d2h_bytes_per_step": int(buf.rgb.nbytes + buf.opacity.nbytes),
                   "ms_per_frame": statistics.median(e2e_t) * 1e3,
                   "path": "paper_2504_06598_b200.multi_gpu.render_distributed() on every rank: tile shards traced "
                           "and shaded per GPU, one NCCL gather to rank 0, unpacked on its GPU, f64 AccumBuffer "
                           "copied to rank 0's host; wall clock on rank 0 between barriers"}
    elif rank == 0:
        render(asset, front_camera(), st, device=local)  # warm (allocates scratch)
        e2e_t = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            buf = render(asset, front_camera(), st, device=local)
            e2e_t.append(time.perf_counter() - t0)
        e2e = {"value": rays_per_frame / statistics.median(e2e_t) / 1e6, "unit": "Mrays/s",
               "h2d_bytes_per_step": 192, "d2h_bytes_per_step": int(buf.rgb.nbytes + buf.opacity.nbytes),
               "ms_per_frame": statistics.median(e2e_t) * 1e3,
               "path": "paper_2504_06598_b200.render() -> srt_render (C ABI): fused trace+shade on the GPU; the last "
                       "pass stores the AccumBuffer (H,W,3)+(H,W) float64 straight into pooled mapped page-locked host "
                       "memory (device->host over PCIe during the walk), stream synchronised before render() returns; "
                       "h2d = camera + settings kernel parameters (SrtCamera 112 B + SrtRenderParams 80 B), scene resident"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        r = _cpu_baseline_sample(asset, threads)
        cpu = {"value": r["rays"] / r["seconds"] / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "port",
               "sample": f"every 2nd pixel in x and y of the same 1080p frame ({r['rays']} rays), trig-hash "
                         f"restatement bitwise equal to the reference, prebuilt SAH BVH "
                         f"({r['bvh_build_s']:.2f} s C build)"}

    if rank == 0:
        clocks = sampler.summary()
        line = {
            "metric": "Mrays/s", "value": value, "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "width": WIDTH, "height": HEIGHT, "n_gaussians": N_PRIMS,
                       "spp": SPP, "nslots": NSLOTS, "sh_degree": SH_DEG,
                       "parallelism": f"tile-shard x{world}" + (" + NCCL gather" if world > 1 else ""),
                       "l2": "256 MiB flush written between steps, outside the per-step CUDA events",
                       "scene_setup_s": setup_s, "lbvh_build_s": lbvh_s, "bvh": sc.bvh_info(),
                       "ms_per_frame": ms_per_step, "wall_s_timed_region": wall},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic_per_launch(),
                         "kernel": "k_trace_packet (fused walk + SH shade + accumulate)", "kernel_ms": trace_avg_ms,
                         "algorithmic_bytes_per_walk": BYTES_PER_WALK, "walks_per_launch": walks_per_launch,
                         "peak_source": peak_src},
            "roofline_issue": _issue_roofline(trace_avg_ms, clocks),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * st.passes + (args.steps if world > 1 else 0),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
