#!/usr/bin/env python
"""Benchmark of the aligned-MSD / path-CV / close-structure hot path on B200.

    python bench.py [--config C] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one pass of the hot path over one batch of the config's synthetic
input (BASELINE.json configs; inputs resident in HBM for ``value``; host
pinned buffers with H2D/D2H inside the timed region for ``e2e``).  Multi-GPU
runs are launched with torchrun; the work is sharded per DESIGN.md
("Multi-GPU"), timed with CUDA events and reduced as the max over ranks.
``--impl reference`` times the C restatement of the reference CPU path
(oracle/c, all host cores) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
FALLBACK_BF16 = 1590.0  # TF/s


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sustained": p.get("bf16_tflops_sustained"),
                "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm": FALLBACK_HBM, "bf16": FALLBACK_BF16, "bf16_sustained": 1400.0,
                "src": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------- workloads
def load_workload(cfg, small=False):
    from paper_1801_02362_b200 import synth

    if cfg == 0:
        return synth.config0()
    if cfg == 1:
        return synth.config1(T=2000) if small else synth.config1()
    raise SystemExit(f"config {cfg} not wired into bench.py yet")


CONFIG_NAMES = {
    0: "config0: path-CV N=22 L=20 T=1000 fp64 exact",
    1: "config1: close-structure N=304 L=500 T=20000 fp64",
}


class OursConfig01:
    """Configs 0/1: fp64 path-CV (exact) / close-structure replay."""

    def __init__(self, cfg, wl, device):
        import torch

        from paper_1801_02362_b200 import engine

        self.cfg, self.wl, self.device = cfg, wl, device
        self.pcv = engine.PathCV(torch.from_numpy(wl.landmarks).to(device), wl.lam, wl.q)
        self.frames_dev = torch.from_numpy(wl.frames).to(device)
        self.frames_host = torch.from_numpy(wl.frames).pin_memory()
        self.T, self.n = wl.frames.shape[0], wl.frames.shape[1]
        self.last = None

    def step(self, frames):
        if self.cfg == 0:
            self.last = self.pcv.evaluate(frames, grad=True)
        else:
            self.last = self.pcv.close_replay(frames, self.wl.eps, grad=True)
        return self.last

    def step_device(self):
        return self.step(self.frames_dev)

    def step_e2e(self):
        import torch

        out = self.step(self.frames_host.to(self.device, non_blocking=True))
        res = [out["s"], out["z"]] + ([out["refresh"], out["dxy"]] if self.cfg == 1 else [])
        host = [r.to("cpu", non_blocking=True) for r in res]
        torch.cuda.current_stream().synchronize()
        return host

    def e2e_bytes(self):
        h2d = self.frames_host.numel() * self.frames_host.element_size()
        d2h = self.T * 8 * 2 + (self.T * 9 if self.cfg == 1 else 0)
        return h2d, d2h

    units_per_step = property(lambda self: self.T)
    metric = "path-CV frames/s"
    unit = "frames/s"


# algorithmic work per kernel launch
def kernel_work(name, runner):
    """(kind, amount) per launch: kind 'bytes' (HBM roofline) or 'flop'."""
    T, n = runner.T, runner.n
    L = runner.wl.landmarks.shape[0]
    npad = ((n + 31) // 32) * 32
    if name == "mc_cov_f64":
        return "fp64_flop", 18.0 * n * T * L
    if name == "mc_fit_dense":
        return "bytes", T * L * (72 + 8 + 72 + 1)
    if name == "mc_pathcv_weights":
        return "bytes", T * L * 8 * 2
    if name == "mc_pathcv_grad":
        return "bytes", T * npad * 3 * 8 + T * n * 3 * 8 * 2
    if name == "mc_center":
        return "bytes", T * n * 3 * 8 + T * 3 * npad * 8
    return "bytes", 0.0


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1801_02362_b200 import _lib

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        dist_mod.init_process_group("nccl", device_id=device)
        dist = dist_mod
    cfg = args.config
    wl = load_workload(cfg)
    runner = OursConfig01(cfg, wl, device)
    # configs 0/1 do not shard (sequential close-structure chain; tiny config 0):
    # every rank runs an independent replica
    for _ in range(args.warmup):
        runner.step_device()
    torch.cuda.synchronize()

    def timed(fn, k):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = e0.elapsed_time(e1) / k
        if dist:
            t = torch.tensor([ms], device=device, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    launches0 = _lib.COUNTERS["launches"]
    with ClockSampler(local_rank) as clk:
        ms = timed(runner.step_device, args.steps)
    clocks = clk.summary()
    launches = (_lib.COUNTERS["launches"] - launches0) // max(1, args.steps) * args.steps
    # end-to-end through the public API with host buffers
    runner.step_e2e()
    ms_e2e = timed(runner.step_e2e, args.steps)
    h2d, d2h = runner.e2e_bytes()
    # per-kernel live timing (CUDA events around each launch, on the launch stream)
    _lib.start_profile()
    for _ in range(max(1, min(args.steps, 3))):
        runner.step_device()
    prof = _lib.stop_profile()
    pk = peaks()
    total = sum(t for _, t in prof.values()) or 1.0
    top = max(prof.items(), key=lambda kv: kv[1][1])
    name, (cnt, tms) = top
    avg_ms = tms / cnt
    kind, amount = kernel_work(name, runner)
    if kind == "bytes":
        achieved = amount / (avg_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s", "frac": achieved / pk["hbm"]}
    else:
        achieved = amount / (avg_ms * 1e-3) / 1e12
        fp64_peak = 37.0  # TF/s nominal B200 FP64 (no measured figure in MEASURED_PEAKS.json)
        roof = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "peak_src": "nominal B200 FP64 (not measured)"}
    roof.update({"kernel": name, "share_of_step": tms / total, "avg_launch_ms": avg_ms, "traffic": None,
                 "peak_src": roof.get("peak_src", pk["src"])})
    kernels = {k: {"launches": c, "ms_per_step": t / max(1, min(args.steps, 3)), "share": t / total}
               for k, (c, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])}
    units = runner.units_per_step * world
    line = {
        "metric": runner.metric, "value": units / (ms * 1e-3), "unit": runner.unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py)",
        "config": {"workload": CONFIG_NAMES[cfg], "frames_per_rank": runner.T, "landmarks": int(wl.landmarks.shape[0]),
                   "atoms": runner.n, "parallelism": f"replicas x{world}" if world > 1 else "single",
                   "l2": "inputs re-read each step; working set (S/R/D buffers) > L2"},
        "e2e": {"value": units / (ms_e2e * 1e-3), "unit": runner.unit, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e},
        "gpu_launches": launches, "clocks": clocks, "roofline": roof, "kernels": kernels,
    }
    if cfg == 1 and runner.last is not None:
        line["config"]["refresh_fraction"] = float(runner.last["refresh"].float().mean().item())
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, wl, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_baseline(cfg, wl, args, seconds=12.0):
    """C restatement of the reference CPU path on a bounded sample (all host cores)."""
    from oracle import c_oracle as C

    threads = C.max_threads()
    frames = wl.frames
    if cfg == 0:
        fn = lambda fr: C.path_cv_exact(fr, wl.landmarks, wl.lam, wl.q)  # noqa: E731
    else:
        fn = lambda fr: C.close_replay(fr, wl.landmarks, wl.lam, wl.eps, wl.q)  # noqa: E731
    # calibrate the sample to ~`seconds` of CPU work
    k = min(frames.shape[0], 64)
    t0 = time.perf_counter()
    fn(frames[:k])
    dt = time.perf_counter() - t0
    k2 = int(min(frames.shape[0], max(k, k * seconds / max(dt, 1e-6))))
    t0 = time.perf_counter()
    fn(frames[:k2])
    dt = time.perf_counter() - t0
    return {"value": k2 / dt, "unit": "frames/s", "cores": threads, "kind": "port",
            "sample": f"first {k2} frames of the {CONFIG_NAMES[cfg].split(':')[0]} workload, "
                      f"oracle/c (C restatement of geometry.py + SPEC msd/colvar), OpenMP {threads} threads"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    wl = load_workload(cfg)
    from oracle import c_oracle as C

    threads = C.max_threads()
    frames = wl.frames
    L = wl.landmarks.shape[0]
    if cfg == 0:
        fn = lambda fr: C.path_cv_exact(fr, wl.landmarks, wl.lam, wl.q)  # noqa: E731
        sample = frames
    else:
        fn = lambda fr: C.close_replay(fr, wl.landmarks, wl.lam, wl.eps, wl.q)  # noqa: E731
        sample = frames[:1000]
    for _ in range(args.warmup):
        fn(sample[: max(1, len(sample) // 10)])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn(sample)
    dt = (time.perf_counter() - t0) / args.steps
    v = len(sample) / dt
    line = {
        "impl": "reference", "metric": "path-CV frames/s", "value": v, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py)",
        "config": {"workload": CONFIG_NAMES[cfg], "frames_per_step": len(sample), "landmarks": L,
                   "atoms": int(frames.shape[1])},
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"{len(sample)} frames per step, oracle/c OpenMP {threads} threads"},
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=int(os.environ.get("MC_BENCH_CONFIG", 1)))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline leg")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
