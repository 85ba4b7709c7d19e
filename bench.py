#!/usr/bin/env python
"""Benchmark of the aligned-MSD / path-CV / close-structure hot path on B200.

    python bench.py [--config C] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one pass of the hot path over one batch of the config's synthetic
input (BASELINE.json configs).  ``value`` is whole-job throughput with the
inputs resident in HBM; ``e2e`` is the same metric through the public API
with host (pinned) inputs, H2D and the D2H of the step's result inside the
timed region.  Multi-GPU runs (torchrun) shard the frames across ranks (no
data-path collective), time with CUDA events and take
the max over ranks.  ``--impl reference`` times the C restatement of the
reference CPU path (oracle/c, all host cores) on a bounded sample.

Default workload: config 4 (the largest config, the one BASELINE.json's
1/2/4/8-GPU scaling is stated on) — path-CV frames/s.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
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

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(r[1]) for r in rows) if v is not None]
        smax = [v for v in (num(r[2]) for r in rows) if v is not None]
        power = [v for v in (num(r[3]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(power) if power else None}


CONFIG_NAMES = {
    0: "config0: path-CV N=22 L=20 T=1000 fp64 exact",
    1: "config1: close-structure N=304 L=500 T=20000 fp64",
    2: "config2: all-pairs MSD matrix T=65536 L=4096 N=1000 fp32 (exact)",
    3: "config3: multi-walker close structure W=256 x 1000 steps N=2500 L=2048 fp32",
    4: "config4: path-CV s,z,grads N=10000 L=8192 T=131072 fp32",
}
CONFIG_SHAPES = {2: dict(seed=2, T=65536, L=4096, N=1000, n_endpoints=16),
                 4: dict(seed=4, T=131072, L=8192, N=10000, n_endpoints=32)}


# ----------------------------------------------------------------- runners
class Config01:
    """Configs 0/1: fp64 exact path-CV / close-structure replay (replicas across ranks)."""

    metric, unit, dtype = "path-CV frames/s", "frames/s", "f64"

    def __init__(self, cfg, device, rank, world):
        import torch

        from paper_1801_02362_b200 import engine, synth

        self.cfg, self.device = cfg, device
        self.wl = synth.config0() if cfg == 0 else synth.config1()
        self.pcv = engine.PathCV(torch.from_numpy(self.wl.landmarks).to(device), self.wl.lam, self.wl.q)
        self.frames_dev = torch.from_numpy(self.wl.frames).to(device)
        self.frames_host = torch.from_numpy(self.wl.frames).pin_memory()
        self.T, self.n, self.L = self.wl.frames.shape[0], self.wl.frames.shape[1], self.wl.landmarks.shape[0]
        # config 0 is launch-bound (~0.12 ms of kernels): the evaluate pipeline is
        # replayed from a CUDA graph (engine.PathCVGraph), status checked once per step
        self.graph = self.pcv.graph(self.T) if cfg == 0 and os.environ.get("MC_GRAPH", "1") == "1" else None
        self.last = None
        self.parallelism = f"replicas x{world}" if world > 1 else "single"
        self.scaling = "weak"

    def _step(self, frames):
        if self.cfg == 0 and self.graph is not None:
            self.last = self.graph.evaluate(frames)
        elif self.cfg == 0:
            self.last = self.pcv.evaluate(frames, grad=True)
        else:
            self.last = self.pcv.close_replay(frames, self.wl.eps, grad=True)
        return self.last

    def step_device(self):
        return self._step(self.frames_dev)

    def step_profile(self):
        """Per-kernel CUDA-event profile: the eager launches of the graphed pipeline."""
        if self.cfg == 0:
            self.last = self.pcv.evaluate(self.frames_dev, grad=True, cap=self.L)
            return self.last
        return self.step_device()

    def step_e2e(self):
        import torch

        out = self._step(self.frames_host if self.graph is not None else
                         self.frames_host.to(self.device, non_blocking=True))
        if self.graph is not None:
            self.graph.check()
        res = [out["s"], out["z"]] + ([out["refresh"], out["dxy"]] if self.cfg == 1 else [])
        host = [r.to("cpu", non_blocking=True) for r in res]
        torch.cuda.current_stream().synchronize()
        return host

    def e2e_bytes(self):
        return self.frames_host.numel() * 8, self.T * 16 + (self.T * 9 if self.cfg == 1 else 0)

    def units(self):
        return self.T

    def kernel_work(self, name):
        T, n, L = self.T, self.n, self.L
        npad = ((n + 31) // 32) * 32
        if name == "mc_cov_f64":  # on DMMA (cov_dmma_f64_kernel) unless MC_COV_F64=1
            return ("fp64_flop" if os.environ.get("MC_COV_F64") == "1" else "fp64_tensor_flop"), 18.0 * n * T * L
        if name == "mc_fit_dense":
            return "bytes", T * L * (72 + 8 + 72 + 1)
        if name == "mc_pathcv_weights":
            return "bytes", T * L * 8 * 2
        if name == "mc_pathcv_grad":
            return "bytes", T * npad * 3 * 8 + T * n * 3 * 8 * 2
        if name == "mc_center":
            return "bytes", T * n * 3 * 8 + T * 3 * npad * 8
        return "bytes", 0.0

    def extra(self):
        d = {}
        if self.cfg == 1 and self.last is not None:
            d["refresh_fraction"] = float(self.last["refresh"].float().mean().item())
        return d


class Config3:
    """Config 3: W walkers x 1000 steps, each with its own floating close structure
    (fp32 coordinates, fp64 finalisation; exact fp64 path).  Walkers are sharded
    across ranks (independent objects, no collective)."""

    metric, unit = "path-CV frames/s", "frames/s"
    dtype = ("f32 coordinates; one-term FP16 tcgen05 screen of the refresh frames -> close-structure lifetime "
             "windows -> covariances and refresh fits on tcgen05 kind::i8 (exact int8 row digits) -> fp64 Eq. 5 / "
             "weights -> gradient contraction (DMMA for windows wider than 117 landmarks)")

    def __init__(self, device, rank, world, walkers_override=None):
        from paper_1801_02362_b200 import dist as D
        from paper_1801_02362_b200 import engine, synth

        # weak scaling: every rank replays its own W walkers (disjoint seeds of one
        # global walker set), no data-path collective
        W = walkers_override or 256
        self.steps, self.n, self.L = 1000, 2500, 2048
        off, cnt = rank * W, W
        self.wl = synth.walkers_device(3, world * W, self.steps, self.n, self.L, device, off, cnt)
        self.device = device
        self.W_all, self.Wloc = world * W, cnt
        self.T = cnt * self.steps
        import torch

        self.pcv = engine.PathCV(torch.from_numpy(self.wl.landmarks).to(device), self.wl.lam, self.wl.q)
        self.frames_dev = self.wl.frames
        try:
            self.frames_host = self.frames_dev.cpu().pin_memory()
        except RuntimeError:
            self.frames_host = self.frames_dev.cpu()
        self.parallelism = f"walker-sharded dp{world}" if world > 1 else "single"
        self.scaling = "weak"
        self.last = None

    def _step(self, frames):
        self.last = self.pcv.close_replay(frames, self.wl.eps, grad=True)
        return self.last

    def step_device(self):
        return self._step(self.frames_dev)

    def step_e2e(self):
        import torch

        out = self._step(self.frames_host.to(self.device, non_blocking=True))
        if not hasattr(self, "_host"):
            self._host = {k: torch.empty(out[k].shape, dtype=out[k].dtype).pin_memory()
                          for k in ("ds", "dz", "s", "z", "refresh", "dxy")}
        for k, h in self._host.items():  # the whole result: gradients, s, z, refresh log, D(x, y)
            h.copy_(out[k], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self._host

    def e2e_bytes(self):
        return self.T * self.n * 12, self.T * (2 * self.n * 3 * 4 + 8 + 8 + 1 + 8)

    def units(self):
        return self.T

    def kernel_work(self, name):
        T, n, L = self.T, self.n, self.L
        if name == "mc_cov_f64":
            return "fp64_flop", 18.0 * n * T * L
        if name == "mc_cov_dmma":  # dense S [T, L, 9]: 9 fp64 FMA per atom and pair on DMMA
            return "fp64_tensor_flop", 18.0 * n * T * L
        if name in ("mc_pathcv_grad_i8", "mc_pathcv_grad_i8_wide") and self.last is not None:
            # executed int8 MMA work: per (frame, significant landmark, atom) 18 multiply-adds
            # (2 CVs x 3 x 3) x the 10 kept digit products (tcgen05.mma kind::i8)
            return "int8_tensor_op", 2.0 * 10.0 * 18.0 * n * float(self.last["nsig"].double().sum().item())
        if name == "mc_pathcv_grad_block" and self.last is not None:
            return "fp64_tensor_flop", 36.0 * n * float(self.last["nsig"].double().sum().item())
        if name == "mc_fit_dense":
            return "bytes", T * L * (72 + 8 + 72 + 1)
        if name in ("mc_refine_i8", "mc_refine_i8_close") and self.last is not None and "window_cnt" in self.last:
            # pruned replay: every frame's covariances over its close structure's window
            # (9 multiply-adds per pair and atom x 10 digit products)
            return "int8_tensor_op_refine", 2.0 * 10.0 * 9.0 * n * float(self.last["window_cnt"].double().sum().item())
        return "bytes", 0.0

    def extra(self):
        d = {"walkers": self.W_all, "walkers_per_rank": self.Wloc, "steps": self.steps}
        if self.last is not None:
            d["refresh_fraction"] = float(self.last["refresh"].float().mean().item())
            if "window_cnt" in self.last:
                d["mean_window"] = float(self.last["window_cnt"].float().mean().item())
                d["mean_significant"] = float(self.last["nsig"].float().mean().item())
        return d


class ConfigTC:
    """Configs 2/4: fp32 path on tcgen05 (3xTF32 estimate) + exact fp64 refinement.
    Frames are sharded across ranks; landmarks are replicated (no collective)."""

    def __init__(self, cfg, device, rank, world, frames_override=None, shard="frames"):
        import torch

        from paper_1801_02362_b200 import engine, synth

        self.cfg, self.device = cfg, device
        shp = dict(CONFIG_SHAPES[cfg])
        if frames_override:
            shp["T"] = frames_override
        self.shard = shard
        if shard.startswith("landmarks") and cfg != 4:
            raise SystemExit("--shard landmarks applies to config 4 (path-CV)")
        if shard in ("landmarks", "landmarks-allgather", "landmarks-routed"):
            # the north_star's variant.  "landmarks": the survey's
            # two-phase plan -- rank g screens its landmark shard for every frame (one
            # all-gather of the frames' screening operand, O(T) minima / windows), then refits
            # and differentiates its T/G home frames against the replicated landmarks;
            # "landmarks-routed": frames routed to the shards their admissible tiles live on,
            # gradient rows come back home.  Strong scaling (total work fixed), each rank
            # copies only its home frames.
            from paper_1801_02362_b200 import dist as Dd

            T_all = shp["T"]
            off, cnt = Dd.shard_range(T_all, rank, world)
        elif shard == "landmarks-replicated":
            # every rank holds all T frames and its landmark shard; per-frame minima /
            # partials / straddling gradient rows are exchanged over NCCL
            T_all, off, cnt = shp["T"], 0, shp["T"]
        else:
            # strong scaling: the config's fixed frame set (T frames) is split across the
            # ranks, T / G frames each, landmarks replicated, no data-path collective
            from paper_1801_02362_b200 import dist as Dd

            T_all = shp["T"]
            off, cnt = Dd.shard_range(T_all, rank, world)
        self.wl = synth.interp_config_device(shp["seed"], T_all, shp["L"], shp["N"], shp["n_endpoints"], device,
                                             frame_offset=off, frame_count=cnt)
        self.T_all, self.T = T_all, cnt
        self.n, self.L = shp["N"], shp["L"]
        self._off, self._c0 = off, 0
        lms = torch.from_numpy(self.wl.landmarks).to(device)
        if shard == "landmarks":  # two-phase, phase 1 routed (each frame's operand to the shards it needs)
            self.pcv = engine.PathCVTC(lms, self.wl.lam, self.wl.q, shard=(rank, world, Dd.tile_bounds(self.L, world)),
                                       route=True, two_phase=True)
        elif shard == "landmarks-allgather":  # two-phase, every frame's operand all-gathered
            self.pcv = engine.PathCVTC(lms, self.wl.lam, self.wl.q, shard=(rank, world), two_phase=True)
        elif shard == "landmarks-routed":
            self.pcv = engine.PathCVTC(lms, self.wl.lam, self.wl.q, shard=(rank, world, Dd.tile_bounds(self.L, world)),
                                       route=True)
        else:
            self.pcv = engine.PathCVTC(lms, self.wl.lam, self.wl.q,
                                       shard=(rank, world) if shard == "landmarks-replicated" else None)
        if shard.startswith("landmarks"):
            from paper_1801_02362_b200 import dist as Dd

            self._comm = Dd.DistComm() if world > 1 else None
            self.L_local = self.pcv.L
        self.frames_dev = self.wl.frames
        self.chunk = 24576
        try:
            self.frames_host = self.frames_dev.cpu().pin_memory()
            self.host_kind = "pinned"
        except RuntimeError:
            self.frames_host = self.frames_dev.cpu()
            self.host_kind = "pageable (pinning failed)"
        if shard == "landmarks":
            self.parallelism = (f"landmark-sharded x{world}, two-phase routed (NCCL: each frame's one-term screening "
                                "operand to the shards its coarse hull meets, all-reduce MIN of the per-frame "
                                "estimate minimum, windows back home; refits and gradients frame-sharded against "
                                "replicated landmarks)")
            self.scaling = "strong"
            self.replicated_units = False
        elif shard == "landmarks-allgather":
            self.parallelism = (f"landmark-sharded x{world}, two-phase (NCCL: one all-gather of the frames' one-term "
                                "screening operand, all-reduce MIN of per-frame bounds, all-gather of per-shard "
                                "windows; refits and gradients frame-sharded against replicated landmarks)")
            self.scaling = "strong"
            self.replicated_units = False
        elif shard == "landmarks-routed":
            self.parallelism = (f"landmark-sharded x{world}, frame-routed (NCCL: frames to their shards, "
                                "per-frame min/partials, gradient rows home)")
            self.scaling = "strong"
            self.replicated_units = True  # value = the T global frames / the slowest rank's time
        elif shard == "landmarks-replicated":
            self.parallelism = f"landmark-sharded x{world} (NCCL: per-frame min/partials + straddling rows)"
            self.scaling = "strong"
            self.replicated_units = True  # every rank evaluates the same T frames
        else:
            self.parallelism = (f"frame-sharded x{world} (T/{world} frames per rank, landmarks replicated, "
                                "no collective)") if world > 1 else "single"
            self.scaling = "strong"
        self.last = None
        if cfg == 2:
            self.metric, self.unit = "aligned-MSD pairs/s", "pairs/s"
            self.D = torch.empty((self.T, self.L), dtype=torch.float32, device=device)
        else:
            self.metric, self.unit = "path-CV frames/s", "frames/s"
            # metadynamics bias over (s, z) for the fused-force end-to-end variant: 256 hills
            # spread along the path (direct summation, SPEC bias_and_force)
            from paper_1801_02362_b200.metadynamics import HillStore

            self.hills = HillStore(2, 1, 1.0, [16.0, 0.005], device=device)
            hr = np.random.default_rng(44)
            for k, c in enumerate(zip(hr.uniform(0, self.L - 1, 256), hr.uniform(0.0, 0.02, 256))):
                self.hills.deposit(torch.tensor(c, dtype=torch.float64), k)
        if cfg == 2:
            self.dtype = ("f32 coordinates; every pair's covariance on tcgen05 kind::i8 with exact int8 row digits "
                          "(int32 accumulation, fp64 recombination) + fused fp64 fit")
        else:
            self.dtype = ("f32 coordinates; one-term FP16 tcgen05 screen (rigorous bound) -> exact fp64 refits "
                          "(tcgen05 kind::i8, exact int8 row digits) -> fp64 weights -> gradient contraction on "
                          "tcgen05 kind::i8 with exact int8 "
                          "digits (int32 accumulation, fp64 recombination)")

    def _step(self, frames, D=None):
        if self.cfg == 2:
            self.last = self.pcv.msd_matrix(frames) if D is None else self._msd_into(frames, D)
        elif self.shard.startswith("landmarks"):
            from paper_1801_02362_b200 import dist as Dd

            if self.shard in ("landmarks", "landmarks-allgather"):
                # home offsets / totals of chunked calls follow from the gathered counts
                steps = self.pcv.two_phase_steps(frames, None, None, grad=True)
            elif self.shard == "landmarks-routed":
                steps = self.pcv.routed_steps(frames, self._off + self._c0, self.T_all, grad=True)
            else:
                steps = self.pcv.sharded_steps(frames, grad=True)
            self.last = Dd.drive(steps, self._comm) if self._comm else Dd.drive_lockstep([steps])[0]
        else:
            self.last = self.pcv.evaluate(frames, grad=True)
        return self.last

    def _msd_into(self, frames, D):
        return self.pcv.msd_matrix(frames, out=D)

    def step_device(self):
        return self._step(self.frames_dev, self.D if self.cfg == 2 else None)

    def e2e_chunks(self, d2h_bound=False, taper=False):
        """Chunk boundaries of the streamed step.  The H2D copy (2.16 us/frame at
        55.6 GB/s) is slower than the compute (~2.5 ms + 1.72 us/frame per chunk on
        config 4), so the step is copy-bound and ends one chunk-compute after the
        last copy: chunk sizes shrink geometrically (x0.87) towards a last chunk of
        T/16, so each chunk's compute finishes under the next chunk's copy and only
        a small compute is exposed at the end, while chunks stay large enough for
        the pruning bands and frame groups to stay tight (sweeps:
        tools/_diag/e2e_sched.py, tools/_diag/e2e_timeline.py)."""
        env = os.environ.get("MC_E2E_CHUNKS")  # "first,steady[,growth[,taper]]" | "list:n1,n2,..." (knob)
        if not env and self.cfg == 2:
            # config 2 is compute-bound (12 KB in, 16 KB out per frame): few large chunks,
            # small first / last ones (tools/_diag/e2e_c2.sh: 188.8 -> 182.4 ms)
            e = max(32, (self.T // 32) // 32 * 32)
            mid = (self.T - 2 * e) // 2
            sizes = [e, mid, self.T - 2 * e - mid, e] if self.T > 4 * e else [self.T]
            out, c0 = [], 0
            for n in sizes:
                out.append((c0, n))
                c0 += n
            return out
        if not env and d2h_bound:
            # the whole result back (ds, dz: 2x the input bytes): the D2H stream is the
            # bottleneck, so it must start early -- a small first chunk, doubling to a steady
            # size; the tail is short because every chunk's compute is far below its D2H
            steady = max(1024, min(self.T // 8, 16384) // 32 * 32)
            ramp = []
            size = 1024
            while size < steady:
                ramp.append(size)
                size *= 2
            # taper (the fused-force step, as many bytes back as in): the last chunks shrink
            # again so the final compute + D2H after the last H2D is short
            tail = list(reversed(ramp)) if taper and self.T > 2 * sum(ramp) + steady else []
            sizes, left = [], self.T - sum(tail)
            for n in ramp + [steady] * max(0, left):
                if left <= 0:
                    break
                n = min(n, left)
                sizes.append(n)
                left -= n
            sizes += tail
            out, c0 = [], 0
            for n in sizes:
                out.append((c0, n))
                c0 += n
            return out
        if not env:
            div = int(os.environ.get("MC_E2E_TAIL", "16"))  # last chunk = T / div (sweep knob)
            tail = [max(1024, (self.T // div) // 32 * 32)]
            while sum(tail) < self.T:
                nxt = int(tail[-1] / 0.87) // 32 * 32
                tail.append(min(nxt, self.T - sum(tail)))
            out, c0 = [], 0
            for n in reversed(tail):
                out.append((c0, n))
                c0 += n
            return out
        first, steady, growth, taper = self.chunk // 6, self.chunk, 1.5, True
        if env and env.startswith("list:"):
            sizes = [int(x) for x in env[5:].split(",")]
            out, c0 = [], 0
            for n in sizes:
                n = min(n, self.T - c0)
                if n <= 0:
                    break
                out.append((c0, n))
                c0 += n
            if c0 < self.T:
                out.append((c0, self.T - c0))
            return out
        if env:
            parts = [float(x) for x in env.split(",")]
            first, steady = int(parts[0]), int(parts[1])
            growth = parts[2] if len(parts) > 2 else 2.0
            taper = bool(int(parts[3])) if len(parts) > 3 else True
        ramp, size = [], max(1, first)
        while size < steady:
            ramp.append(int(size))
            size = max(size + 1, int(size * growth))
        head, tail = list(ramp), (list(reversed(ramp)) if taper else [])
        sizes, left = [], self.T
        while left > 0:
            if head:
                n = head.pop(0)
            elif left > sum(tail) + steady:
                n = steady
            elif tail and left > sum(tail):
                n = left - sum(tail)
            elif tail:
                n = tail.pop(0)
            else:
                n = steady
            n = min(n, left)
            sizes.append(n)
            left -= n
        out, c0 = [], 0
        for n in sizes:
            out.append((c0, n))
            c0 += n
        return out

    def step_e2e(self, force=False):
        """Public API with host frames: chunked H2D on a copy stream, double-buffered
        against the compute of the previous chunk, then D2H of the whole result (config 4:
        ds, dz, s, z -- or with force=True the fused bias force F, s, z, V)."""
        import torch

        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(device=self.device)
        comp = torch.cuda.current_stream()
        cps = self._copy_stream
        outs = []
        chunks = self.e2e_chunks(d2h_bound=(self.cfg == 4), taper=force)

        def issue(ch):
            c0, n = ch
            with torch.cuda.stream(cps):
                buf = self.frames_host[c0:c0 + n].to(self.device, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cps)
            return buf, ev

        nxt = issue(chunks[0]) if chunks else None
        for i, _ in enumerate(chunks):
            fr, ev = nxt
            if i + 1 < len(chunks):
                nxt = issue(chunks[i + 1])
            comp.wait_event(ev)
            fr.record_stream(comp)
            if self.cfg == 2:
                # the [n, L] result goes back on its own stream into pinned memory, so the
                # D2H of chunk i overlaps the compute of chunk i + 1 (full-duplex PCIe)
                if not hasattr(self, "_d2h_stream"):
                    self._d2h_stream = torch.cuda.Stream(device=self.device)
                    self._d_host = torch.empty((self.T, self.L), dtype=torch.float32).pin_memory()
                D = self._step(fr)
                done = torch.cuda.Event()
                done.record(comp)
                c0, n = chunks[i]
                with torch.cuda.stream(self._d2h_stream):
                    self._d2h_stream.wait_event(done)
                    D.record_stream(self._d2h_stream)
                    self._d_host[c0:c0 + n].copy_(D, non_blocking=True)
                if i + 1 == len(chunks):
                    comp.wait_stream(self._d2h_stream)
                    outs.append(self._d_host)
            else:
                self._c0 = chunks[i][0]  # home offset of this chunk (frame-routed landmark shards)
                if force:
                    o = self.pcv.evaluate(fr, grad=False, bias=self.hills)
                    res = [o["force"], o["s"], o["z"], o["V"]]
                else:
                    o = self._step(fr)
                    res = [o["ds"], o["dz"], o["s"], o["z"]]
                # the step's whole result back to the host, on its own stream (full-duplex
                # PCIe: chunk i's D2H overlaps chunk i + 1's H2D and compute); pinned
                # double-buffered host slots (stream order makes slot reuse safe)
                done = torch.cuda.Event()
                done.record(comp)
                slot = self._host_slots(chunks, force)[i % 2]
                n = chunks[i][1]
                with torch.cuda.stream(self._d2h_stream):
                    self._d2h_stream.wait_event(done)
                    for r, h in zip(res, slot):
                        r.record_stream(self._d2h_stream)
                        h[:n].copy_(r, non_blocking=True)
                if i + 1 == len(chunks):
                    comp.wait_stream(self._d2h_stream)
                    outs.append(slot)
        self._c0 = 0
        comp.synchronize()
        return outs

    def _host_slots(self, chunks, force):
        """Two pinned host slots for the chunk results (gradients or force + per-frame scalars)."""
        import torch

        key = "force" if force else "grad"
        if not hasattr(self, "_slots"):
            self._slots = {}
            self._d2h_stream = torch.cuda.Stream(device=self.device)
        if key not in self._slots:
            m = max(n for _, n in chunks)
            big = 1 if force else 2
            self._slots[key] = [[torch.empty((m, self.n, 3), dtype=torch.float32).pin_memory() for _ in range(big)] +
                                [torch.empty((m,), dtype=torch.float64).pin_memory() for _ in range(4 - big)]
                                for _ in range(2)]
        return self._slots[key]

    def step_e2e_force(self):
        """The metadynamics consumer's call: s, z, V and the fused bias force F [T, n, 3]
        (one tensor-core contraction, no ds / dz) back to the host."""
        return self.step_e2e(force=True)

    def e2e_bytes(self, force=False):
        h2d = self.T * self.n * 3 * 4
        if self.cfg == 2:
            d2h = self.T * self.L * 4
        elif force:
            d2h = self.T * self.n * 3 * 4 + self.T * 3 * 8  # F, s, z, V
        else:
            d2h = 2 * self.T * self.n * 3 * 4 + self.T * 2 * 8  # ds, dz, s, z
        return h2d, d2h

    def units(self):
        return self.T * self.L if self.cfg == 2 else self.T

    def kernel_work(self, name):
        T, n, L = self.T, self.n, self.L
        if name in ("mc_msd_tf32", "mc_msd_tf32_2sm"):
            return "tensor_flop", 3.0 * 18.0 * n * T * L
        if name in ("mc_msd_f16", "mc_msd_f16_2sm"):
            terms = self.pcv.screen_terms if self.cfg == 4 else 3
            pairs = T * L
            if self.cfg == 4 and self.last is not None and "screen_tiles" in self.last:
                tiles = int(self.last["screen_tiles"].item())
                pairs = T * self.pcv.coarse.numel() + tiles * 128 * 48  # coarse + banded
            return "tensor_flop_f16", terms * 18.0 * n * pairs
        if name in ("mc_pathcv_grad_i8", "mc_pathcv_grad_i8_wide") and self.last is not None:
            # executed int8 MMA work: per (frame, significant landmark, atom) 18 multiply-adds
            # (2 CVs x 3 x 3) x the 10 kept digit products (tcgen05.mma kind::i8)
            return "int8_tensor_op", 2.0 * 10.0 * 18.0 * n * float(self.last["nsig"].double().sum().item())
        if name == "mc_pathcv_grad_block" and self.last is not None:
            # useful fp64 work: 18 FMA (U^s, U^z: 2 CVs x 3 x 3) per significant pair and atom
            return "fp64_tensor_flop", 36.0 * n * float(self.last["nsig"].double().sum().item())
        if name == "mc_refine_i8":
            # executed int8 MMA work: 9 multiply-adds (3 x 3) per (pair, atom) x the 10 kept digit
            # products; pairs = every pair (config 2) or the window pairs (config 4)
            if self.cfg == 2:
                pairs = float(T * L)
            elif self.last is not None:
                pairs = float(self.last["window_cnt"].double().sum().item())
            else:
                pairs = 0.0
            return "int8_tensor_op_refine", 2.0 * 10.0 * 9.0 * n * pairs
        if name in ("mc_center_split16", "mc_center_split16_uniform"):
            return "bytes", T * n * 3 * 4 + 2 * T * 3 * (((n + 31) // 32) * 32) * 2
        if name == "mc_refine":
            if self.cfg == 2:
                return "fp64_tensor_flop", 18.0 * n * T * L
            if self.last is not None:  # exact refits of the window pairs: 9 FMA per pair and atom
                return "fp64_tensor_flop", 18.0 * n * float(self.last["window_cnt"].double().sum().item())
            return "fp64_tensor_flop", 0.0
        if name == "mc_center_split":
            return "bytes", T * n * 3 * 4 + 2 * T * 3 * (((n + 15) // 16) * 16) * 4
        if name == "mc_pathcv_grad":
            return "bytes", T * n * 3 * 4 + T * n * 3 * 4 * 2
        if name == "mc_candidates":
            return "bytes", T * L * 4
        return "bytes", 0.0

    def extra(self):
        d = {"pairs_per_step": self.T * self.L, "host_buffers": self.host_kind}
        if self.shard.startswith("landmarks"):
            d["landmarks_per_rank"] = self.pcv.L
        if self.cfg == 4 and self.last is not None:
            d["mean_window"] = float(self.last["window_cnt"].float().mean().item())
            d["mean_significant"] = float(self.last["nsig"].float().mean().item())
            if "screen_tiles" in self.last:
                ntl = (self.L + 47) // 48
                full = ((self.T + 127) // 128) * ntl
                d["screen_tiles_computed_frac"] = int(self.last["screen_tiles"].item()) / full
                d["screen"] = "one-term FP16, metric-pruned (coarse stride %d)" % (self.L // self.pcv.coarse.numel())
        return d


DMMA_PEAK_TF = 36.2  # measured mma.sync f64 rate on this pool's B200 (profiles/r02_dmma_probe_b200.txt)


def _int8_roof(amount, step_ms, pk, basis=None):
    """Roofline of an int8 tcgen05 kernel: executed int8 ops per second against twice the
    measured bf16 GEMM rate (kind::i8 issues twice the multiply-adds of kind::f16 per cycle:
    8192 vs 4096 per SM, tools/_diag/i8_probe.cu)."""
    ach = amount / (step_ms * 1e-3) / 1e12
    sustained = 2.0 * (pk.get("bf16_sustained") or pk["bf16"])
    return {"bound": "tensor", "achieved": ach, "peak": sustained, "unit": "TOPS (int8)", "frac": ach / sustained,
            "peak_src": f"2 x bf16_tflops_sustained from {pk['src']} (kind::i8 = 2x the kind::f16 MAC rate, "
                        "measured by tools/_diag/i8_probe.cu)",
            "peak_burst": 2.0 * pk["bf16"], "frac_of_burst": ach / (2.0 * pk["bf16"]),
            "flop_basis": basis or ("executed int8 multiply-adds x 2: 10 digit products x 18 per (frame, "
                                    "significant landmark, atom)")}


def measured_traffic(kernel, cfg, T):
    """DRAM bytes per launch of `kernel` from a committed ncu --set full capture of
    this workload (profiles/traffic.json), else None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            tab = json.load(f)
        v = tab.get(kernel, {}).get(f"config{cfg}:T{T}")
        return v
    except (OSError, ValueError):
        return None


def tf32_peak_measure(device):
    """cuBLAS TF32 GEMM rate on this box (cross-check of the derived peak)."""
    import torch

    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn((8192, 8192), device=device)
        b = torch.randn((8192, 8192), device=device)
        for _ in range(3):
            a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2 * 8192 ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None
    finally:
        torch.backends.cuda.matmul.allow_tf32 = False


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
    if cfg in (0, 1):
        runner = Config01(cfg, device, rank, world)
    elif cfg == 3:
        runner = Config3(device, rank, world, args.walkers)
    else:
        runner = ConfigTC(cfg, device, rank, world, args.frames, args.shard)
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
    launches = _lib.COUNTERS["launches"] - launches0
    # end-to-end through the public API with host buffers
    runner.step_e2e()
    ms_e2e = timed(runner.step_e2e, args.steps)
    h2d, d2h = runner.e2e_bytes()
    e2e_force = None
    if hasattr(runner, "step_e2e_force") and cfg == 4 and runner.shard == "frames":
        runner.step_e2e_force()
        ms_f = timed(runner.step_e2e_force, args.steps)
        h2f, d2f = runner.e2e_bytes(force=True)
        e2e_force = {"value": None, "ms_per_step": ms_f, "h2d_bytes_per_step": h2f * (world if runner.scaling == "weak" else 1),
                     "d2h_bytes_per_step": d2f * (world if runner.scaling == "weak" else 1),
                     "what": "evaluate(frames, grad=False, bias=HillStore): s, z, V and the metadynamics bias force "
                             "F = -(dV/ds ds + dV/dz dz) [T, n, 3] from one fused int8 tensor-core contraction "
                             "(SPEC bias_and_force), all copied back to pinned host memory"}
    # live per-kernel timing: CUDA events around each launch on the launch stream
    nprof = max(1, min(args.steps, 2))
    _lib.start_profile()
    for _ in range(nprof):
        getattr(runner, "step_profile", runner.step_device)()
    prof = _lib.stop_profile()
    pk = peaks()
    total = sum(t for _, t in prof.values()) or 1.0
    name, (cnt, tms) = max(prof.items(), key=lambda kv: kv[1][1])
    avg_ms = tms / cnt
    step_ms = tms / nprof  # the kernel's time per step (all its launches)
    gk_names = ("mc_pathcv_grad_i8", "mc_pathcv_grad_i8_wide")
    if name in gk_names:  # the int8 contraction's work spans its narrow and wide kernels
        step_ms = sum(prof[k][1] for k in gk_names if k in prof) / nprof
    kind, amount = runner.kernel_work(name)
    tf32_cublas = tf32_peak_measure(device) if kind == "tensor_flop" and rank == 0 else None
    if kind == "bytes":
        ach = amount / (step_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": pk["hbm"], "unit": "GB/s", "frac": ach / pk["hbm"],
                "peak_src": pk["src"]}
    elif kind == "tensor_flop":
        ach = amount / (step_ms * 1e-3) / 1e12
        # the kernel runs for ~1 s inside a multi-second step: the sustained
        # (power-capped) figure is the right denominator; burst reported beside it
        sustained = pk.get("bf16_sustained") or pk["bf16"]
        peak = sustained / 2.0
        roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_src": f"TF32 = bf16_tflops_sustained/2 from {pk['src']} (TF32 runs at half the bf16 rate; "
                            "kernel timed inside a long step)",
                "peak_burst": pk["bf16"] / 2.0, "frac_of_burst": ach / (pk["bf16"] / 2.0),
                "cublas_tf32_measured": tf32_cublas, "flop_basis": "executed 3xTF32 (3 x 18 n per pair)"}
    elif kind == "tensor_flop_f16":
        ach = amount / (step_ms * 1e-3) / 1e12
        sustained = pk.get("bf16_sustained") or pk["bf16"]
        roof = {"bound": "tensor", "achieved": ach, "peak": sustained, "unit": "TFLOP/s", "frac": ach / sustained,
                "peak_src": f"bf16_tflops_sustained from {pk['src']} (kind::f16 runs at the bf16 rate; "
                            "kernel timed inside a long step)",
                "peak_burst": pk["bf16"], "frac_of_burst": ach / pk["bf16"],
                "flop_basis": "executed FP16 MMAs: terms x 18 n per pair (config 4 screen: one-term hi x hi; "
                              "split-precision estimate: 3 terms)"}
    elif kind == "fp64_tensor_flop":
        ach = amount / (step_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": DMMA_PEAK_TF, "unit": "TFLOP/s", "frac": ach / DMMA_PEAK_TF,
                "peak_src": "fp64 tensor cores (DMMA.8x8x4) measured on this pool's B200: 36.2 TF/s "
                            "(profiles/r02_dmma_probe_b200.txt from tools/_diag/dmma_probe.cu; "
                            "MEASURED_PEAKS.json has no fp64 figure)",
                "flop_basis": "useful fp64 flops (significant / window pairs); executed includes window-union padding"}
    elif kind == "int8_tensor_op":
        roof = _int8_roof(amount, step_ms, pk)
    elif kind == "int8_tensor_op_refine":
        roof = _int8_roof(amount, step_ms, pk, "executed int8 multiply-adds x 2: 10 digit products x 9 per "
                                               "(refit pair, atom)")
    else:
        ach = amount / (step_ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": ach, "peak": 37.0, "unit": "TFLOP/s", "frac": ach / 37.0,
                "peak_src": "nominal B200 FP64 37 TF/s (not measured)"}
    traffic = measured_traffic(name, cfg, runner.T)
    roof.update({"kernel": "+".join(k for k in gk_names if k in prof) if name in gk_names else name,
                 "share_of_step": step_ms * nprof / total, "avg_launch_ms": avg_ms, "traffic": traffic,
                 "traffic_unit": "bytes per launch (dram read + write)",
                 "traffic_src": "profiles/traffic.json (ncu --set full, same workload)" if traffic else None})
    kernels = {k: {"launches": c, "ms_per_step": t / nprof, "share": t / total}
               for k, (c, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])}
    # the gradient contraction's own roofline (int8 tensor pipe) when it is not the top kernel
    roof_grad = None
    if name not in gk_names and any(k in prof for k in gk_names):
        gk, gamount = runner.kernel_work("mc_pathcv_grad_i8")
        gc = sum(prof[k][0] for k in gk_names if k in prof)
        gt = sum(prof[k][1] for k in gk_names if k in prof)
        if gk == "int8_tensor_op":
            roof_grad = _int8_roof(gamount, gt / nprof, pk)
            roof_grad.update({"kernel": "+".join(k for k in gk_names if k in prof), "share_of_step": gt / total,
                              "avg_launch_ms": gt / gc})
    roof_refine = None
    if name != "mc_refine_i8" and "mc_refine_i8" in prof and hasattr(runner, "pcv"):
        rk, ramount = runner.kernel_work("mc_refine_i8")
        rc, rt = prof["mc_refine_i8"]
        if rk == "int8_tensor_op_refine":
            roof_refine = _int8_roof(ramount, rt / nprof, pk, "executed int8 multiply-adds x 2: 10 digit products x 9 "
                                                              "per (refit pair, atom)")
            roof_refine.update({"kernel": "mc_refine_i8", "share_of_step": rt / total, "avg_launch_ms": rt / rc})
    units = runner.units() * world if runner.scaling == "weak" else runner.units()
    if dist and runner.scaling == "strong" and not getattr(runner, "replicated_units", False):
        t = torch.tensor([float(units)], device=device, dtype=torch.float64)
        dist.all_reduce(t)
        units = float(t.item())
    # bytes per step of the whole job: every rank copies its own frames and results
    h2d_tot, d2h_tot = h2d * world, d2h * world
    if e2e_force is not None:
        e2e_force["value"] = units / (e2e_force["ms_per_step"] * 1e-3)
        e2e_force["unit"] = runner.unit
        e2e_force["h2d_bytes_per_step"] *= world
        e2e_force["d2h_bytes_per_step"] *= world
    line = {
        "metric": runner.metric, "value": units / (ms * 1e-3), "unit": runner.unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": runner.scaling, "vs_baseline": None, "dtype": runner.dtype,
        "data": "synthetic (seeded; synth.py, configs 2/4 generated on device)",
        "config": {"workload": CONFIG_NAMES[cfg], "frames_per_rank": runner.T, "landmarks": runner.L,
                   "atoms": runner.n, "parallelism": runner.parallelism,
                   "l2": "working set > L2 (126 MB): frames/operands re-read from HBM every step"},
        "e2e": {"value": units / (ms_e2e * 1e-3), "unit": runner.unit,
                "h2d_bytes_per_step": h2d_tot,
                "d2h_bytes_per_step": d2h_tot, "ms_per_step": ms_e2e,
                "what": "the public API with pinned host frames: chunked H2D, evaluate(), and the whole result "
                        "(config 4: ds, dz, s, z; config 2: the MSD matrix) back to pinned host memory"},
        "gpu_launches": launches, "clocks": clocks, "roofline": roof, "kernels": kernels,
    }
    if e2e_force is not None:
        line["e2e_bias_force"] = e2e_force
    if roof_grad is not None:
        line["roofline_gradient"] = roof_grad
    if roof_refine is not None:
        line["roofline_refits"] = roof_refine
    line["config"].update(runner.extra())
    if cfg == 4 and getattr(runner, "last", None) is not None and "window_cnt" in runner.last:
        # the BASELINE metric's other half: aligned-MSD pairs/s of the same step -- every
        # (frame, landmark) pair is covered (screened or pruned with a certified bound) and
        # the window pairs are refit exactly in fp64
        exact = float(runner.last["window_cnt"].double().sum().item()) * (world if runner.scaling == "weak" else 1)
        line["aligned_msd_pairs_per_s"] = {
            "value": exact / (ms * 1e-3), "unit": "pairs/s",
            "what": "exact fp64 aligned MSDs per second: the window pairs refit in fp64 (those that reach s, z and "
                    "the gradients); every other (frame, landmark) pair is excluded by the certified one-term "
                    "screen bound or the metric pruning, not computed",
            "screened_pairs_per_s": units * runner.L / (ms * 1e-3)}
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, runner, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _cpu_fn(cfg, wl):
    from oracle import c_oracle as C

    if cfg == 0:
        return lambda fr: C.path_cv_exact(fr, wl.landmarks, wl.lam, wl.q)
    if cfg in (1, 3):
        return lambda fr: C.close_replay(fr, wl.landmarks, wl.lam, wl.eps, wl.q)
    if cfg == 2:
        return lambda fr: C.msd_matrix(fr, wl.landmarks[:256])
    return lambda fr: C.path_cv_exact(fr, wl.landmarks, wl.lam, wl.q)


def cpu_baseline(cfg, runner, args, seconds=12.0):
    """C restatement of the reference CPU path on a bounded sample (all host cores)."""
    from oracle import c_oracle as C

    threads = C.max_threads()
    wl = runner.wl
    if cfg in (0, 1):
        frames = wl.frames
    elif cfg == 3:
        frames = wl.frames[0].double().cpu().numpy()  # walker 0's trajectory (sequential chain)
    else:
        frames = wl.frames[:256].double().cpu().numpy()
    fn = _cpu_fn(cfg, wl)
    # a first small sample, then one sized to ~`seconds` of CPU work; oracle/c runs the
    # (frame, landmark) fits in parallel over pairs, so every thread is busy either way
    k = min(frames.shape[0], 2 if cfg in (2, 4) else (16 if cfg == 3 else 64))
    t0 = time.perf_counter()
    fn(frames[:k])
    dt = time.perf_counter() - t0
    k2 = int(min(frames.shape[0], max(k, k * seconds / max(dt, 1e-6))))
    if k2 > k:
        t0 = time.perf_counter()
        fn(frames[:k2])
        dt = time.perf_counter() - t0
    else:
        k2 = k
    if cfg == 2:
        value, unit = k2 * 256 / dt, "pairs/s"
        sample = f"{k2} frames x 256 landmarks of config2 (exact kearsley fits)"
    else:
        value, unit = k2 / dt, "frames/s"
        sample = f"{k2} frames of the {CONFIG_NAMES[cfg].split(':')[0]} workload"
    return {"value": value, "unit": unit, "cores": threads, "kind": "port",
            "sample": sample + f", oracle/c (C restatement of geometry.py + SPEC msd/colvar), OpenMP {threads} threads"}


def run_reference(args, rank, world):
    """Reference arm: the C port of the reference CPU path, rank 0 only, all host cores."""
    if rank != 0:
        return
    from oracle import c_oracle as C
    from paper_1801_02362_b200 import synth

    cfg = args.config
    threads = C.max_threads()
    if cfg in (0, 1):
        wl = synth.config0() if cfg == 0 else synth.config1()
        sample = wl.frames if cfg == 0 else wl.frames[:1000]
        L, n = wl.landmarks.shape[0], wl.frames.shape[1]
    elif cfg == 3:
        wl = synth.walkers_device(3, 256, 1000, 2500, 2048, "cpu", 0, 1)
        sample = wl.frames[0, :60].double().numpy()
        L, n = 2048, 2500
    else:
        shp = CONFIG_SHAPES[cfg]
        rng_frames = 16  # >= the host's cores worth of frames per step (fits run in parallel over pairs)
        wl = _host_sample(cfg, rng_frames)
        sample = wl.frames
        L, n = wl.landmarks.shape[0], shp["N"]
    fn = _cpu_fn(cfg, wl)
    for _ in range(args.warmup):
        fn(sample[: max(1, len(sample) // 4)])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn(sample)
    dt = (time.perf_counter() - t0) / args.steps
    if cfg == 2:
        v, unit, metric = len(sample) * 256 / dt, "pairs/s", "aligned-MSD pairs/s"
    else:
        v, unit, metric = len(sample) / dt, "frames/s", "path-CV frames/s"
    line = {
        "impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py)",
        "config": {"workload": CONFIG_NAMES[cfg], "frames_per_step": len(sample), "landmarks": L, "atoms": n},
        "cpu_baseline": {"value": v, "unit": unit, "cores": threads, "kind": "port",
                         "sample": f"{len(sample)} frames per step" + (" x 256 landmarks" if cfg == 2 else "") +
                                   f", oracle/c OpenMP {threads} threads"},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _host_sample(cfg, nframes):
    """A few frames of config 2/4 on the host (numpy generator path) for the CPU arm."""
    from paper_1801_02362_b200 import synth

    shp = CONFIG_SHAPES[cfg]
    rng = np.random.default_rng(shp["seed"])
    ends = rng.normal(0.0, 0.3, size=(shp["n_endpoints"], shp["N"], 3))
    lms = synth.make_landmarks(rng, ends, shp["L"], dtype=np.float32)
    fr, _, _ = synth._interp_frames(rng, ends, shp["L"], nframes, shp["N"], 1e-3, 0.5, np.float32)
    wl = synth._finish(f"config{cfg}-sample", fr.astype(np.float64), lms)
    return wl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=int(os.environ.get("MC_BENCH_CONFIG", 4)))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=0, help="override T (configs 2/4) for quick runs")
    ap.add_argument("--walkers", type=int, default=0, help="override W (config 3) for quick runs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline leg")
    ap.add_argument("--shard", default="frames", choices=["frames", "landmarks", "landmarks-allgather",
                                                          "landmarks-routed", "landmarks-replicated"],
                    help="multi-GPU split of config 4: frames (strong, no collective) or landmarks (strong, NCCL; "
                         "two-phase with a routed screen (default), two-phase with the screening operand "
                         "all-gathered, frame-routed, or with every frame replicated on every rank)")
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
