"""The paper's analytical performance model (SPEC [MODULE] perf, SPEC.md:350-412;
PAPER §Theoretical Speedup, Eq. 7): expensive-MSD computations per step of the
original and close-structure methods, the acceleration condition, Amdahl's law,
and the identity check of a toy run's counters against the model.

Pure host functions (no device work): the model is what the device counters of
``toysim`` / ``msd.CloseStructureState`` implement by construction.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError


@dataclass(frozen=True)
class CostModel:
    """N references, neighbour list of M refreshed every L steps (M = 0, L = 1: no
    neighbour list), K mean steps between close-structure reassignments."""

    N: int
    M: int = 0
    L: int = 1
    K: float = 1.0

    def __post_init__(self):
        if self.N < 1 or not (0 <= self.M <= self.N) or self.L < 1 or not (self.K > 0):
            raise ConfigError("N >= 1, 0 <= M <= N, L >= 1, K > 0 (SPEC.md:356)")


def original_cost(m: CostModel) -> float:
    """M + (N - M) / L expensive MSDs per step (PAPER §Theoretical Speedup)."""
    return m.M + (m.N - m.M) / m.L


def close_cost(m: CostModel) -> float:
    """1 + N / K: the x<->y fit every step plus a full refit every K steps on average."""
    return 1.0 + m.N / m.K


def msd_speedup(m: CostModel) -> float:
    return original_cost(m) / close_cost(m)


def accelerates(m: CostModel) -> bool:
    """Strict: M + (N - M)/L > 1 + N/K."""
    return original_cost(m) > close_cost(m)


def amdahl(p: float, s: float) -> float:
    """Eq. 7: S = 1 / ((1 - p) + p / s), p in [0, 1] the accelerated fraction, s > 0."""
    if not (0.0 <= p <= 1.0):
        raise ConfigError("p must lie in [0, 1]")
    if not (s > 0):
        raise ConfigError("s must be > 0 (SPEC.md:386)")
    return 1.0 / ((1.0 - p) + p / s)


def measured_vs_model(report, N: int, M: int | None = None, L: int = 1, updates: int = 0):
    """Identity check of a toy run (toysim.RunReport) against the model:
    close mode -> measured expensive per step == 1 + N reassign / steps; original mode
    -> M + (N - M) updates / steps (no neighbour list: N).  Returns a dict with the
    measured and model values and their difference (exactly 0 by construction)."""
    steps = int(report.steps)
    if steps < 1:
        raise ConfigError("report has no steps")
    measured = report.expensive_count / steps
    if report.mode == "close":
        model = 1.0 + N * report.reassign_count / steps
    elif report.mode == "original":
        m = N if M is None else M
        model = m + (N - m) * (updates / steps)
    else:
        raise ConfigError(f"mode {report.mode!r} has no cost model")
    return {"mode": report.mode, "measured": measured, "model": model, "difference": measured - model,
            "measured_K": report.measured_K}


def model_report(N: int, M: int = 0, L: int = 1, K: float = 1.0, p: float | None = None) -> dict:
    """The numbers of the SPEC's `model` command (acceptance criteria 1-2):
    original cost, close cost, MSD speed-up, acceleration flag and, given the
    accelerated fraction p, the Amdahl whole-run projection."""
    m = CostModel(N, M, L, K)
    out = {"original_cost": original_cost(m), "close_cost": close_cost(m), "msd_speedup": msd_speedup(m),
           "accelerates": accelerates(m)}
    if p is not None:
        out["amdahl"] = amdahl(p, out["msd_speedup"])
    return out
