"""Demand traces and batched analytical re-planning.

Mirrors the trace half of the reference's ``sliceserve.workload``
(workload.py:61-167: ``DemandTrace``, ``TraceShape``, ``gen_trace``,
``predict``, CSV load/save) and the planning half of ``run_day``
(workload.py:223-311) without the discrete-event simulator, which is out of
scope (it is a sequential event loop, not planner work).  Without simulated
edge factors the day's plans depend only on the trace: bin i is planned at
the predictor's demand (mean of the last five actual bins x (1 + slack); the
first bin bootstraps from its own demand), and an infeasible bin falls back to
the plan at the highest serviceable demand, computed once per day
(workload.py:267-275).  Every bin is independent, so the whole day is one
``plan_batch`` call on the GPU (plus at most one ``max_demand``).
"""

from __future__ import annotations

import csv
import math
import statistics
from collections import deque
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import ConfigError
from .plan_types import PlannerOptions, PlanRequest, PlanResult, SearchSpace

PREDICTOR_WINDOW = 5


@dataclass(frozen=True)
class DemandTrace:
    """Mean request rate per contiguous time bin (reference workload.py:61-88)."""

    bins: tuple[tuple[int, float], ...]
    bin_s: float = 300.0

    def __post_init__(self) -> None:
        if not self.bins:
            raise ConfigError("trace must contain at least one bin")
        if self.bin_s <= 0:
            raise ConfigError("bin width must be positive")
        for pos, (idx, demand) in enumerate(self.bins):
            if idx != pos:
                raise ConfigError(
                    f"bin indices must be contiguous from 0; found {idx} at position {pos}"
                )
            if demand < 0 or not math.isfinite(demand):
                raise ConfigError(f"bin {idx}: demand must be finite and >= 0, got {demand}")

    @property
    def demands(self) -> tuple[float, ...]:
        return tuple(d for _, d in self.bins)

    def __len__(self) -> int:
        return len(self.bins)


@dataclass
class PredictorState:
    """Rolling demand history feeding the per-bin prediction (workload.py:91-98)."""

    slack: float = 0.05
    window: deque = field(default_factory=lambda: deque(maxlen=PREDICTOR_WINDOW))

    def observe(self, demand_rps: float) -> None:
        self.window.append(float(demand_rps))


def predict(state: PredictorState) -> float:
    """Mean of the recent window, padded by the slack fraction (workload.py:101-105)."""
    if not state.window:
        raise ConfigError("cannot predict demand from empty history")
    return statistics.fmean(state.window) * (1.0 + state.slack)


@dataclass(frozen=True)
class TraceShape:
    """Knobs for the synthetic diurnal demand curve (workload.py:108-124)."""

    amplitude: float = 0.5
    base: float = 1.0
    noise_sigma: float = 0.05
    bins: int = 288
    bin_s: float = 300.0

    def __post_init__(self) -> None:
        if self.bins < 1:
            raise ConfigError("trace must have at least one bin")
        if self.noise_sigma < 0:
            raise ConfigError("noise sigma must be >= 0")
        if self.base < 0 or self.amplitude < 0:
            raise ConfigError("base and amplitude must be >= 0")


def gen_trace(shape: TraceShape, scale_to_max_rps: float, seed: int) -> DemandTrace:
    """Sinusoidal day curve plus seeded noise, peak bin scaled to ``scale_to_max_rps``
    exactly; bit-identical to reference workload.py:127-143 (same numpy stream)."""
    if scale_to_max_rps < 0:
        raise ConfigError("scale-to-max must be >= 0")
    rng = np.random.default_rng(seed)
    noise = (rng.normal(0.0, shape.noise_sigma, shape.bins) if shape.noise_sigma
             else np.zeros(shape.bins))
    phase = 2.0 * math.pi * np.arange(shape.bins) / shape.bins
    raw = shape.base + shape.amplitude * np.sin(phase - math.pi / 2.0) + noise
    raw = np.maximum(raw, 0.0)
    peak = float(raw.max())
    if peak <= 0.0:
        raise ConfigError("trace shape is identically zero; cannot scale to a maximum")
    demands = [float(r / peak) * scale_to_max_rps for r in raw]
    return DemandTrace(tuple(enumerate(demands)), bin_s=shape.bin_s)


TRACE_HEADER = ("bin_index", "demand_rps")


def save_trace(path: str | Path, trace: DemandTrace) -> None:
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(TRACE_HEADER)
        for idx, demand in trace.bins:
            writer.writerow([idx, repr(demand)])


def load_trace(path: str | Path, bin_s: float = 300.0) -> DemandTrace:
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None or tuple(h.strip() for h in header) != TRACE_HEADER:
            raise ConfigError(f"{path}: expected header {','.join(TRACE_HEADER)}")
        try:
            bins = tuple((int(row[0]), float(row[1])) for row in reader if row)
        except (ValueError, IndexError) as exc:
            raise ConfigError(f"{path}: malformed trace row ({exc})") from exc
    return DemandTrace(bins, bin_s=bin_s)


def predicted_demands(trace: DemandTrace, slack: float = 0.05) -> list[float]:
    """The planning demand of every bin, as run_day computes it (workload.py:245-249)."""
    st = PredictorState(slack=slack)
    out = []
    for _, actual in trace.bins:
        out.append(predict(st) if st.window else actual * (1.0 + slack))
        st.observe(actual)
    return out


@dataclass(frozen=True)
class DayPlan:
    """The plan serving one bin (run_day's BinResult without the simulator report)."""

    bin_index: int
    demand_rps: float
    predicted_rps: float
    plan: PlanResult
    used_fallback: bool


def plan_day(app, profile, trace: DemandTrace, slice_budget: int, space: SearchSpace,
             slack: float = 0.05, options: PlannerOptions | None = None,
             device: int | None = None, part: tuple[int, int] | None = None) -> list[DayPlan]:
    """run_day's planning decisions for a whole trace in one GPU batch.

    Same plans as the reference loop with no simulated factor history
    (factor_overrides None): ``plan()`` at each bin's predicted demand, and the
    memoised ``max_demand`` plan for bins whose prediction is infeasible.
    ``part = (lo, hi)`` plans only bins lo..hi-1 (the predictions still run over
    the whole trace: each depends on the bins before it) -- one rank's share.
    """
    from . import planner

    preds = predicted_demands(trace, slack)
    lo, hi = part if part is not None else (0, len(preds))
    bins = trace.bins[lo:hi]
    preds = preds[lo:hi]
    reqs = [PlanRequest(d, slice_budget, space, slack) for d in preds]
    results = planner.plan_batch(app, profile, reqs, options, device=device) if reqs else []
    fallback = None
    out = []
    for (idx, actual), pred, res in zip(bins, preds, results):
        used = False
        if not res.feasible:
            if fallback is None:
                fallback = planner.max_demand(app, profile, slice_budget, space, slack, options).plan
            res, used = fallback, True
        out.append(DayPlan(idx, actual, pred, res, used))
    return out


def plan_days(app, profile, traces: Sequence[DemandTrace], slice_budget: int,
              spaces: Sequence[SearchSpace], slack: float = 0.05,
              options: PlannerOptions | None = None) -> dict:
    """configs[4]'s ablation sweep: plan_day for every (trace, space) pair."""
    return {(i, sp.label): plan_day(app, profile, tr, slice_budget, sp, slack, options)
            for i, tr in enumerate(traces) for sp in spaces}
