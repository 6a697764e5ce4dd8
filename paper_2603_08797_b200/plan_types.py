"""Planner request/result types -- the data half of the drop-in boundary.

Field names, defaults and semantics follow the reference planner
(reference pkg/src/sliceserve/planner.py:60-149 for the request side,
216-240 / 321-327 / 686-706 / 1116-1122 / 1181-1188 for the results) so a
caller can swap ``sliceserve.planner`` for ``paper_2603_08797_b200.planner``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Iterable, Mapping

from .errors import ConfigError
from .profiles import Key

__all__ = [
    "SearchSpace",
    "ALL_SPACES",
    "PlanRequest",
    "PlannerOptions",
    "Configuration",
    "ConstraintVerdict",
    "SolverStats",
    "PlanResult",
    "MaxDemandResult",
    "OracleCaps",
    "BINDING_PRIORITY",
    "binding_from_kills",
    "binding_from_verdicts",
    "plan_result_to_dict",
]


@dataclass(frozen=True)
class SearchSpace:
    """A/S/T feature toggles (reference planner.py:60-104)."""

    accuracy_scaling: bool = False
    spatial_partitioning: bool = False
    task_graph_informed: bool = False

    @property
    def label(self) -> str:
        on = [c for c, f in (("A", self.accuracy_scaling), ("S", self.spatial_partitioning),
                             ("T", self.task_graph_informed)) if f]
        return "+".join(on) or "Unopt"

    @classmethod
    def from_label(cls, label: str) -> "SearchSpace":
        if label == "Unopt":
            return cls()
        parts = label.split("+")
        if not parts or not set(parts) <= {"A", "S", "T"} or len(set(parts)) != len(parts):
            raise ConfigError(f"unknown search space label {label!r}")
        return cls("A" in parts, "S" in parts, "T" in parts)

    def is_subset(self, other: "SearchSpace") -> bool:
        mine = (self.accuracy_scaling, self.spatial_partitioning, self.task_graph_informed)
        theirs = (other.accuracy_scaling, other.spatial_partitioning, other.task_graph_informed)
        return all(a <= b for a, b in zip(mine, theirs))


# sweep/CSV row order: Unopt, T, A, A+T, S, S+T, A+S, A+S+T (reference planner.py:107-119)
ALL_SPACES: tuple[SearchSpace, ...] = tuple(
    SearchSpace(a, s, t)
    for s in (False, True)
    for a in (False, True)
    for t in (False, True)
)


@dataclass(frozen=True)
class PlanRequest:
    demand_rps: float
    slice_budget: int
    space: SearchSpace = SearchSpace(True, True, True)
    slack: float = 0.05
    factor_overrides: Mapping[tuple[str, str], float] | None = None

    def __post_init__(self) -> None:
        if not math.isfinite(self.demand_rps) or self.demand_rps < 0:
            raise ConfigError(f"demand must be finite and non-negative, got {self.demand_rps}")
        if self.slice_budget < 0:
            raise ConfigError(f"slice budget must be non-negative, got {self.slice_budget}")
        if self.slack < 0:
            raise ConfigError(f"slack must be non-negative, got {self.slack}")
        for edge, val in (self.factor_overrides or {}).items():
            if val < 0:
                raise ConfigError(f"factor override for {edge} is negative")


@dataclass(frozen=True)
class PlannerOptions:
    pareto_width: int = 512
    exhaustive_limit: int = 2_000
    eps: float = 1e-9
    mix_fractions: tuple[float, ...] = (0.25, 0.5, 0.75)
    feasible_only: bool = False


@dataclass(frozen=True, eq=True)
class Configuration:
    """A full instance-count assignment and every quantity derived from it."""

    m: tuple[tuple[Key, int], ...]
    entry_demand_rps: float
    latency_ms: dict[str, float]
    capacity_rps: dict[str, float]
    demand_rps: dict[str, float]
    slices: dict[str, int]
    accuracy: dict[str, float]
    fanout: dict[tuple[str, str], float]
    hput: dict[Key, float]
    path_accuracy: dict[tuple[str, ...], float]
    total_slices: int
    a_obj: float
    a_max: float
    objective: float
    structurally_infeasible: tuple[str, ...]

    __hash__ = None  # type: ignore[assignment]

    @property
    def active_keys(self) -> tuple[Key, ...]:
        return tuple(k for k, _ in self.m)


@dataclass(frozen=True)
class ConstraintVerdict:
    name: str  # latency | throughput | resources | accuracy | coverage
    subject: str
    passed: bool
    margin: float


@dataclass(frozen=True)
class SolverStats:
    nodes: int
    wall_ms: float
    pool_sizes: dict[str, int] = field(default_factory=dict)
    truncated_tasks: tuple[str, ...] = ()

    __hash__ = None  # type: ignore[assignment]


@dataclass(frozen=True)
class PlanResult:
    feasible: bool
    config: Configuration | None
    objective: float | None
    a_max: float
    binding_constraint: str | None
    verdicts: tuple[ConstraintVerdict, ...]
    stats: SolverStats

    __hash__ = None  # type: ignore[assignment]


@dataclass(frozen=True)
class MaxDemandResult:
    demand_rps: float
    plan: PlanResult
    probes: int

    __hash__ = None  # type: ignore[assignment]


@dataclass(frozen=True)
class OracleCaps:
    max_tasks: int = 2
    max_variants: int = 2
    max_segments: int = 2
    max_batches: int = 2
    max_count: int = 3
    max_assignments: int = 2_000_000


# tie order when several constraints block equally (reference planner.py:709)
BINDING_PRIORITY = ("throughput", "latency", "resources", "accuracy", "coverage")


def binding_from_kills(kills: Mapping[str, int]) -> str:
    """Most kills wins, ties by BINDING_PRIORITY; none -> throughput (planner.py:712-714)."""
    best = None
    for name in BINDING_PRIORITY:
        if best is None or kills.get(name, 0) > kills.get(best, 0):
            best = name
    return best if kills.get(best, 0) else "throughput"


def binding_from_verdicts(verdicts: Iterable[ConstraintVerdict]) -> str | None:
    """First failed constraint in priority order; coverage reads as throughput (717-725)."""
    failed = [v for v in verdicts if not v.passed]
    if not failed:
        return None
    names = {v.name for v in failed}
    for name in BINDING_PRIORITY:
        if name in names:
            return "throughput" if name == "coverage" else name
    return failed[0].name


def plan_result_to_dict(result: PlanResult) -> dict:
    """JSON view, wall time omitted (reference planner.py:1278-1331)."""
    doc: dict = {
        "feasible": result.feasible,
        "objective": result.objective,
        "a_max": result.a_max,
        "binding_constraint": result.binding_constraint,
        "stats": {
            "nodes": result.stats.nodes,
            "pool_sizes": dict(sorted(result.stats.pool_sizes.items())),
            "truncated_tasks": list(result.stats.truncated_tasks),
        },
        "verdicts": [
            {"name": v.name, "subject": v.subject, "passed": v.passed, "margin": v.margin}
            for v in result.verdicts
        ],
    }
    c = result.config
    if c is None:
        doc["config"] = None
        return doc
    doc["config"] = {
        "m": [
            {"task": k[0], "variant": k[1], "mig": k[2].mig, "mps": k[2].mps, "batch": k[3],
             "count": n}
            for k, n in c.m
        ],
        "entry_demand_rps": c.entry_demand_rps,
        "latency_ms": dict(sorted(c.latency_ms.items())),
        "capacity_rps": dict(sorted(c.capacity_rps.items())),
        "demand_rps": dict(sorted(c.demand_rps.items())),
        "slices": dict(sorted(c.slices.items())),
        "accuracy": dict(sorted(c.accuracy.items())),
        "fanout": [{"src": e[0], "dst": e[1], "value": v} for e, v in sorted(c.fanout.items())],
        "path_accuracy": [
            {"path": list(p), "value": v} for p, v in sorted(c.path_accuracy.items())
        ],
        "total_slices": c.total_slices,
        "a_obj": c.a_obj,
        "objective": c.objective,
    }
    return doc
