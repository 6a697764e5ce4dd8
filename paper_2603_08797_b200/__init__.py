"""B200-native (sm_100a) drop-in for JigsawServe's allocation-planner hot path.

``paper_2603_08797_b200.planner`` mirrors the reference ``sliceserve.planner``
API; the candidate enumeration, evaluation, SLO filtering, argmax and the
max-demand sweep run in hand-written CUDA (libjsv.so, include/jsv.h).
"""

from .errors import ConfigError, GeometryError, GraphError, NativeError, ProfileError, SliceServeError
from .model import (
    AppSpec,
    ModelVariant,
    Task,
    TaskGraph,
    app_from_dict,
    load_app,
    propagate_demand,
    system_accuracy,
)
from .plan_types import (
    ALL_SPACES,
    Configuration,
    ConstraintVerdict,
    MaxDemandResult,
    PlannerOptions,
    PlanRequest,
    PlanResult,
    SearchSpace,
    SolverStats,
    plan_result_to_dict,
)
from .profiles import (
    ProfileEntry,
    ProfileTable,
    SegmentType,
    SynthKnobs,
    load_knobs,
    load_profile,
    save_profile,
    synth_profile,
)

__all__ = [
    "SliceServeError", "GraphError", "ConfigError", "ProfileError", "GeometryError", "NativeError",
    "AppSpec", "ModelVariant", "Task", "TaskGraph", "app_from_dict", "load_app",
    "propagate_demand", "system_accuracy",
    "ProfileEntry", "ProfileTable", "SegmentType", "SynthKnobs", "load_knobs", "load_profile",
    "save_profile", "synth_profile",
    "ALL_SPACES", "Configuration", "ConstraintVerdict", "MaxDemandResult", "PlannerOptions",
    "PlanRequest", "PlanResult", "SearchSpace", "SolverStats", "plan_result_to_dict",
    "plan", "max_demand", "derive_configuration", "validate_configuration",
]


def __getattr__(name):
    # the planner entry points load libjsv.so lazily on first use
    if name in ("plan", "max_demand", "derive_configuration", "validate_configuration",
                "plan_uninformed", "plan_batch", "max_demand_grid"):
        from . import planner
        return getattr(planner, name)
    raise AttributeError(name)
