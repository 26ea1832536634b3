"""B200-native plan-search engine for Saturn (arXiv 2311.02840).

The Solver's joint search over the Trial Runner's profile table -- per-job
parallelism technique and GPU count plus a job order, each candidate
list-scheduled to its makespan -- runs as hand-written sm_100a CUDA
(csrc/sat_engine.cu) behind a C ABI (include/saturn_engine.h).  This package
is the host side: the reference's domain/profiling API mirror, table
marshalling, and the planners (Saturn, re-solve, Random, Optimus, Current
Practice) that all evaluate candidates on the device.
"""

from . import errors
from .domain import (ClusterSpec, JobSpec, NodeSpec, Plan, PlanEntry, RunConfig, RunningContext,
                     TechniqueSpec, Workload, check_plan, feasible_configs, memory_feasible,
                     validate_workload)
from .problem import SearchProblem, SolveOptions, build_problem, choose_delta
from .profiling import (ProfileTable, SyntheticExecutor, TableExecutor, build_profile_table,
                        estimate_runtime, feasible_entries)

__all__ = [
    "errors", "ClusterSpec", "JobSpec", "NodeSpec", "Plan", "PlanEntry", "RunConfig", "RunningContext",
    "TechniqueSpec", "Workload", "check_plan", "feasible_configs", "memory_feasible", "validate_workload",
    "SearchProblem", "SolveOptions", "build_problem", "choose_delta", "ProfileTable", "SyntheticExecutor",
    "TableExecutor", "build_profile_table", "estimate_runtime", "feasible_entries",
    "plan_saturn", "resolve", "plan_random", "plan_random_best", "plan_optimus", "plan_current_practice",
    "solve",
]


def __getattr__(name):
    # planners import torch lazily so the host-side API stays importable without it
    if name in ("plan_saturn", "resolve", "plan_random", "plan_random_best", "plan_optimus",
                "plan_current_practice", "solve", "optimus_marginal_gain", "evaluate_fixed"):
        from . import planners
        return getattr(planners, name)
    raise AttributeError(name)
