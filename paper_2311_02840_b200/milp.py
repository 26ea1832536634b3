"""The reference's ``jointsched.milp`` entry points, answered by the B200 engine.

``pkg/src/jointsched/milp/__init__.py:3-6`` declares a time-indexed MILP package whose
modules are missing.  The names a caller of the solver uses are
provided here with the SPEC's contracts, so ``jointsched.milp`` can be pointed at this
module:

    build_milp(table, jobs, cluster, delta, running_context=None) -> MilpInstance
    choose_delta(...)
    branch_and_bound(instance, opts=None) -> MilpSolution
    brute_force_schedule(instance) -> MilpSolution
    decode_plan(instance, solution) -> Plan

The instance is the engine's dense problem (options, grid durations d = ceil(T/delta),
horizon K) rather than explicit x[j,c,n,i] columns: ``branch_and_bound`` is the GPU
bound-and-prune search (exact; Feasible only when the engine must sample), and
``brute_force_schedule`` the full scan of the candidate space.  The LP machinery
(``solve_bounded_lp``, ``solve_lp_relaxation``, ``dump_instance`` / ``parse_instance``)
has no counterpart: the search does not relax anything.

Ties: the winner is the lowest candidate index among equal makespans (SURVEY.md A1,
the lexicographic rule of SPEC.md:249 applied to (options, order)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from . import errors as E
from .problem import K_MAX_DEFAULT, TIME_GRID, SearchProblem, SolveOptions, build_problem, choose_delta

__all__ = ["BnbOptions", "MilpInstance", "MilpSolution", "branch_and_bound", "brute_force_schedule",
           "build_milp", "choose_delta", "decode_plan"]


@dataclass
class MilpInstance:
    """interval length delta, horizon K, per-option durations d[j, c]."""

    problem: SearchProblem
    workload: object
    table: object
    running_context: object = None
    options: SolveOptions = field(default_factory=SolveOptions)
    min_runtime_sum: float = 0.0     # sum_j min over all feasible entries of T[j, c] (before pruning)

    @property
    def delta(self) -> float:
        return self.problem.delta

    @property
    def horizon(self) -> int:
        """K = ceil(sum_j min_c T[j, c] / delta): the sequential-best schedule fits."""
        return math.ceil(self.min_runtime_sum / self.problem.delta)

    def durations(self) -> dict:
        """(job id, technique, g) -> d[j, c] grid intervals (max over eligible nodes)."""
        p = self.problem
        out = {}
        for j, jid in enumerate(p.job_ids):
            for o in range(int(p.radix[j])):
                cfg = p.options[j][o][0]
                out[(jid, cfg.technique, cfg.gpus)] = int(p.dur_i32[j, o].max())
        return out


@dataclass
class BnbOptions:
    """gaps are met exactly (the search is exact); node_limit caps the exact
    search -- beyond it the engine samples and reports Feasible."""

    abs_gap: float = 1e-6
    rel_gap: float = 1e-6
    node_limit: int | None = None


@dataclass
class MilpSolution:
    """job -> (c, n, i), objective seconds, status, nodes explored."""

    assignment: dict
    objective: float
    status: str                      # "Optimal" | "Feasible(gap)" | "Infeasible"
    node_count: int
    plan: object = None
    search: object = None


def build_milp(table, jobs, cluster=None, delta: float | None = None, running_context=None, *, techniques=None,
               k_max: int = K_MAX_DEFAULT) -> MilpInstance:
    """SPEC.md:192-196.  ``delta=None`` chooses it per SPEC.md:246; an explicit delta whose
    horizon exceeds ``k_max`` raises HorizonOverflow (errors.py:77-81)."""
    from .planners import _as_workload

    workload = _as_workload(jobs, cluster, techniques)
    opts = SolveOptions(delta=delta, k_max=k_max, time_mode=TIME_GRID)
    prob = build_problem(table, workload, opts, running_context)
    full = build_problem(table, workload, SolveOptions(delta=prob.delta, k_max=1 << 30, prune=False),
                         running_context)
    total = 0.0
    for j in range(full.J):                                    # job-id order, left to right
        total += min(float(full.runtime[j, o, n]) for o in range(int(full.radix[j])) for n in range(full.N)
                     if (int(full.node_mask[j, o]) >> n) & 1)
    return MilpInstance(problem=prob, workload=workload, table=table, running_context=running_context,
                        options=opts, min_runtime_sum=total)


def _solution(inst: MilpInstance, sol, status: str, node_count: int) -> MilpSolution:
    p = inst.problem
    assignment = {}
    for j, jid in enumerate(p.job_ids):
        e = sol.plan.entries[jid]
        c = p.option_src[j][sol.options[j]]                    # index into feasible_entries
        assignment[jid] = (c, e.node, int(round(e.start_time / p.delta)))
    return MilpSolution(assignment=assignment, objective=sol.plan.predicted_makespan, status=status,
                        node_count=node_count, plan=sol.plan, search=sol.search)


def branch_and_bound(inst: MilpInstance, opts: BnbOptions | None = None, *, group=None, device=None) -> MilpSolution:
    """SPEC.md:210-214 on the GPU: exact bound-and-prune where it applies (one node), the full
    scan otherwise while the space is enumerable, sampled (status Feasible) beyond."""
    from .planners import solve_problem

    opts = opts or BnbOptions()
    so = SolveOptions(**{**inst.options.__dict__})
    if opts.node_limit is not None:
        so.max_exhaustive = min(so.max_exhaustive, int(opts.node_limit))
        so.max_bnb = min(so.max_bnb, int(opts.node_limit))
    sol = solve_problem(inst.problem, inst.workload, so, inst.running_context, group=group, device=device)
    st = sol.search.stats or {}
    nodes = int(st.get("pair_nodes", 0)) + int(st.get("pruned_tasks", 0)) if st else int(sol.search.evaluated)
    status = "Optimal" if sol.status == "Optimal" else "Feasible(gap)"
    return _solution(inst, sol, status, nodes)


def brute_force_schedule(inst: MilpInstance, *, group=None, device=None) -> MilpSolution:
    """exact optimum by enumerating the whole candidate space (GPU full scan)."""
    from .planners import solve_problem

    so = SolveOptions(**{**inst.options.__dict__, "kernel": "tree", "search": "exhaustive"})
    if not (inst.problem.N == 1 and inst.problem.J >= 3):
        so.kernel = "index"
    sol = solve_problem(inst.problem, inst.workload, so, inst.running_context, group=group, device=device)
    return _solution(inst, sol, "Optimal", int(sol.search.evaluated))


def decode_plan(inst: MilpInstance, solution: MilpSolution):
    """start = i * delta, predicted makespan = objective."""
    if solution.status == "Infeasible":
        raise E.PlanFailure("no solution to decode")
    if solution.plan is not None:
        return solution.plan
    from .planners import _types_for

    Plan, PlanEntry, RunConfig = _types_for(inst.workload)
    p = inst.problem
    entries = {}
    for j, jid in enumerate(p.job_ids):
        c, node, i = solution.assignment[jid]
        o = p.option_src[j].index(c)
        cfg = p.options[j][o][0]
        entries[jid] = PlanEntry(config=RunConfig(technique=cfg.technique, gpus=cfg.gpus), node=node,
                                 start_time=i * p.delta)
    return Plan(entries=entries, predicted_makespan=solution.objective)
