"""Planners on the B200 engine -- the reference's Solver / baseline API.

  plan_saturn(table, jobs, cluster, delta_opts, running_context)
  resolve(...)          = plan_saturn with a RunningContext
  plan_random(table, jobs, cluster, seed)
  plan_random_best(...) best of a batch of seeds (Random over >=1e9 seeds)
  optimus_marginal_gain / plan_optimus
  plan_current_practice

``jobs`` may be a workload (anything with ``jobs``, ``cluster`` and
``techniques``) or a job list with ``cluster`` and ``techniques=`` given.  The
objects may be this package's dataclasses or the reference's pydantic models;
the returned Plan is of the caller's type family.

Every candidate plan is list-scheduled on the GPU; the host only marshals the
table (problem.py), runs the O(J x G) Optimus allocator, and turns the
engine's winner into a Plan.
"""

from __future__ import annotations

import sys
from dataclasses import dataclass, field

import numpy as np

from . import domain as D
from . import errors as E
from .engine import SRC_EXPLICIT, SRC_INDEX, SRC_SEED, Engine, NativeProblem, SearchResult
from .problem import TIME_GRID, SearchProblem, SolveOptions, build_problem

_ENGINES: dict = {}


def get_engine(device=None) -> Engine:
    import torch

    idx = torch.cuda.current_device() if device is None else (torch.device(device).index or 0)
    eng = _ENGINES.get(idx)
    if eng is None:
        eng = _ENGINES[idx] = Engine(idx)
    return eng


@dataclass
class _WorkloadView:
    """The SPEC.md:276 call shape ``(table, jobs, cluster, techniques=...)`` seen as a workload:
    the attributes plus the ``job(id)`` / ``technique(name)`` lookups a ``Workload`` offers
    (core.py:132-142), which ``check_plan`` (core.py:271) and the simulator use."""

    jobs: tuple
    cluster: object
    techniques: tuple

    def job(self, job_id: str):
        for j in self.jobs:
            if j.id == job_id:
                return j
        raise KeyError(job_id)

    def technique(self, name: str):
        for t in self.techniques:
            if t.name == name:
                return t
        raise KeyError(name)


def _as_workload(jobs, cluster=None, techniques=None):
    if hasattr(jobs, "jobs") and hasattr(jobs, "cluster"):
        return jobs
    if cluster is None or techniques is None:
        raise E.InvariantViolation("workload", "pass a workload, or jobs with cluster and techniques")
    return _WorkloadView(tuple(jobs), cluster, tuple(techniques))


def _family(workload):
    """The module defining the caller's domain objects (the reference's ``jointsched.core`` for
    its pydantic models, ``domain`` for this package's dataclasses)."""
    probe = workload.jobs[0] if workload.jobs else workload
    return sys.modules.get(type(probe).__module__)


def _types_for(workload):
    """(Plan, PlanEntry, RunConfig) classes of the caller's domain family."""
    mod = _family(workload)
    if mod is not None and all(hasattr(mod, n) for n in ("Plan", "PlanEntry", "RunConfig")):
        return mod.Plan, mod.PlanEntry, mod.RunConfig
    return D.Plan, D.PlanEntry, D.RunConfig


def _validator_for(workload):
    """The caller's own plan validator: ``check_plan`` of the module that defines its domain
    objects (core.py:254-287 for reference objects), else this package's ``domain.check_plan``."""
    mod = _family(workload)
    fn = getattr(mod, "check_plan", None) if mod is not None else None
    return fn if callable(fn) else D.check_plan


def _opts(delta_opts) -> SolveOptions:
    if delta_opts is None:
        return SolveOptions()
    if isinstance(delta_opts, SolveOptions):
        return delta_opts
    if isinstance(delta_opts, dict):
        return SolveOptions(**delta_opts)
    if isinstance(delta_opts, (int, float)):
        return SolveOptions(delta=float(delta_opts))
    raise E.InvariantViolation("delta_opts", f"unsupported {type(delta_opts).__name__}")


@dataclass
class Solution:
    """A plan plus how it was found (the reference's MilpSolution analogue)."""

    plan: object
    status: str                 # "Optimal" (space exhausted, or makespan == lower bound), "Sampled" or
                                # "Local" (heuristic, see `gap`)
    makespan: float             # grid intervals or seconds
    objective: float            # seconds (= plan.predicted_makespan)
    problem: SearchProblem
    search: SearchResult | None
    options: list               # option digit per job (problem's job axis)
    order: list                 # submission order (job axis indices)
    runtimes: dict = field(default_factory=dict)   # job id -> seconds of the chosen option/node
    lower_bound: float | None = None               # makespan lower bound (same unit as makespan)
    cursor: object = None                          # resumable solves: the search cursor (resume.py)

    @property
    def gap(self) -> float:
        """Relative optimality gap (0 when proven optimal)."""
        if self.status == "Optimal" or not self.lower_bound:
            return 0.0
        return max(0.0, (self.makespan - self.lower_bound) / self.lower_bound)


def _decode(engine: Engine, prob: SearchProblem, nprob: NativeProblem, workload, source: int, seed: int,
            ident=None, explicit=None):
    """Replay candidates on the device (one launch, one read-back); build their Plans.
    One candidate (``ident`` or a 1-D ``explicit`` row) -> one tuple; a 2-D ``explicit``
    batch -> a list of tuples, row by row."""
    batch = explicit is not None and np.ndim(explicit) == 2
    schedule = engine.schedule(nprob, source, seed, ids=None if ident is None else [ident],
                               explicit=None if explicit is None else np.atleast_2d(explicit))
    out = [_plan_of(prob, workload, schedule, r) for r in range(len(schedule[3]))]
    return out if batch else out[0]


def _plan_of(prob: SearchProblem, workload, schedule, r: int):
    opt, node, start, ms = schedule
    Plan, PlanEntry, RunConfig = _types_for(workload)
    grid = prob.time_mode == TIME_GRID
    scale = prob.delta if grid else 1.0
    entries, runtimes = {}, {}
    for j, job_id in enumerate(prob.job_ids):
        o, n = int(opt[r, j]), int(node[r, j])
        cfg = prob.options[j][o][0]
        s = float(start[r, j]) * scale
        entries[job_id] = PlanEntry(config=RunConfig(technique=cfg.technique, gpus=cfg.gpus),
                                    node=prob.node_ids[n], start_time=s)
        runtimes[job_id] = float(prob.runtime[j, o, n])
    predicted = float(ms[r]) * scale
    plan = Plan(entries=entries, predicted_makespan=predicted)
    return plan, [int(x) for x in opt[r]], float(ms[r]), runtimes


class _nvtx:
    """NVTX range around a host stage of a solve (visible in Nsight timelines next to the
    library's own sat_* ranges); a no-op where torch's NVTX binding is unavailable."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        try:
            import torch

            torch.cuda.nvtx.range_push(self.name)
            self.on = True
        except Exception:  # noqa: BLE001
            self.on = False
        return self

    def __exit__(self, *exc):
        if self.on:
            import torch

            torch.cuda.nvtx.range_pop()


def solve(table, jobs, cluster=None, delta_opts=None, running_context=None, *, techniques=None,
          group=None, device=None, validate: bool = True, checkpoint=None,
          time_budget_s: float | None = None) -> Solution:
    """Solver.solve / re-solve on the engine (build -> search -> decode -> check).

    ``checkpoint`` (a file path) and/or ``time_budget_s``: run the exact search resumably
    (resume.py) -- when the budget runs out the search state is saved to ``checkpoint`` and the
    Solution has status "Suspended" (the best plan found so far, or plan None); calling again
    with the same checkpoint continues where it stopped."""
    workload = _as_workload(jobs, cluster, techniques)
    opts = _opts(delta_opts)
    with _nvtx("saturn.build_problem"):
        prob = build_problem(table, workload, opts, running_context)
    if checkpoint is not None or time_budget_s is not None:
        return _solve_resumable(prob, workload, opts, running_context, checkpoint, time_budget_s, device,
                                validate)
    with _nvtx("saturn.solve_problem"):
        return solve_problem(prob, workload, opts, running_context, group=group, device=device,
                             validate=validate)


def _solve_resumable(prob, workload, opts, running_context, checkpoint, time_budget_s, device, validate):
    import os

    from . import resume as R

    eng = get_engine(device)
    cur = None
    if checkpoint is not None and os.path.exists(checkpoint):
        cur = R.SearchCursor.load(checkpoint)
        if cur.digest != R.problem_digest(prob):
            cur = None                                  # a stale checkpoint of another problem
    if cur is None:
        cur = R.start_cursor(eng, prob, opts)
    with _nvtx("saturn.search_resumable"):
        R.run_cursor(eng, prob, cur, time_budget_s)
    found = R.cursor_result(prob, cur)
    plan, options, runtimes, ms = None, [], {}, float("inf")
    if found is not None:
        ms, index = found
        nprob = NativeProblem(prob, cur.idx_bits)
        plan, options, ms2, runtimes = _decode(eng, prob, nprob, workload, SRC_INDEX, 0, ident=index)
        if ms2 != ms:
            raise E.errors_for(workload.jobs[0]).PlanFailure(f"replay makespan {ms2} != search makespan {ms}")
    if cur.done:
        if checkpoint is not None and os.path.exists(checkpoint):
            os.remove(checkpoint)
        if plan is None:
            raise E.errors_for(workload.jobs[0]).PlanFailure("search produced no candidate")
        if validate:
            target = workload
            if running_context is not None:
                keep = set(prob.job_ids)
                target = _WorkloadView(tuple(j for j in workload.jobs if j.id in keep), workload.cluster,
                                       tuple(workload.techniques))
            _validator_for(workload)(plan, target, runtimes)
        status, lb = "Optimal", ms
    else:
        if checkpoint is not None:
            cur.save(checkpoint)
        status, lb = "Suspended", prob.lower_bound()
    order = prob.decode_index(found[1])[1] if found is not None else []
    return Solution(plan=plan, status=status, makespan=ms, lower_bound=lb,
                    objective=plan.predicted_makespan if plan is not None else float("inf"), problem=prob,
                    search=None, options=options, order=order, runtimes=runtimes,
                    cursor=cur)


def solve_problem(prob: SearchProblem, workload, opts: SolveOptions, running_context=None, *, group=None,
                  device=None, validate: bool = True) -> Solution:
    """Search -> decode -> check for an already marshalled problem (the milp facade's entry)."""
    err = E.errors_for(workload.jobs[0] if workload.jobs else workload)
    eng = get_engine(device)
    baselines = []

    def greedy_baselines(mode):
        # heuristic searches also weigh the greedy baselines as incumbents (the B&B's "initial
        # incumbent from rounding"): the plan is never worse than them.  Built on
        # the host while the search's first kernels run.
        if mode != "exhaustive":
            for builder in (optimus_allocation, current_practice_allocation):
                b_opts, b_order = builder(prob)
                baselines.append((np.array(list(b_opts) + list(b_order), dtype=np.uint8), list(b_order),
                                  builder.__name__))

    try:
        with _nvtx("saturn.search"):
            res = eng.search(prob, opts, group=group, replay=True, on_launched=greedy_baselines)
        nprob = NativeProblem(prob, res.idx_bits) if res.replay is None else None
        if res.kernel == "local":
            # replay the winning walker to get its final candidate, then schedule it explicitly
            if res.state is not None:          # recorded by the search launch
                o_, r_ = res.state
            else:
                o_, r_ = eng.local_search_state(nprob, res.source, res.seed, res.index, opts.max_rounds,
                                                stop_ms=res.stats.get("stop_ms", -1))
            explicit = np.array(list(o_) + list(r_), dtype=np.uint8)
        incumbent = None
        nexp = NativeProblem(prob, 62) if (baselines or res.kernel == "local") else None
        # device schedules (option, node, start, makespan) of the winner and the baselines; a
        # Plan is built only for the one returned (the others are compared by makespan)
        if res.kernel == "local":
            # the winner's final candidate and the baselines: one explicit batch, one launch
            sched = eng.schedule(nexp, SRC_EXPLICIT, 0, explicit=np.stack([explicit] + [b[0] for b in baselines]))
            win, rows = (sched, 0), [(sched, 1 + i) for i in range(len(baselines))]
        else:
            if res.replay is not None:          # replayed on the device behind the search
                win = (res.replay, 0)
            else:
                src = SRC_INDEX if res.exhaustive else res.source
                win = (eng.schedule(nprob, src, res.seed, ids=[res.index]), 0)
            bs = eng.schedule(nexp, SRC_EXPLICIT, 0, explicit=np.stack([b[0] for b in baselines])) if baselines else None
            rows = [(bs, i) for i in range(len(baselines))]
        ms = float(win[0][3][win[1]])
        for (bsch, r), (_, b_order, name) in zip(rows, baselines):
            b_ms = float(bsch[3][r])
            if b_ms < ms and (incumbent is None or b_ms < incumbent[0]):
                incumbent = (b_ms, (bsch, r), b_order, name)
        if incumbent is None:
            plan, options, ms, runtimes = _plan_of(prob, workload, win[0], win[1])
    except (E.SchedulerError, err.SchedulerError):      # ours or the caller family's: as raised
        raise
    except Exception as exc:  # CUDA / NCCL trouble -> PlanFailure (ReplanFailure on re-solve)
        cls = err.ReplanFailure if running_context is not None else err.PlanFailure
        raise cls(f"engine failure: {exc}") from exc
    if ms != res.makespan:
        raise err.PlanFailure(f"winner replay makespan {ms} != search makespan {res.makespan}")
    if res.exhaustive:
        order = prob.decode_index(res.index)[1]
    elif res.kernel == "local":
        order = [int(x) for x in explicit[prob.J:]]
    else:
        w_start = win[0][2][win[1]]
        order = sorted(range(prob.J), key=lambda j: (float(w_start[j]), j))
    if incumbent is not None:
        _, (bsch, r), order, source_name = incumbent
        plan, options, ms, runtimes = _plan_of(prob, workload, bsch, r)
        res.stats = {**(res.stats or {}), "incumbent": source_name}
    makespan = ms
    if validate:
        # the caller's own check_plan; a re-solve's plan covers the unfinished jobs only, so it
        # is checked against that sub-workload (runtimes carry the +rho of moved jobs)
        target = workload
        if running_context is not None:
            keep = set(prob.job_ids)
            target = _WorkloadView(tuple(j for j in workload.jobs if j.id in keep), workload.cluster,
                                   tuple(workload.techniques))
        with _nvtx("saturn.check_plan"):
            _validator_for(workload)(plan, target, runtimes)
    status = "Optimal" if res.exhaustive else ("Local" if res.kernel == "local" else "Sampled")
    if res.exhaustive:
        lb = makespan
    elif res.kernel == "local" and prob.time_mode == TIME_GRID:
        lb = res.stats["lower_bound"]   # prob.lower_bound(), computed once by the search (its stop target)
    else:
        lb = prob.lower_bound()
    if not res.exhaustive and makespan <= lb:
        status = "Optimal"          # a heuristic plan meeting the lower bound is optimal (bound proof)
    if res.proven and incumbent is None:
        # sat_search_dp: no candidate of the whole space is one interval shorter
        status, lb = "Optimal", makespan
    return Solution(plan=plan, status=status, makespan=makespan, lower_bound=lb,
                    objective=plan.predicted_makespan, problem=prob, search=res, options=options,
                    order=order, runtimes=runtimes)


def plan_saturn(table, jobs, cluster=None, delta_opts=None, running_context=None, *, techniques=None,
                group=None, device=None):
    """the joint (technique, GPU count, order) optimum as a Plan."""
    return solve(table, jobs, cluster, delta_opts, running_context, techniques=techniques,
                 group=group, device=device).plan


def resolve(table, workload, running_context, delta_opts=None, *, group=None, device=None):
    """Introspection re-solve: all unfinished jobs re-planned from now
    (start times relative to the tick); a running job pays rho on any option whose
    (technique, g, node) differs from what it holds.  Returns the Plan (use ``solve`` for the
    full Solution)."""
    return solve(table, workload, None, delta_opts, running_context, group=group, device=device).plan


# --------------------------------------------------------------------------
# Random baseline on the same engine
# --------------------------------------------------------------------------

def _baseline_problem(table, workload, opts, running_context=None) -> SearchProblem:
    """Baselines choose among ALL feasible entries (no dominance prune)."""
    o = SolveOptions(**{**opts.__dict__, "prune": False})
    return build_problem(table, workload, o, running_context)


def plan_random(table, jobs, cluster=None, seed: int = 0, delta_opts=None, running_context=None, *,
                techniques=None, device=None):
    """SplitMix64(seed): one below(|C_j|) per job in id order, then shuffle(order); list-scheduled."""
    workload = _as_workload(jobs, cluster, techniques)
    opts = _opts(delta_opts)
    prob = _baseline_problem(table, workload, opts, running_context)
    eng = get_engine(device)
    nprob = NativeProblem(prob, 62)
    plan, _, _, _ = _decode(eng, prob, nprob, workload, SRC_SEED, seed, ident=0)
    return plan


def plan_random_best(table, jobs, cluster=None, seed0: int = 0, n_seeds: int = 1 << 20, delta_opts=None, *,
                     techniques=None, group=None, device=None) -> Solution:
    """Best Random plan over seeds seed0 .. seed0+n_seeds-1 (lowest seed on ties)."""
    workload = _as_workload(jobs, cluster, techniques)
    opts = _opts(delta_opts)
    prob = _baseline_problem(table, workload, opts)
    eng = get_engine(device)
    sopts = SolveOptions(**{**opts.__dict__, "search": "sampled", "budget": n_seeds})
    res = eng.search(prob, sopts, group=group, source=SRC_SEED, seed=seed0)
    idx_bits, _ = prob.key_bits(n_seeds)
    nprob = NativeProblem(prob, idx_bits)
    plan, options, ms, runtimes = _decode(eng, prob, nprob, workload, SRC_SEED, seed0, ident=res.index)
    return Solution(plan=plan, status="Sampled", makespan=ms, objective=plan.predicted_makespan, problem=prob,
                    search=res, options=options, order=[], runtimes=runtimes)


# --------------------------------------------------------------------------
# Optimus -- host allocator, device schedule
# --------------------------------------------------------------------------

def _best_runtime_all(prob: SearchProblem, jobs=None) -> list:
    """Per job: g -> (runtime seconds, option) minimising runtime over techniques at that g
    (earliest option on ties); runtime on the job's fastest eligible node.  One array pass
    over the problem's [J, Cmax, N] tables (or the rows of ``jobs``), then a short loop per job
    over its options."""
    if jobs is None:            # whole problem: computed once per problem (arrays are final)
        hit = prob.extra.get("_best_runtime_all")
        if hit is not None:
            return [dict(d) for d in hit]
    sel = slice(None) if jobs is None else list(jobs)
    N = prob.N
    elig = ((prob.node_mask[sel, :, None] >> np.arange(N, dtype=np.uint32)) & 1).astype(bool)
    rt_all = np.where(elig, prob.runtime[sel], np.inf).min(axis=2).tolist()
    any_all = elig.any(axis=2).tolist()
    gpus_all = prob.gpus[sel].tolist()
    out_all = []
    for j, R in enumerate(prob.radix[sel].tolist()):
        if not all(any_all[j][:R]):
            raise ValueError("min() arg is an empty sequence")  # an option no node can run
        out: dict = {}
        for o, (g, r) in enumerate(zip(gpus_all[j][:R], rt_all[j][:R])):
            if g not in out or r < out[g][0]:
                out[g] = (r, o)
        out_all.append(out)
    if jobs is None:
        prob.extra["_best_runtime_all"] = [dict(d) for d in out_all]
    return out_all


def _best_runtime_by_g(prob: SearchProblem, j: int) -> dict:
    """`_best_runtime_all` for one job."""
    return _best_runtime_all(prob, [j])[0]


def _problem_gain(prob: SearchProblem, j: int, g: int, best=None) -> float:
    """Marginal gain on a marshalled problem (runtimes already include remaining batches)."""
    best = best if best is not None else _best_runtime_by_g(prob, j)
    if g not in best or (g + 1) not in best:
        return 0.0
    return max(0.0, best[g][0] - best[g + 1][0])


def optimus_marginal_gain(table, job, g: int, remaining_batches: int | None = None) -> float:
    """best_runtime(job, g) - best_runtime(job, g+1), best_runtime = least
    (latency x remaining batches) over the techniques profiled at that g; 0 if g+1 (or g) has no
    finite entry, and never negative (a harmful GPU has no gain)."""
    import math

    rem = int(job.total_batches if remaining_batches is None else remaining_batches)

    def best_rt(k):
        lats = [lat for (jid, _tech, gg), lat in table.entries.items() if jid == job.id and gg == k
                and math.isfinite(lat)]
        return min(lats) * rem if lats else None

    a, b = best_rt(g), best_rt(g + 1)
    if a is None or b is None:
        return 0.0
    return max(0.0, a - b)


def optimus_allocation(prob: SearchProblem) -> tuple:
    """(option per job, submission order) of the Optimus baseline.

    Waves: jobs FIFO (id order) while the sum of their minimum feasible g fits the
    cluster's GPUs; each gets its min g, then free GPUs go one at a time to the job
    with the largest marginal gain (lower job first on ties) while the gain is > 0.
    Order: wave, then descending g, then job id."""
    J = prob.J
    total = int(prob.node_gpus.sum())
    node_max = int(prob.node_gpus.max())
    best = _best_runtime_all(prob)
    gmin = [min(b) for b in best]
    alloc = [0] * J
    waves = []
    j = 0
    while j < J:
        wave = [j]
        used = gmin[j]
        j += 1
        while j < J and used + gmin[j] <= total:
            used += gmin[j]
            wave.append(j)
            j += 1
        for k in wave:
            alloc[k] = gmin[k]
        free = total - used
        while free > 0:
            pick, pick_gain = -1, 0.0
            for k in wave:
                if alloc[k] + 1 > node_max:
                    continue
                gain = _problem_gain(prob, k, alloc[k], best[k])
                if gain > pick_gain:
                    pick, pick_gain = k, gain
            if pick < 0:
                break
            alloc[pick] += 1
            free -= 1
        waves.append(wave)
    options = [best[k][alloc[k]][1] for k in range(J)]
    order = []
    for wave in waves:
        order.extend(sorted(wave, key=lambda k: (-alloc[k], k)))
    return options, order


def _explicit_solution(table, workload, opts, running_context, builder, device) -> Solution:
    prob = _baseline_problem(table, workload, opts, running_context)
    options, order = builder(prob)
    eng = get_engine(device)
    nprob = NativeProblem(prob, 62)
    explicit = np.array(list(options) + list(order), dtype=np.uint8)
    plan, opts_out, ms, runtimes = _decode(eng, prob, nprob, workload, SRC_EXPLICIT, 0, explicit=explicit)
    return Solution(plan=plan, status="Fixed", makespan=ms, objective=plan.predicted_makespan, problem=prob,
                    search=None, options=opts_out, order=list(order), runtimes=runtimes)


def plan_optimus(table, jobs, cluster=None, delta_opts=None, running_context=None, *, techniques=None,
                 device=None):
    workload = _as_workload(jobs, cluster, techniques)
    return _explicit_solution(table, workload, _opts(delta_opts), running_context, optimus_allocation,
                              device).plan


def current_practice_allocation(prob: SearchProblem) -> tuple:
    """Each job alone on a full node (largest feasible g if a full node does not fit), fastest
    technique at that g; jobs in id order, each on the earliest-free node."""
    node_max = int(prob.node_gpus.max())
    options = []
    for best in _best_runtime_all(prob):
        g = node_max if node_max in best else max(best)
        options.append(best[g][1])
    return options, list(range(prob.J))


def plan_current_practice(table, jobs, cluster=None, delta_opts=None, *, techniques=None, device=None):
    workload = _as_workload(jobs, cluster, techniques)
    return _explicit_solution(table, workload, _opts(delta_opts), None, current_practice_allocation,
                              device).plan


def evaluate_fixed(table, workload, options, order, delta_opts=None, running_context=None, device=None,
                   prune: bool = False) -> Solution:
    """Schedule one explicit candidate -- option digit per job (problem job axis, option order of
    the pruned lists when prune=True, of feasible_entries otherwise) and a submission order."""
    opts = _opts(delta_opts)
    if prune:
        prob = build_problem(table, workload, opts, running_context)
    else:
        prob = _baseline_problem(table, workload, opts, running_context)
    eng = get_engine(device)
    explicit = np.array(list(options) + list(order), dtype=np.uint8)
    plan, opts_out, ms, runtimes = _decode(eng, prob, NativeProblem(prob, 62), workload, SRC_EXPLICIT, 0,
                                           explicit=explicit)
    return Solution(plan=plan, status="Fixed", makespan=ms, objective=plan.predicted_makespan, problem=prob,
                    search=None, options=opts_out, order=list(order), runtimes=runtimes)


__all__ = [
    "Solution", "solve", "solve_problem", "plan_saturn", "resolve", "plan_random", "plan_random_best",
    "optimus_marginal_gain", "optimus_allocation", "plan_optimus", "current_practice_allocation",
    "plan_current_practice", "evaluate_fixed", "get_engine",
]
