"""Introspection driver: event-driven execution of a Plan with periodic re-solves
(the caller of the Solver's re-solve path).

    simulate(workload, table, plan0, opts) -> SimReport
    remaining_batches(...)
    apply_replan(...)

The reference ships only the types this module consumes (``RunningContext``,
core.py:211-223; ``Plan``, core.py:106-120); the simulator itself is SPEC text.
Semantics frozen here:

* A plan is a dispatch list: each job runs on its planned node with its planned
  (technique, g) and starts at the first instant >= its planned start at which the
  node has g free GPUs (GPUs held by running or checkpointing jobs are busy).  A
  capacity-feasible plan with exact profiles therefore executes verbatim.
* A running job progresses one batch per profiled latency (``estimate_runtime``
  semantics, profiling.py:147-151).
* At every multiple of R (R > 0, jobs unfinished) the state is frozen:
  remaining = total - floor(done); running jobs report the
  (technique, g, node) they hold; the replanner is called with that
  ``RunningContext`` and its plan (start times relative to the tick) is adopted.
* apply_replan: a running job whose new entry keeps its (technique, g, node) and
  starts at the tick continues uninterrupted; any other running job is
  checkpointed -- its run segment ends at the tick with floor(done) batches, it
  holds its old GPUs for rho seconds (SPEC.md:389 capacity during the drain), and
  then follows its new entry.  Pending jobs take their new entries.
* A replanner failure keeps the old plan and the run continues.
* Events at equal times: Finish (and checkpoint end) < IntrospectionTick < Start,
  then job id.  Everything is deterministic.

Host-side by design: one event per job state change plus one re-solve per tick;
every candidate plan of every re-solve is evaluated on the GPU engine.
"""

from __future__ import annotations

import csv
import heapq
import io
import json
import math
import time
from dataclasses import dataclass, field

from . import errors as E

EPS = 1e-9

# event classes, in tie order
EV_FINISH, EV_TICK, EV_START = 0, 1, 2


@dataclass
class SimOptions:
    """introspection interval R (0 disables) and checkpoint overhead rho.

    ``replanner``: "saturn" (plan_saturn re-solve on the engine), "optimus" (Optimus-
    Dynamic), or a callable ``(table, workload, running_context) -> Plan``
    whose start times are relative to the tick."""

    introspection_interval: float = 0.0
    checkpoint_overhead: float = 30.0
    replanner: object = "saturn"
    delta_opts: object = None
    planner: str = "saturn"
    seed: int | None = None
    max_ticks: int = 100000

    def __post_init__(self):
        if not self.introspection_interval >= 0:
            raise E.InvariantViolation("introspection_interval", "must be >= 0")
        if not self.checkpoint_overhead >= 0:
            raise E.InvariantViolation("checkpoint_overhead", "must be >= 0")


@dataclass
class Segment:
    job: str
    technique: str
    gpus: int
    node: str
    start: float
    end: float
    batches: int
    kind: str = "run"            # "run" | "checkpoint"


@dataclass
class SimReport:
    """SPEC.md:359-362."""

    makespan: float
    timeline: list
    replan_count: int
    checkpoint_count: int
    checkpoint_time_total: float
    profiling_time_total: float
    planner: str
    seed: int | None
    replan_failures: int = 0
    solve_stats: list = field(default_factory=list)   # per re-solve: (tick, candidates, device_s, wall_s)

    def to_dict(self) -> dict:
        return {
            "makespan": self.makespan, "replan_count": self.replan_count,
            "checkpoint_count": self.checkpoint_count, "checkpoint_time_total": self.checkpoint_time_total,
            "profiling_time_total": self.profiling_time_total, "planner": self.planner, "seed": self.seed,
            "replan_failures": self.replan_failures,
            "timeline": [s.__dict__.copy() for s in self.timeline],
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True)

    def timeline_csv(self) -> str:
        """job,technique,gpus,node,start_s,end_s,batches (run segments)."""
        out = io.StringIO()
        w = csv.writer(out, lineterminator="\n")
        w.writerow(["job", "technique", "gpus", "node", "start_s", "end_s", "batches"])
        for s in sorted(self.timeline, key=lambda s: (s.start, s.job)):
            if s.kind == "run":
                w.writerow([s.job, s.technique, s.gpus, s.node, repr(s.start), repr(s.end), s.batches])
        return out.getvalue()


@dataclass
class _Job:
    spec: object
    lat: dict                      # (technique, g) -> per-batch latency
    state: str = "pending"         # pending | running | checkpointing | done
    tech: str = ""
    gpus: int = 0
    node: str = ""
    planned: float = 0.0           # absolute planned start (pending)
    remaining: int = 0             # batches left at the start of the current / next segment
    seg_start: float = 0.0
    token: int = 0                 # invalidates stale finish / checkpoint-end events
    finish: float = 0.0
    held: tuple = ()               # (node, gpus) held while checkpointing
    next_entry: tuple = ()         # (tech, g, node, planned) to follow after the checkpoint


def remaining_batches(job: _Job, clock: float) -> int:
    """total - floor(done); Pending -> its remaining; Done -> 0."""
    if job.state == "done":
        return 0
    if job.state != "running":
        return job.remaining
    lat = job.lat[(job.tech, job.gpus)]
    done = math.floor((clock - job.seg_start) / lat + EPS)
    return max(1, job.remaining - done)


def _latencies(table, workload) -> dict:
    from .profiling import feasible_entries

    out = {}
    for job in workload.jobs:
        out[job.id] = {(cfg.technique, cfg.gpus): float(lat) for cfg, lat in feasible_entries(table, job, workload)}
    return out


def _replanner(opts: SimOptions):
    rp = opts.replanner
    if callable(rp):
        return rp
    from . import planners as PL

    if rp == "saturn":
        return lambda table, workload, ctx: PL.resolve(table, workload, ctx, opts.delta_opts)
    if rp in ("optimus", "optimus_dynamic"):
        return lambda table, workload, ctx: PL.plan_optimus(table, workload, None, opts.delta_opts,
                                                             running_context=ctx)
    raise E.InvariantViolation("replanner", f"unknown replanner {rp!r}")


class _Sim:
    def __init__(self, workload, table, plan0, opts: SimOptions):
        self.w = workload
        self.table = table
        self.opts = opts
        self.lat = _latencies(table, workload)
        self.jobs = {}
        for spec in workload.jobs:
            if spec.id not in plan0.entries:
                raise E.InvalidPlan(f"plan0 misses job {spec.id}")
            self.jobs[spec.id] = _Job(spec=spec, lat=self.lat[spec.id], remaining=int(spec.total_batches))
        self.free = {n.id: int(n.gpu_count) for n in workload.cluster.nodes}
        self.events = []
        self.seq = 0
        self.clock = 0.0
        self.timeline = []
        self.replans = 0
        self.failures = 0
        self.ckpts = 0
        self.solve_stats = []
        self._adopt(plan0, 0.0, running_ok=False)

    # ---- events ------------------------------------------------------------------
    def push(self, t: float, kind: int, job: str = "", token: int = 0):
        self.seq += 1
        heapq.heappush(self.events, (t, kind, job, self.seq, token))

    def _entry(self, plan, job_id):
        e = plan.entries[job_id]
        return e.config.technique, int(e.config.gpus), e.node, float(e.start_time)

    def _adopt(self, plan, now: float, running_ok: bool):
        """apply_replan for every unfinished job in `plan`."""
        rho = float(self.opts.checkpoint_overhead)
        for job_id in sorted(plan.entries):
            j = self.jobs.get(job_id)
            if j is None or j.state == "done":
                continue
            tech, g, node, s_rel = self._entry(plan, job_id)
            if (tech, g) not in j.lat:
                raise E.InvalidPlan(f"job {job_id}: ({tech}, {g}) is not a feasible entry")
            planned = now + s_rel
            if j.state == "running":
                if running_ok and (tech, g, node) == (j.tech, j.gpus, j.node) and s_rel <= EPS:
                    continue                                   # unchanged: keeps running
                self._checkpoint(j, now, rho, (tech, g, node, planned))
            elif j.state == "checkpointing":
                j.next_entry = (tech, g, node, planned)
            else:
                j.tech, j.gpus, j.node, j.planned = tech, g, node, planned
                self.push(planned, EV_START, job_id)

    def _checkpoint(self, j: _Job, now: float, rho: float, next_entry: tuple):
        lat = j.lat[(j.tech, j.gpus)]
        done = min(j.remaining - 1, math.floor((now - j.seg_start) / lat + EPS))
        done = max(0, done)
        self.timeline.append(Segment(j.spec.id, j.tech, j.gpus, j.node, j.seg_start, now, done))
        j.remaining -= done
        j.state = "checkpointing"
        j.held = (j.node, j.gpus)
        j.next_entry = next_entry
        j.token += 1
        self.ckpts += 1
        self.timeline.append(Segment(j.spec.id, j.tech, j.gpus, j.node, now, now + rho, 0, kind="checkpoint"))
        self.push(now + rho, EV_FINISH, j.spec.id, j.token)

    # ---- dispatch ------------------------------------------------------------------
    def dispatch(self, now: float):
        pend = sorted((j.planned, jid) for jid, j in self.jobs.items() if j.state == "pending")
        for planned, jid in pend:
            if planned > now + EPS * max(1.0, abs(now)):
                continue
            j = self.jobs[jid]
            if self.free[j.node] >= j.gpus:
                self.free[j.node] -= j.gpus
                j.state = "running"
                j.seg_start = now
                j.token += 1
                j.finish = now + j.remaining * j.lat[(j.tech, j.gpus)]
                self.push(j.finish, EV_FINISH, jid, j.token)

    # ---- main loop -------------------------------------------------------------------
    def run(self):
        R = float(self.opts.introspection_interval)
        if R > 0:
            self.push(R, EV_TICK)
        ticks = 0
        replan = _replanner(self.opts) if R > 0 else None
        while self.events:
            t, kind, jid, _seq, token = heapq.heappop(self.events)
            self.clock = t
            if kind == EV_FINISH:
                j = self.jobs[jid]
                if token != j.token:
                    continue
                if j.state == "running":
                    self.free[j.node] += j.gpus
                    self.timeline.append(Segment(jid, j.tech, j.gpus, j.node, j.seg_start, t, j.remaining))
                    j.remaining = 0
                    j.state = "done"
                    j.finish = t
                elif j.state == "checkpointing":
                    node, g = j.held
                    self.free[node] += g
                    j.held = ()
                    tech, gg, nd, planned = j.next_entry
                    j.tech, j.gpus, j.node, j.planned = tech, gg, nd, max(planned, t)
                    j.state = "pending"
                    self.push(j.planned, EV_START, jid)
            elif kind == EV_TICK:
                if all(j.state == "done" for j in self.jobs.values()):
                    continue
                ticks += 1
                if ticks > self.opts.max_ticks:
                    raise E.PlanFailure("introspection tick limit reached")
                self._tick(t, replan)
                self.push(t + R, EV_TICK)
            # starts come after every finish and tick of the same instant
            if not self.events or self.events[0][0] > t:
                self.dispatch(t)
        if any(j.state != "done" for j in self.jobs.values()):
            raise E.PlanFailure("simulation ended with unfinished jobs (plan could not be dispatched)")

    def _tick(self, now: float, replan):
        from . import domain
        from .planners import _family

        # the caller's own RunningContext (core.py:211-223 for reference objects)
        RunningContext = getattr(_family(self.w), "RunningContext", domain.RunningContext)  # noqa: N806
        remaining, current = {}, {}
        for jid, j in sorted(self.jobs.items()):
            if j.state == "done":
                continue
            remaining[jid] = remaining_batches(j, now)
            if j.state == "running":
                current[jid] = (j.tech, j.gpus, j.node)
        ctx = RunningContext(remaining=remaining, current=current,
                             checkpoint_cost=float(self.opts.checkpoint_overhead))
        t0 = time.perf_counter()
        try:
            plan = replan(self.table, self.w, ctx)
        except E.SchedulerError:
            self.failures += 1                     # keep the old plan, continue
            return
        except Exception:                          # engine trouble -> ReplanFailure semantics
            self.failures += 1
            return
        self.solve_stats.append((now, time.perf_counter() - t0))
        self.replans += 1
        self._adopt(plan, now, running_ok=True)

    def report(self) -> SimReport:
        makespan = max((j.finish for j in self.jobs.values()), default=0.0)
        return SimReport(
            makespan=makespan, timeline=self.timeline, replan_count=self.replans,
            checkpoint_count=self.ckpts, checkpoint_time_total=self.ckpts * float(self.opts.checkpoint_overhead),
            profiling_time_total=float(getattr(self.table, "profiling_cost", 0.0)), planner=self.opts.planner,
            seed=self.opts.seed, replan_failures=self.failures, solve_stats=self.solve_stats)


def simulate(workload, table, plan0, opts: SimOptions | None = None) -> SimReport:
    """Execute plan0 with introspection."""
    sim = _Sim(workload, table, plan0, opts or SimOptions())
    sim.run()
    return sim.report()


def apply_replan(sim: _Sim, new_plan, now: float) -> None:
    """SPEC.md:383-391 on a live simulation state (exposed for tests)."""
    sim._adopt(new_plan, now, running_ok=True)


def verify_report(report: SimReport, workload) -> None:
    """SimReport invariants: work conservation, per-node capacity over every
    segment (checkpoint drains included), makespan = last segment end."""
    from .domain import sweep_capacity

    per_job: dict = {}
    for s in report.timeline:
        per_job[s.job] = per_job.get(s.job, 0) + s.batches
    for job in workload.jobs:
        if per_job.get(job.id, 0) != int(job.total_batches):
            raise E.InvalidPlan(f"job {job.id}: {per_job.get(job.id, 0)} batches run, total {job.total_batches}")
    sweep_capacity([(s.node, s.gpus, s.start, s.end) for s in report.timeline], workload.cluster)
    last = max((s.end for s in report.timeline if s.kind == "run"), default=0.0)
    if abs(last - report.makespan) > 1e-6 * max(1.0, last):
        raise E.InvalidPlan(f"makespan {report.makespan} != last segment end {last}")
