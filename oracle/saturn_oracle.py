"""CPU ORACLE for the Saturn plan-search hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module, and only as the checker / CPU baseline.  The
product path (paper_2311_02840_b200) never imports it.

It is a literal, slow restatement of the reference's semantics, written
independently of the product code:

* profile-table side: feasible_configs / memory rule (core.py:145-182),
  feasible_entries (profiling.py:154-161), estimate_runtime (profiling.py:147-151),
  synthetic latency (profiling.py:25-43), SplitMix64 (rng.py:10-56);
* solver side (the reference's milp/planners modules are missing, so SPEC text):
  choose_delta and the grid, the exhaustive candidate
  space and lexicographic tie-break (SPEC.md:219-227, 249 -> SURVEY.md A1),
  list scheduling "earliest-fit" with explicit GPU ids,
  plan_random draws, Optimus, Current
  Practice, the re-solve duration transform;
* independent optimum checks: brute_force_schedule over (option, node, start
  interval) tuples and the time-indexed MILP
  solved by HiGHS through scipy.optimize.milp.

Pinning: tests/test_golden.py (test_oracle_profile_table_matches_reference, test_rng_vectors,
test_spec_examples_oracle) checks this module against golden vectors
produced by running the reference package itself (tests/golden/make_golden.py)
and against the SPEC.md known-answer examples.  Plan identity for the solver has
no reference implementation to pin against (the reference milp module does not
import); the optimum VALUE is pinned by HiGHS and brute force, and the winner identity of the
headline solves by tests/golden/make_winners.py (HiGHS optimum + the C oracle's scan from
index 0 to the first candidate reaching it).
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


# ---------------------------------------------------------------- rng.py:10-56
def mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class Rng:
    def __init__(self, state):
        self.state = state & MASK64

    def next_u64(self):
        self.state = (self.state + GOLDEN) & MASK64
        return mix(self.state)

    def uniform(self):
        return (self.next_u64() >> 11) / float(1 << 53)

    def below(self, n):
        limit = (1 << 64) - ((1 << 64) % n)
        while True:
            r = self.next_u64()
            if r < limit:
                return r % n

    def shuffle(self, items):
        for i in range(len(items) - 1, 0, -1):
            j = self.below(i + 1)
            items[i], items[j] = items[j], items[i]


def substream(seed, *salts):
    s = seed & MASK64
    for salt in salts:
        s = mix(((s ^ (salt & MASK64)) + GOLDEN) & MASK64)
    return Rng(s)


# ---------------------------------------------------------------- core.py:145-182
def fits(job, tech, g, mem):
    if tech.archetype == "offloaded":
        return True
    shard = 1.0 if tech.archetype == "replicated" else float(g)
    return job.model_memory / shard + job.activation_memory <= mem + 1e-12


def configs_of(job, cluster, techniques):
    top = max(n.gpu_count for n in cluster.nodes)
    out = []
    for t in techniques:
        for g in range(t.min_gpus, top + 1):
            if any(n.gpu_count >= g and fits(job, t, g, n.gpu_memory) for n in cluster.nodes):
                out.append((t.name, g))
    return out


def latency(job, tech, g, cluster):
    """SyntheticExecutor.profile (profiling.py:66-70 -> 25-43)."""
    mems = [n.gpu_memory for n in cluster.nodes if n.gpu_count >= g]
    if not mems or not fits(job, tech, g, max(mems)):
        return math.inf
    s, k = tech.serial_fraction, tech.comm_overhead
    return tech.offload_multiplier * job.base_batch_time * ((1.0 - s) / g + s + k * (g - 1))


def profile_entries(workload):
    """build_profile_table(workload, SyntheticExecutor) entries (profiling.py:122-144)."""
    ent = {}
    for job in workload.jobs:
        for tname, g in configs_of(job, workload.cluster, workload.techniques):
            tech = next(t for t in workload.techniques if t.name == tname)
            ent[(job.id, tname, g)] = latency(job, tech, g, workload.cluster)
    return ent


def options_of(entries, job, workload):
    """feasible_entries (profiling.py:154-161): [(tech, g, latency)] finite, canonical order."""
    out = []
    for tname, g in configs_of(job, workload.cluster, workload.techniques):
        lat = entries.get((job.id, tname, g), math.inf)
        if math.isfinite(lat):
            out.append((tname, g, lat))
    return out


# ---------------------------------------------------------------- problem
@dataclass
class Problem:
    """Dense restatement of one solve (oracle-owned layout)."""

    job_ids: list
    node_ids: list
    node_gpus: list
    options: list          # per job: [(tech, g)]
    gpus: list             # per job: [g]
    eligible: list         # per job: [[bool per node]]
    runtime: list          # per job: [[seconds per node]]  (inf where not eligible)
    dur: list              # per job: [[grid intervals per node]] (or seconds in float mode)
    delta: float
    grid: bool
    release: list = field(default_factory=list)
    init_free: list = field(default_factory=list)   # per node: [free time per GPU id]

    @property
    def J(self):
        return len(self.job_ids)

    @property
    def N(self):
        return len(self.node_ids)

    @property
    def radix(self):
        return [len(o) for o in self.options]

    @property
    def space(self):
        return math.prod(self.radix) * math.factorial(self.J)


def build(entries, workload, *, k_max=48, delta=None, prune=None, grid=True, context=None):
    """Restatement of the solver's table -> (options, T, delta, d) step.

    entries: the profile table's dict (reference ProfileTable.entries works).
    context: (remaining: dict, current: dict, rho) for a re-solve."""
    jobs = sorted(workload.jobs, key=lambda j: j.id)
    if context is not None:
        remaining, current, rho = context
        jobs = [j for j in jobs if remaining.get(j.id, 0) > 0]
    else:
        remaining, current, rho = {j.id: j.total_batches for j in jobs}, {}, 0.0
    nodes = list(workload.cluster.nodes)
    techs = {t.name: t for t in workload.techniques}
    rows = []
    for job in jobs:
        row = []
        for tname, g, lat in options_of(entries, job, workload):
            el, rt = [], []
            for n in nodes:
                ok = n.gpu_count >= g and fits(job, techs[tname], g, n.gpu_memory)
                el.append(ok)
                if not ok:
                    rt.append(math.inf)
                    continue
                t = remaining[job.id] * lat
                cur = current.get(job.id)
                if cur is not None and tuple(cur) != (tname, g, n.id):
                    t = t + rho
                rt.append(t)
            row.append(((tname, g), el, rt))
        rows.append(row)
    mins = [min(t for _, _, rt in row for t in rt) for row in rows]
    if delta is None:
        acc = 0.0
        for m in mins:
            acc += m
        delta = max(acc / k_max, min(mins) / 4.0)
    if prune is None:
        prune = len(nodes) == 1
    kept = []
    for row in rows:
        if not prune:
            kept.append(row)
            continue
        def cost(rt):
            return math.ceil(rt[0] / delta) if grid else rt[0]
        per_g = {}
        for i, (cfg, el, rt) in enumerate(row):
            g = cfg[1]
            if g not in per_g or cost(rt) < per_g[g][1]:
                per_g[g] = (i, cost(rt))
        keep, last = [], None
        for g in sorted(per_g):
            i, c = per_g[g]
            if last is None or c < last:
                keep.append(i)
                last = c
        kept.append([row[i] for i in sorted(keep)])
    dur = []
    for row in kept:
        dur.append([[(math.ceil(t / delta) if grid else t) if math.isfinite(t) else math.inf for t in rt]
                    for _, _, rt in row])
    return Problem(
        job_ids=[j.id for j in jobs], node_ids=[n.id for n in nodes], node_gpus=[n.gpu_count for n in nodes],
        options=[[cfg for cfg, _, _ in row] for row in kept], gpus=[[cfg[1] for cfg, _, _ in row] for row in kept],
        eligible=[[el for _, el, _ in row] for row in kept], runtime=[[rt for _, _, rt in row] for row in kept],
        dur=dur, delta=delta, grid=grid, release=[0] * len(jobs),
        init_free=[[0] * n.gpu_count for n in nodes])


# ---------------------------------------------------------------- candidate codec
def decode_index(prob, index):
    J = prob.J
    conf, perm = divmod(index, math.factorial(J))
    opts = [0] * J
    for j in reversed(range(J)):
        conf, opts[j] = divmod(conf, prob.radix[j])
    pool = list(range(J))
    order = []
    for k in range(J):
        d, perm = divmod(perm, math.factorial(J - 1 - k))
        order.append(pool.pop(d))
    return opts, order


def encode_index(prob, opts, order):
    conf = 0
    for j in range(prob.J):
        conf = conf * prob.radix[j] + opts[j]
    pool = list(range(prob.J))
    rank = 0
    for k, job in enumerate(order):
        d = pool.index(job)
        pool.pop(d)
        rank += d * math.factorial(prob.J - 1 - k)
    return conf * math.factorial(prob.J) + rank


def decode_stream(prob, rng):
    """plan_random draw order: below(|C_j|) per job in id order, then shuffle."""
    opts = [rng.below(r) for r in prob.radix]
    order = list(range(prob.J))
    rng.shuffle(order)
    return opts, order


def candidate(prob, source, seed, ident):
    if source == "index":
        return decode_index(prob, ident)
    if source == "substream":
        return decode_stream(prob, substream(seed, ident))
    if source == "seed":
        return decode_stream(prob, Rng(seed + ident))
    raise ValueError(source)


# ---------------------------------------------------------------- list scheduler
def list_schedule(prob, opts, order, record=False):
    """Per-GPU free times with explicit GPU ids.  For each job in order: on every eligible
    node the job could start at its g-th smallest free time (max with the release) and
    would end d(node) later; choose the node that finishes it earliest (lowest node index
    on ties -- with node-independent durations that is the earliest-starting node); the g
    earliest-free GPUs (lowest id on ties) run the job."""
    free = [list(f) for f in prob.init_free]
    starts, nodes = {}, {}
    for j in order:
        o = opts[j]
        g = prob.gpus[j][o]
        best = None
        for n in range(prob.N):
            if not prob.eligible[j][o][n] or prob.node_gpus[n] < g:
                continue
            t = sorted(free[n])[g - 1]
            t = max(t, prob.release[j])
            end = t + prob.dur[j][o][n]
            if best is None or end < best[0]:
                best = (end, t, n)
        e, s, n = best
        ids = sorted(range(prob.node_gpus[n]), key=lambda k: (free[n][k], k))[:g]
        for k in ids:
            free[n][k] = e
        starts[j], nodes[j] = s, n
    ms = max(max(f) for f in free if f)
    if record:
        return ms, starts, nodes
    return ms


def search(prob, source="index", seed=0, lo=0, hi=None):
    """Lowest (makespan, id) over candidates [lo, hi) of a source."""
    hi = prob.space if hi is None else hi
    best = None
    for ident in range(lo, hi):
        ms = list_schedule(prob, *candidate(prob, source, seed, ident))
        if best is None or ms < best[0]:
            best = (ms, ident)
    return best


# ---------------------------------------------------------------- baselines
def best_by_g(prob, j):
    out = {}
    for o, g in enumerate(prob.gpus[j]):
        rt = min(t for t in prob.runtime[j][o] if math.isfinite(t))
        if g not in out or rt < out[g][0]:
            out[g] = (rt, o)
    return out


def optimus(prob):
    total = sum(prob.node_gpus)
    top = max(prob.node_gpus)
    best = [best_by_g(prob, j) for j in range(prob.J)]
    gmin = [min(b) for b in best]
    alloc = [0] * prob.J
    order = []
    j = 0
    while j < prob.J:
        wave, used = [j], gmin[j]
        j += 1
        while j < prob.J and used + gmin[j] <= total:
            wave.append(j)
            used += gmin[j]
            j += 1
        for k in wave:
            alloc[k] = gmin[k]
        spare = total - used
        while spare > 0:
            cand = []
            for k in wave:
                g = alloc[k]
                if g + 1 > top or g not in best[k] or g + 1 not in best[k]:
                    continue
                gain = max(0.0, best[k][g][0] - best[k][g + 1][0])
                if gain > 0:
                    cand.append((-gain, k))
            if not cand:
                break
            _, k = min(cand)
            alloc[k] += 1
            spare -= 1
        order += sorted(wave, key=lambda k: (-alloc[k], k))
    return [best[k][alloc[k]][1] for k in range(prob.J)], order


def current_practice(prob):
    top = max(prob.node_gpus)
    opts = []
    for j in range(prob.J):
        b = best_by_g(prob, j)
        g = top if top in b else max(b)
        opts.append(b[g][1])
    return opts, list(range(prob.J))


# ---------------------------------------------------------------- independent optima
def brute_force_schedule(prob, horizon=None):
    """enumerate per-job (option, node, start interval) with a capacity
    check (grid mode only).  Returns the optimum makespan in intervals."""
    assert prob.grid
    K = horizon if horizon is not None else sum(min(min(d) for d in row) for row in prob.dur)
    choices = []
    for j in range(prob.J):
        cj = []
        for o, g in enumerate(prob.gpus[j]):
            for n in range(prob.N):
                if not prob.eligible[j][o][n]:
                    continue
                d = prob.dur[j][o][n]
                for i in range(0, K - d + 1):
                    cj.append((i + d, g, n, i, d))
        choices.append(cj)
    best = math.inf
    for combo in itertools.product(*choices):
        ms = max(c[0] for c in combo)
        if ms >= best:
            continue
        ok = True
        for n in range(prob.N):
            use = [0] * K
            for end, g, nn, i, d in combo:
                if nn == n:
                    for t in range(i, i + d):
                        use[t] += g
            if max(use) > prob.node_gpus[n]:
                ok = False
                break
        if ok:
            best = ms
    return best


def milp_optimum(prob, horizon=None, time_limit=60.0):
    """Time-indexed MILP of SPEC.md:182-200 (C1 one start per job, C2 per-node capacity per
    interval, C3 M >= completion) solved with HiGHS; horizon K = sum of per-job min d (always
    feasible).  Returns the optimal M in intervals."""
    import numpy as np
    from scipy.optimize import Bounds, LinearConstraint, milp

    assert prob.grid
    K = horizon if horizon is not None else sum(min(min(x for x in d if math.isfinite(x)) for d in row)
                                                for row in prob.dur)
    var = []
    for j in range(prob.J):
        for o, g in enumerate(prob.gpus[j]):
            for n in range(prob.N):
                if not prob.eligible[j][o][n]:
                    continue
                d = prob.dur[j][o][n]
                for i in range(0, K - d + 1):
                    var.append((j, g, n, i, d))
    nv = len(var) + 1                      # last variable = M
    rows, lo, hi = [], [], []
    for j in range(prob.J):                # C1
        r = np.zeros(nv)
        for v, (jj, *_rest) in enumerate(var):
            if jj == j:
                r[v] = 1
        rows.append(r); lo.append(1); hi.append(1)
    for n in range(prob.N):                # C2
        for t in range(K):
            r = np.zeros(nv)
            for v, (_j, g, nn, i, d) in enumerate(var):
                if nn == n and i <= t < i + d:
                    r[v] = g
            rows.append(r); lo.append(-np.inf); hi.append(prob.node_gpus[n])
    for j in range(prob.J):                # C3: M - sum (i+d) x >= 0
        r = np.zeros(nv)
        r[-1] = 1
        for v, (jj, _g, _n, i, d) in enumerate(var):
            if jj == j:
                r[v] = -(i + d)
        rows.append(r); lo.append(0); hi.append(np.inf)
    c = np.zeros(nv)
    c[-1] = 1
    integrality = np.ones(nv)
    integrality[-1] = 0
    bounds = Bounds(np.zeros(nv), np.concatenate([np.ones(nv - 1), [np.inf]]))
    res = milp(c, constraints=LinearConstraint(np.array(rows), lo, hi), integrality=integrality,
               bounds=bounds, options={"time_limit": time_limit})
    if res.status != 0:
        raise RuntimeError(f"HiGHS status {res.status}: {res.message}")
    return int(round(res.fun))
