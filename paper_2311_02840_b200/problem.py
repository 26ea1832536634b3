"""Marshal (profile table, workload, re-solve context) into the engine's dense problem.

This is the host half of the Solver's ``build_milp`` step (SPEC.md:192-196,
244-249) restricted to what the list-scheduling search needs:

* option lists per job: ``feasible_entries`` order (profiling.py:154-161),
  optionally reduced by an exact dominance prune (single node only);
* runtimes ``T = remaining x latency`` (profiling.py:147-151) plus the
  checkpoint cost rho for a running job whose (technique, g, node) changes
  (core.py:211-223);
* the time grid ``delta = max(sum_j min T / K_max, min_j min T / 4)``
   and grid durations ``d = ceil(T / delta)``,
  computed once here in float64 and shipped as integers -- the device never
  recomputes them;
* the candidate index space of SURVEY.md Appendix A1:
  ``index = c * J! + p`` with ``c`` the mixed-radix option code (job 0 most
  significant) and ``p`` the lexicographic (Lehmer) rank of the order.

Everything here runs once per solve; the per-candidate work is on the device.
"""

from __future__ import annotations

import math
from itertools import chain, repeat
from dataclasses import dataclass, field

import numpy as np

from . import errors as E
from .domain import RunConfig, feasible_configs, node_eligible
from .profiling import INFEASIBLE

TIME_GRID = "grid"
TIME_FLOAT = "float"
K_MAX_DEFAULT = 48
INF_I32 = 0x3FFFFFFF        # device "never free" sentinel (ghost slots)
MAX_LANES = 32              # nodes x padded GPUs must fit one warp


@dataclass
class SolveOptions:
    """The reference's delta_opts plus the engine's search knobs."""

    time_mode: str = TIME_GRID
    k_max: int = K_MAX_DEFAULT
    delta: float | None = None          # explicit interval length (seconds)
    prune: bool | None = None           # None: on for single-node clusters
    search: str = "auto"                # auto | exhaustive | sampled | local
    max_exhaustive: int = 1 << 36       # auto -> full scan when the space is <= this (~2 s worst case)
    max_bnb: int = 1 << 52              # auto -> exact bound-and-prune (one node, grid) up to this
    budget: int = 1 << 28               # sampled candidates when not exhaustive
    seed: int = 7                       # sampled stream: candidate i = substream(seed, i)
    walkers: int = 1 << 16              # local search: walkers at most (walker w starts at candidate w)
    wave: int | None = None             # local search: first wave (then x4 per wave); stops at the bound.
                                        # None: 2048 walkers of one warp (< 24 jobs), one resident
                                        # generation (2 x SMs) of 16-warp walkers (>= 24 jobs)
    max_rounds: int = 4096              # local search: rounds of 32 moves per walker
    ls_stop: bool = True                # local search: a walk ends at the lower bound (same result)
    ls_start: str = "greedy"            # local search: walker w starts at the greedy candidate perturbed
                                        # by substream(seed, w) ("greedy"), or at candidate w of the
                                        # sampled stream ("sampled")
    kernel: str = "auto"                # auto (bnb when it applies) | tree | index | bnb
    prove: bool = True                  # local search on one node: prove / improve the best makespan
                                        # with the state-space search (sat_search_dp) after a wave
    dp_states: int = 1 << 21            # state budget of one sat_search_dp call (all levels)
    dp_max_jobs: int = 20               # attempt the proof only up to this many jobs: beyond, the
                                        # state space explodes unless the slack is tiny, and a
                                        # failed attempt costs its whole budget (cfg4 at T = 8:
                                        # ~80 ms to exhaust 4 M states)
    dp_exact: bool = True               # several nodes: an inconclusive prover answer is asked again on
                                        # exact (labelled) states, which return a candidate (ABI v8)
    dp_at_bound: bool = True            # one node: ask sat_search_dp about the lower bound itself on a
                                        # side stream while the first local-search wave runs
    share_incumbent: bool = True        # several ranks: one incumbent cell over NVLink peer memory


@dataclass
class SearchProblem:
    job_ids: list
    jobs: list
    node_ids: list
    node_gpus: np.ndarray          # int32 [N]
    G: int                         # padded slots per node (power of two)
    W: int                         # lanes per candidate segment (8, 16 or 32)
    options: list                  # per job: [(RunConfig, latency)] after prune
    option_src: list               # per job: index of each kept option in feasible_entries
    radix: np.ndarray              # int32 [J]
    gpus: np.ndarray               # int32 [J, Cmax]
    node_mask: np.ndarray          # uint32 [J, Cmax]  bit n = option runnable on node n
    runtime: np.ndarray            # float64 [J, Cmax, N] seconds (0 where not runnable)
    dur_i32: np.ndarray            # int32 [J, Cmax, N] grid intervals
    release_i32: np.ndarray        # int32 [J]
    release_f64: np.ndarray        # float64 [J]
    init_free_i32: np.ndarray      # int32 [N, G] ascending per node, INF on ghost slots
    init_free_f64: np.ndarray      # float64 [N, G]
    time_mode: str
    delta: float
    pruned: bool
    resolve: bool = False
    extra: dict = field(default_factory=dict)

    # ---- derived sizes -------------------------------------------------
    @property
    def J(self) -> int:
        return len(self.job_ids)

    @property
    def N(self) -> int:
        return len(self.node_ids)

    @property
    def Cmax(self) -> int:
        return int(self.gpus.shape[1])

    @property
    def space(self) -> int:
        """Number of exhaustive candidates: prod(radix) * J!."""
        return math.prod(int(r) for r in self.radix) * math.factorial(self.J)

    def weights(self) -> list:
        """Mixed-radix weight of each job's option digit (job 0 most significant)."""
        w, out = 1, [0] * self.J
        for j in range(self.J - 1, -1, -1):
            out[j] = w
            w *= int(self.radix[j])
        return out

    def makespan_bound(self) -> int:
        """Upper bound on any grid makespan (sum of worst durations + offsets)."""
        worst = int(self.dur_i32.reshape(self.J, -1).max(axis=1).sum()) if self.J else 0
        real = self.init_free_i32[self.init_free_i32 < INF_I32]
        return worst + int(real.max() if real.size else 0) + int(self.release_i32.max() if self.J else 0)

    def lower_bound(self) -> float:
        """A makespan lower bound of every candidate (grid intervals or seconds): the latest
        committed free time, each job's earliest possible end, and the area bound
        (total GPU time >= initial commitments + every job's least g * d).  Computed once per
        problem (the arrays are not modified after build_problem)."""
        hit = self.extra.get("_lower_bound")
        if hit is not None:
            return hit
        grid = self.time_mode == TIME_GRID
        d = np.asarray(self.dur_i32 if grid else self.runtime, dtype=np.float64)
        init = self.init_free_i32 if grid else self.init_free_f64
        rel = np.asarray(self.release_i32 if grid else self.release_f64, dtype=np.float64)
        ng = [int(x) for x in self.node_gpus]
        srt = [sorted(float(init[n, i]) for i in range(ng[n])) for n in range(self.N)]
        real = [float(init[n, i]) for n in range(self.N) for i in range(ng[n])]
        lb = max(real) if real else 0.0
        area = sum(real)
        # g-th smallest initial free time of each node, per option gang size: [J, C, N]
        kth = np.full((self.N, max(max(ng), int(self.gpus.max())) + 1), np.inf)
        for n in range(self.N):
            kth[n, 1:ng[n] + 1] = srt[n]
        g = np.asarray(self.gpus, dtype=np.int64)
        C = g.shape[1]
        valid = (np.arange(C)[None, :] < np.asarray(self.radix)[:, None])[:, :, None] & (
            ((np.asarray(self.node_mask, dtype=np.int64)[:, :, None] >> np.arange(self.N)[None, None, :]) & 1) == 1)
        start = np.maximum(rel[:, None, None], kth[np.arange(self.N)[None, None, :], g[:, :, None]])
        ends = np.where(valid, start + d, np.inf).reshape(self.J, -1).min(axis=1)
        areas = np.where(valid, g[:, :, None] * d, np.inf).reshape(self.J, -1).min(axis=1)
        for j in range(self.J):
            lb = max(lb, float(ends[j]))
            area += float(areas[j])
        total = float(sum(ng))
        lb = max(lb, area / total)
        out = float(math.ceil(lb - 1e-9)) if grid else lb
        self.extra["_lower_bound"] = out
        return out

    def key_bits(self, n_indices: int) -> tuple:
        """(idx_bits, ms_bits) for packing (makespan << idx_bits) | index into 63 bits."""
        idx_bits = max(1, (max(n_indices, 1) - 1).bit_length())
        ms_bits = max(1, self.makespan_bound().bit_length())
        if self.time_mode == TIME_GRID and idx_bits + ms_bits > 63:
            raise E.TooLarge(f"key needs {idx_bits}+{ms_bits} bits > 63")
        return idx_bits, ms_bits

    # ---- candidate codec (host side, used only to explain results) ------
    def decode_index(self, index: int) -> tuple:
        """index -> (option digit per job, submission order); inverse of encode_index."""
        J = self.J
        conf, perm = divmod(int(index), math.factorial(J))
        opts = [0] * J
        for j in range(J - 1, -1, -1):
            conf, opts[j] = divmod(conf, int(self.radix[j]))
        pool = list(range(J))
        order = []
        for k in range(J):
            f = math.factorial(J - 1 - k)
            digit, perm = divmod(perm, f)
            order.append(pool.pop(digit))
        return opts, order

    def encode_index(self, opts, order) -> int:
        J = self.J
        conf = 0
        for j in range(J):
            conf = conf * int(self.radix[j]) + int(opts[j])
        pool = list(range(J))
        rank = 0
        for k, job in enumerate(order):
            digit = pool.index(job)
            pool.pop(digit)
            rank += digit * math.factorial(J - 1 - k)
        return conf * math.factorial(J) + rank


def _pow2_at_least(x: int) -> int:
    p = 1
    while p < x:
        p <<= 1
    return p


def _techniques_of(workload, table):
    techs = getattr(workload, "techniques", None)
    if techs:
        return techs
    raise E.InvariantViolation("techniques", "workload must carry its registered techniques")


def _dominance_prune(cost_rows: list) -> list:
    """Exact single-node prune: per g keep the cheapest option (earliest on ties), then keep
    g only while the cost strictly decreases with g.  Returns kept option indices in their
    original (canonical) order.  cost_rows: [(option_index, g, cost)] in canonical order."""
    best_per_g: dict = {}
    for idx, g, cost in cost_rows:
        cur = best_per_g.get(g)
        if cur is None or cost < cur[1]:
            best_per_g[g] = (idx, cost)
    kept, last = [], None
    for g in sorted(best_per_g):
        idx, cost = best_per_g[g]
        if last is None or cost < last:
            kept.append(idx)
            last = cost
    return sorted(kept)


class _OneNodeRow:
    """One-node option row before the prune: the job's feasible configs `cfgs`, the indices
    `sel` of those with a finite latency `lat`, runtimes t = rem x lat and gang sizes g."""
    __slots__ = ("cfgs", "sel", "lat", "t", "g")

    def __init__(self, cfgs, sel, lat, t, g):
        self.cfgs, self.sel, self.lat, self.t, self.g = cfgs, sel.tolist(), lat, t, g


_ONE_NODE_MEMO: dict = {}
_ONE_NODE_FAST: dict = {}     # (id(job), id(cluster)) -> (job, cluster, techniques, memo entry)
_ARRAY_ROW_MIN = 48          # one-node rows with at least this many configs go through arrays


def _one_node_options(job, workload):
    """(configs, profile-table keys, gang sizes, per-node eligibility) of `feasible_configs`
    (core.py:165-182) for one job, a pure function of immutable inputs memoised by value like
    `feasible_configs` itself.  Eligibility depends on a node only through its shape."""
    cluster = workload.cluster
    fast = _ONE_NODE_FAST.get((id(job), id(cluster)))
    if fast is not None and fast[0] is job and fast[1] is cluster:
        # the same (hashable, hence frozen) objects as a memoised call: skip hashing them
        # (pydantic / dataclass hashes walk every field); techniques compared by identity
        techs, ft = workload.techniques, fast[2]
        if techs is ft or (len(techs) == len(ft) and all(a is b for a, b in zip(techs, ft))):
            return fast[3]
    techniques = tuple(workload.techniques)
    try:
        key = (job, cluster, techniques)
        hit = _ONE_NODE_MEMO.get(key)
    except TypeError:                   # unhashable inputs: compute every time
        key, hit = None, None
    if hit is None:
        cfgs = tuple(feasible_configs(job, workload.cluster, techniques))
        keys = tuple((job.id, c.technique, c.gpus) for c in cfgs)
        tech_by_name = {t.name: t for t in techniques}
        shape_elig: dict = {}
        elig = []
        for c in cfgs:
            row = []
            for n in workload.cluster.nodes:
                k = (c.technique, c.gpus, n.gpu_count, n.gpu_memory)
                e = shape_elig.get(k)
                if e is None:
                    e = shape_elig[k] = node_eligible(job, tech_by_name[c.technique], c.gpus, n)
                row.append(e)
            elig.append(tuple(row))
        elig_arr = np.array(elig, dtype=bool).reshape(len(cfgs), len(workload.cluster.nodes))
        hit = (cfgs, keys, np.array([c.gpus for c in cfgs], dtype=np.int64), tuple(elig), elig_arr)
        if key is not None:
            if len(_ONE_NODE_MEMO) > 1 << 16:
                _ONE_NODE_MEMO.clear()
            _ONE_NODE_MEMO[key] = hit
    if key is not None:
        if len(_ONE_NODE_FAST) > 1 << 16:
            _ONE_NODE_FAST.clear()
        techs = workload.techniques
        _ONE_NODE_FAST[(id(job), id(cluster))] = (job, cluster, techs if isinstance(techs, tuple) else techniques,
                                                  hit)                    # strong refs: ids stay unique
    return hit


def _dominance_prune_arrays(g: np.ndarray, cost: np.ndarray) -> list:
    """`_dominance_prune` over arrays (same result): per g the cheapest option, earliest on
    ties (lexsort by g, cost, index; first of each g), then g kept while the cost strictly
    decreases.  Costs are exact integers (grid) or the runtimes themselves (float)."""
    n = len(g)
    order = np.lexsort((np.arange(n), cost, g))
    gs = g[order]
    first = order[np.r_[True, gs[1:] != gs[:-1]]]          # best option per g, ascending g
    kept, last = [], None
    for idx, c in zip(first.tolist(), cost[first].tolist()):
        if last is None or c < last:
            kept.append(idx)
            last = c
    kept.sort()
    return kept


_TABLE_VIEWS: dict = {}      # id(entries dict) -> _TableView (a few tables at a time)


class _TableView:
    """A profile table's `entries` dict as arrays: its keys (insertion order), its latencies,
    and per requested key sequence the positions of those keys.  The view is reused only while
    the dict provably has the same content -- the same key objects in the same order (a list
    comparison that short-circuits on identity) and bit-equal latencies (one pass over the
    values) -- so a mutated table is re-read, never served stale.  Cheaper than one hashed
    lookup per (job, config) key (config 5: 11 008 lookups, ~1.2 ms) once the key positions
    of a workload are known."""

    __slots__ = ("entries", "keys", "vals", "lat", "index", "pos")

    def __init__(self, entries, keys, vals):
        self.entries, self.keys, self.vals = entries, keys, vals
        self.lat = np.array(vals, dtype=np.float64)
        self.index = None
        self.pos = {}

    @staticmethod
    def of(entries) -> "_TableView":
        # content check on the Python objects themselves: list equality short-circuits on
        # identity, so an unchanged dict costs two list copies (a changed value or key fails
        # the check and rebuilds the view)
        keys, vals = list(entries), list(entries.values())
        v = _TABLE_VIEWS.get(id(entries))
        if v is not None and v.entries is entries and v.keys == keys and v.vals == vals:
            return v
        if len(_TABLE_VIEWS) >= 8:
            _TABLE_VIEWS.clear()
        v = _TABLE_VIEWS[id(entries)] = _TableView(entries, keys, vals)
        return v

    def latencies(self, key_rows, total: int) -> np.ndarray:
        """Latency of every key of the concatenated `key_rows` (tuples of keys; INFEASIBLE when
        absent), i.e. the same array as one `entries.get(key, INFEASIBLE)` per key."""
        sig = tuple(map(id, key_rows))
        hit = self.pos.get(sig)
        if hit is None or len(hit[0]) != len(key_rows) or any(a is not b for a, b in zip(hit[0], key_rows)):
            if self.index is None:
                self.index = {k: i for i, k in enumerate(self.keys)}
            pos = np.fromiter(map(self.index.get, chain.from_iterable(key_rows), repeat(-1)), dtype=np.int64,
                              count=total)
            if len(self.pos) >= 256:                          # bounded: many pools of one table
                self.pos.clear()
            hit = self.pos[sig] = (tuple(key_rows), pos)      # the rows themselves: ids stay unique
        pos = hit[1]
        return np.where(pos >= 0, self.lat[pos], INFEASIBLE)


def _batch_rows(pool, workload, remaining, get, opts, prune: bool, err, entries=None):
    """The marshalling of every job at once when no job has a running configuration: the same
    arrays as the per-job rows in `build_problem`, built with one profile-table pass and
    whole-problem numpy ops instead of per-job / per-option Python (config 5: 64 jobs x 172
    configs; config 4: 32 jobs x 26 configs x 4 nodes).

    Per job, in canonical order: finite-latency configs (profiling.py:154-161), runtime
    t = rem x lat (profiling.py:151) on every node that can host the config, infinite on the
    others; the least runtime for choose_delta; on one node the exact dominance prune of
    `_dominance_prune` -- per (job, g) the cheapest option (earliest on ties), kept while the
    cost strictly decreases with g; the running minimum restarts at every job by offsetting
    integer cost ranks per job."""
    per = [_one_node_options(job, workload) for job in pool]
    J = len(pool)
    counts = np.fromiter((len(p[1]) for p in per), dtype=np.int64, count=J)
    total = int(counts.sum())
    if isinstance(entries, dict) and type(entries) is dict:
        lat_all = _TableView.of(entries).latencies([p[1] for p in per], total)
    else:
        lat_all = np.fromiter(map(get, chain.from_iterable(p[1] for p in per), repeat(INFEASIBLE)),
                              dtype=np.float64, count=total)
    job_all = np.repeat(np.arange(J), counts)
    finite = np.isfinite(lat_all)
    nfin = np.bincount(job_all[finite], minlength=J)
    if (nfin == 0).any():
        raise err.NoFeasibleConfig(pool[int(np.argmax(nfin == 0))].id)
    sel = np.flatnonzero(finite)                       # job-major, canonical order within a job
    job = job_all[sel]
    start_all = np.concatenate(([0], np.cumsum(counts)[:-1]))
    start_sel = np.concatenate(([0], np.cumsum(nfin)[:-1]))
    g = np.concatenate([p[2] for p in per])[sel]
    elig = np.concatenate([p[4] for p in per])[sel]    # [n, N]
    N = elig.shape[1]
    lat = lat_all[sel]
    rem = np.fromiter((remaining[j.id] for j in pool), dtype=np.float64, count=J)
    t = rem[job] * lat                                 # the same IEEE product as rem * lat
    t_node = np.where(elig, t[:, None], INFEASIBLE)    # [n, N]
    row_min = np.minimum.reduceat(t_node.min(axis=1), start_sel)
    if not np.isfinite(row_min).all():
        raise err.NoFeasibleConfig(pool[int(np.argmax(~np.isfinite(row_min)))].id)
    min_rt = row_min.tolist()
    if opts.delta is not None:
        delta = float(opts.delta)
        if not delta > 0:
            raise err.InvariantViolation("delta", "must be > 0")
        horizon = math.ceil(sum(min_rt) / delta)
        if horizon > opts.k_max:
            raise err.HorizonOverflow(horizon, opts.k_max)
    else:
        delta = choose_delta(min_rt, opts.k_max)
    grid = opts.time_mode == TIME_GRID
    n = len(sel)
    if prune:
        cost = np.ceil(t / delta) if grid else t
        # one stable argsort of an exact integer key (job, g, cost rank): within a (job, g)
        # group the cheapest option first, the earliest of equal costs first.  Grid costs are
        # small integers already (any order-preserving rank serves); float costs are ranked.
        cmax = float(cost.max()) if len(cost) else 0.0
        if grid and cmax < (1 << 24):
            crank = cost.astype(np.int64)
            U = int(cmax) + 1
        else:
            _, crank = np.unique(cost, return_inverse=True)
            U = int(crank.max()) + 1
        jg = job.astype(np.int64) * 64 + g
        if J * 64 <= (1 << 16):
            # (job, g) fits 16 bits: a stable radix sort groups it (indices ascending within a
            # group), then per group the least cost and the first index reaching it
            order = np.argsort(jg.astype(np.uint16), kind="stable")
            jgo = jg[order]
            starts = np.flatnonzero(np.r_[True, jgo[1:] != jgo[:-1]])
            co = crank[order]
            cmin = np.minimum.reduceat(co, starts)
            gid = np.cumsum(np.r_[False, jgo[1:] != jgo[:-1]])
            pos = np.where(co == cmin[gid], np.arange(len(co)), len(co))
            first = order[np.minimum.reduceat(pos, starts)]
        else:
            order = np.argsort(jg * U + crank, kind="stable")
            jgo = jg[order]
            first = order[np.r_[True, jgo[1:] != jgo[:-1]]]
        # g kept while the cost strictly decreases: exclusive running minimum of the cost
        # ranks, restarted per job by offsetting each job above every later one
        v = crank[first].astype(np.int64) + (J - job[first]).astype(np.int64) * U
        prev = np.r_[np.iinfo(np.int64).max, np.minimum.accumulate(v)[:-1]]
        kept = np.sort(first[v < prev])
    else:
        kept = np.arange(n)
    kj = job[kept]
    radix = np.bincount(kj, minlength=J).astype(np.int32)
    kstart = np.concatenate(([0], np.cumsum(radix)[:-1]))
    slot = np.arange(len(kept)) - kstart[kj]
    Cmax = int(radix.max())
    gpus = np.zeros((J, Cmax), dtype=np.int32)
    gpus[kj, slot] = g[kept]
    ek = elig[kept]
    runtime = np.zeros((J, Cmax, N), dtype=np.float64)
    runtime[kj, slot, :] = np.where(ek, t[kept][:, None], 0.0)
    mask = np.zeros((J, Cmax), dtype=np.uint32)
    mask[kj, slot] = (ek.astype(np.uint32) << np.arange(N, dtype=np.uint32)[None, :]).sum(axis=1, dtype=np.uint32)
    dq = np.ceil(runtime / delta)
    if (dq >= INF_I32 // 4).any():
        raise err.TooLarge(f"duration {int(dq.max())} intervals overflows the device time type")
    # per job: (config, latency) of the kept options and their index among the finite ones
    local = (kept - start_sel[kj]).tolist()
    cfg_idx = (sel[kept] - start_all[kj]).tolist()
    lat_k = lat[kept].tolist()
    options, option_src = [[] for _ in range(J)], [[] for _ in range(J)]
    for jj, ci, li, lt in zip(kj.tolist(), cfg_idx, local, lat_k):
        options[jj].append((per[jj][0][ci], lt))
        option_src[jj].append(li)
    return options, option_src, radix, gpus, mask, runtime, dq.astype(np.int32), delta


def choose_delta(min_runtimes: list, k_max: int = K_MAX_DEFAULT) -> float:
    """delta = max(sequential-best total / K_max, shortest job / 4).
    Summation is left to right in job-id order (fixed so oracle and engine agree)."""
    total = 0.0
    for t in min_runtimes:
        total += t
    return max(total / k_max, min(min_runtimes) / 4.0)


def build_problem(table, workload, opts: SolveOptions | None = None, running_context=None,
                  jobs=None) -> SearchProblem:
    """Marshal one solve.  ``jobs`` restricts/reorders nothing: the job axis is always the
    selected jobs sorted by id (SPEC.md:249 tie-break key 1)."""
    opts = opts or SolveOptions()
    err = E.errors_for(workload)
    if opts.time_mode not in (TIME_GRID, TIME_FLOAT):
        raise err.InvariantViolation("time_mode", f"unknown {opts.time_mode!r}")
    cluster = workload.cluster
    techniques = _techniques_of(workload, table)
    tech_by_name = {t.name: t for t in techniques}
    pool = list(jobs) if jobs is not None else list(workload.jobs)

    if running_context is not None:
        remaining = {k: int(v) for k, v in running_context.remaining.items() if int(v) > 0}
        pool = [j for j in pool if j.id in remaining]
        current = dict(running_context.current)
        rho = float(running_context.checkpoint_cost)
    else:
        remaining = {j.id: int(j.total_batches) for j in pool}
        current, rho = {}, 0.0
    pool.sort(key=lambda j: j.id)
    nodes = list(cluster.nodes)
    N = len(nodes)
    max_g = max(n.gpu_count for n in nodes)
    G = _pow2_at_least(max_g)
    W = max(8, _pow2_at_least(N * G))
    if N * G > MAX_LANES:
        raise err.TooLarge(f"{N} nodes x {G} padded GPUs exceed one warp ({MAX_LANES} lanes)")

    grid = opts.time_mode == TIME_GRID
    prune = (N == 1) if opts.prune is None else bool(opts.prune)
    if prune and N != 1:
        raise err.InvariantViolation("prune", "the dominance prune is exact only on one node")
    if _BATCH_ROWS and pool and techniques is workload.techniques and not any(j.id in current for j in pool):
        options, option_src, radix, gpus, mask, runtime, dur, delta = _batch_rows(
            pool, workload, remaining, table.entries.get, opts, prune, err, entries=table.entries)
        return _search_problem(pool, nodes, G, W, options, option_src, radix, gpus, mask, runtime, dur,
                               opts, delta, prune, running_context)

    # per job: canonical option list with per-node runtimes
    from .profiling import feasible_entries  # local: avoid a cycle at import time
    shapes = {}                         # (gpu_count, gpu_memory) -> shape index
    node_shape = [shapes.setdefault((n.gpu_count, n.gpu_memory), len(shapes)) for n in nodes]
    shape_rep = [None] * len(shapes)
    for n, sh in zip(nodes, node_shape):
        if shape_rep[sh] is None:
            shape_rep[sh] = n
    rows, row_min = [], []         # row_min[j]: the job's least runtime (None: take it from the row)
    get = table.entries.get
    node_id_list = [n.id for n in nodes]
    for job in pool:
        rem = remaining[job.id]
        cur = current.get(job.id)
        cur = tuple(cur) if cur is not None else None
        if N == 1 and cur is None:
            # one node: every feasible (technique, g) runs on it (core.py:165-182 keeps only
            # configs some node hosts), so the runtime is the plain estimate (profiling.py:151).
            # feasible_entries (profiling.py:154-161) as arrays: rem * lat elementwise is the
            # same IEEE product; per-option tuples are built only for the prune's survivors.
            cfgs, keys, g_all, _, _ = _one_node_options(job, workload)
            if len(keys) < _ARRAY_ROW_MIN:      # short rows: plain tuples beat numpy call overhead
                fin = [(c, lat) for c, lat in zip(cfgs, map(get, keys, repeat(INFEASIBLE))) if math.isfinite(lat)]
                if not fin:
                    raise err.NoFeasibleConfig(job.id)
                ts = [rem * lat for _, lat in fin]
                rows.append([(c, lat, [t]) for (c, lat), t in zip(fin, ts)])
                row_min.append(min(ts))
                continue
            lat_all = np.fromiter(map(get, keys, repeat(INFEASIBLE)), dtype=np.float64, count=len(keys))
            sel = np.flatnonzero(np.isfinite(lat_all))
            if not len(sel):
                raise err.NoFeasibleConfig(job.id)
            lat = lat_all[sel]
            rows.append(_OneNodeRow(cfgs, sel, lat, rem * lat, g_all[sel]))
            row_min.append(rows[-1].t.min().item())
            continue
        if techniques is workload.techniques:
            # several nodes or a running config: runtime = plain estimate on every eligible node
            # (profiling.py:151), + rho off the job's running (technique, g, node);
            # eligibility per (config, node) from the memo
            cfgs, keys, _, elig, _ = _one_node_options(job, workload)
            row = []
            for c, lat, el in zip(cfgs, map(get, keys, repeat(INFEASIBLE)), elig):
                if math.isfinite(lat):
                    t0 = rem * lat
                    if cur is None:
                        row.append((c, lat, [t0 if e else INFEASIBLE for e in el]))
                    else:
                        row.append((c, lat, [(t0 if (c.technique, c.gpus, nid) == cur else t0 + rho)
                                             if e else INFEASIBLE for e, nid in zip(el, node_id_list)]))
            if not row or all(math.isinf(t) for _, _, pn in row for t in pn):
                raise err.NoFeasibleConfig(job.id)
            rows.append(row)
            row_min.append(None)
            continue
        entries = feasible_entries(table, job, workload)
        if not entries:
            raise err.NoFeasibleConfig(job.id)
        row = []
        for cfg, lat in entries:
            tech = tech_by_name[cfg.technique]
            # eligibility depends on the node only through its shape: once per shape
            elig = [node_eligible(job, tech, cfg.gpus, rep) for rep in shape_rep]
            t0 = rem * lat                                    # profiling.py:151
            per_node = []
            for n, sh in zip(nodes, node_shape):
                if not elig[sh]:
                    per_node.append(INFEASIBLE)
                    continue
                t = t0
                if cur is not None and (cfg.technique, cfg.gpus, n.id) != cur:
                    t = t + rho
                per_node.append(t)
            row.append((cfg, lat, per_node))
        if all(math.isinf(t) for _, _, pn in row for t in pn):
            raise err.NoFeasibleConfig(job.id)
        rows.append(row)
        row_min.append(None)

    J = len(pool)
    if J == 0:
        raise err.InvariantViolation("jobs", "nothing to plan")
    min_rt = [m if m is not None else min(min(pn) for _, _, pn in row) for m, row in zip(row_min, rows)]
    if opts.delta is not None:
        delta = float(opts.delta)
        if not delta > 0:
            raise err.InvariantViolation("delta", "must be > 0")
        horizon = math.ceil(sum(min_rt) / delta)
        if horizon > opts.k_max:
            raise err.HorizonOverflow(horizon, opts.k_max)
    else:
        delta = choose_delta(min_rt, opts.k_max)

    kept_rows, kept_src = [], []
    for row in rows:
        if type(row) is _OneNodeRow:
            if prune:
                keep = _dominance_prune_arrays(row.g, np.ceil(row.t / delta) if grid else row.t)
            else:
                keep = range(len(row.t))
            kept_rows.append([(row.cfgs[row.sel[i]], row.lat[i].item(), [row.t[i].item()]) for i in keep])
            kept_src.append(list(keep))
            continue
        if prune:
            ceil = math.ceil
            keep = _dominance_prune([(i, cfg.gpus, ceil(pn[0] / delta)) for i, (cfg, _, pn) in enumerate(row)]
                                    if grid else [(i, cfg.gpus, pn[0]) for i, (cfg, _, pn) in enumerate(row)])
        else:
            keep = list(range(len(row)))
        kept_rows.append([row[i] for i in keep])
        kept_src.append(keep)

    Cmax = max(len(r) for r in kept_rows)
    radix = np.array([len(r) for r in kept_rows], dtype=np.int32)
    # dense tables in one pass: rows padded to Cmax with infeasible options
    pad_rt = [INFEASIBLE] * N
    rt_all = np.array([[pn for _, _, pn in row] + [pad_rt] * (Cmax - len(row)) for row in kept_rows],
                      dtype=np.float64).reshape(J, Cmax, N)
    gpus = np.array([[cfg.gpus for cfg, _, _ in row] + [0] * (Cmax - len(row)) for row in kept_rows],
                    dtype=np.int32).reshape(J, Cmax)
    ok = np.isfinite(rt_all)
    mask = (ok.astype(np.uint32) << np.arange(N, dtype=np.uint32)[None, None, :]).sum(axis=2, dtype=np.uint32)
    runtime = np.where(ok, rt_all, 0.0)
    with np.errstate(invalid="ignore"):
        dq = np.ceil(np.where(ok, rt_all, 0.0) / delta)         # SPEC.md:183, same IEEE ops as math.ceil(t / delta)
    if (dq >= INF_I32 // 4).any():
        raise err.TooLarge(f"duration {int(dq.max())} intervals overflows the device time type")
    dur = dq.astype(np.int32)
    return _search_problem(pool, nodes, G, W, [[(cfg, lat) for cfg, lat, _ in r] for r in kept_rows], kept_src,
                           radix, gpus, mask, runtime, dur, opts, delta, prune, running_context)


_BATCH_ROWS = True           # no running configuration: `_batch_rows`


def _search_problem(pool, nodes, G, W, options, option_src, radix, gpus, mask, runtime, dur, opts, delta, prune,
                    running_context) -> SearchProblem:
    N, J = len(nodes), len(pool)
    init_i = np.full((N, G), INF_I32, dtype=np.int32)
    init_f = np.full((N, G), np.inf, dtype=np.float64)
    for n, node in enumerate(nodes):
        init_i[n, : node.gpu_count] = 0
        init_f[n, : node.gpu_count] = 0.0
    return SearchProblem(
        job_ids=[j.id for j in pool], jobs=pool, node_ids=[n.id for n in nodes],
        node_gpus=np.array([n.gpu_count for n in nodes], dtype=np.int32), G=G, W=W,
        options=options, option_src=option_src,
        radix=radix, gpus=gpus, node_mask=mask, runtime=runtime, dur_i32=dur,
        release_i32=np.zeros(J, dtype=np.int32), release_f64=np.zeros(J, dtype=np.float64),
        init_free_i32=init_i, init_free_f64=init_f, time_mode=opts.time_mode, delta=delta,
        pruned=prune, resolve=running_context is not None,
    )


def option_config(problem: SearchProblem, j: int, o: int) -> RunConfig:
    return problem.options[j][o][0]
