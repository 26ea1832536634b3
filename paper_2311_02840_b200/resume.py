"""Checkpoint / resume of long exhaustive searches ("the search state is just
[lo, hi) plus the best key").

An exhaustive search -- the tree walk's warp tasks, bound-and-prune's, or the index kernel's
candidate ids -- is run as consecutive chunks of its range.  Between chunks the whole state is a
``SearchCursor``: which problem (a digest of the marshalled arrays), which kernel and layout, the
next task / id, the end, and the best packed key so far.  Each chunk starts from that key (it is
written into the device key cell before the launch), so chunked and one-shot searches return the
same (makespan, lowest index); bound-and-prune keeps pruning against it across resumptions.
``planners.solve(..., checkpoint=path, time_budget_s=...)`` saves the cursor as JSON when the
budget runs out (status "Suspended", best plan so far) and continues from it on the next call.
One rank (each rank of a sharded search would keep its own cursor).
"""

from __future__ import annotations

import hashlib
import json
import os
import time
from dataclasses import asdict, dataclass

import numpy as np

from . import errors as E
from .engine import INT64_MAX, SAT_OK, NativeProblem, _vp
from .problem import TIME_GRID, SearchProblem, SolveOptions


@dataclass
class SearchCursor:
    digest: str                 # problem arrays (problem_digest)
    kernel: str                 # "tree" | "bnb" | "index"
    prefix_len: int             # tree / bnb layout (0 for index)
    idx_bits: int
    next: int                   # first task (tree / bnb) or candidate id (index) not yet searched
    end: int
    key: int                    # best packed key so far; INT64_MAX = none (bnb: the seed bound)
    chunks: int = 0             # chunks run so far
    device_seconds: float = 0.0

    @property
    def done(self) -> bool:
        return self.next >= self.end

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=1)

    @classmethod
    def from_json(cls, text: str) -> "SearchCursor":
        return cls(**json.loads(text))

    def save(self, path) -> None:
        tmp = f"{path}.tmp"
        with open(tmp, "w") as f:
            f.write(self.to_json())
        os.replace(tmp, path)                   # a crash never leaves a torn checkpoint

    @classmethod
    def load(cls, path) -> "SearchCursor":
        with open(path) as f:
            return cls.from_json(f.read())


def problem_digest(prob: SearchProblem) -> str:
    """Identity of a marshalled problem: every array the kernels read."""
    h = hashlib.sha256()
    for a in (prob.radix, prob.gpus, prob.node_mask, prob.dur_i32, prob.node_gpus, prob.release_i32,
              prob.init_free_i32):
        arr = np.ascontiguousarray(a)
        h.update(str(arr.shape).encode())
        h.update(arr.tobytes())
    h.update(repr((prob.time_mode, prob.delta)).encode())
    return h.hexdigest()


def start_cursor(eng, prob: SearchProblem, opts: SolveOptions) -> SearchCursor:
    """A fresh cursor for the search engine.search would run (grid time, one rank)."""
    err = E.errors_for(prob.jobs[0]) if prob.jobs else E
    if prob.time_mode != TIME_GRID:
        raise err.TooLarge("resumable search needs grid time (packed keys)")
    mode, n_idx = eng.plan_search(prob, SolveOptions(**{**opts.__dict__, "search": "exhaustive"}))
    digest = problem_digest(prob)
    if eng._tree_ok(prob) and opts.kernel in ("auto", "bnb"):
        seed_ms = eng.seed_bound(prob)
        bits = max(1, (n_idx - 1).bit_length())
        nprob = NativeProblem(prob, bits)
        P = eng.bnb_prefix(nprob, 1 << 15)
        info = eng.tree_plan(nprob, P)
        return SearchCursor(digest, "bnb", info.prefix_len, bits, 0, int(info.n_tasks),
                            (seed_ms << bits) | ((1 << bits) - 1))
    bits, _ = prob.key_bits(n_idx)
    if eng._tree_ok(prob) and opts.kernel in ("tree",):
        info = eng.tree_plan(NativeProblem(prob, bits), 0)
        return SearchCursor(digest, "tree", info.prefix_len, bits, 0, int(info.n_tasks), INT64_MAX)
    return SearchCursor(digest, "index", 0, bits, 0, int(n_idx), INT64_MAX)


def run_cursor(eng, prob: SearchProblem, cur: SearchCursor, time_budget_s: float | None = None,
               chunk: int | None = None, max_chunks: int | None = None) -> SearchCursor:
    """Advance the cursor chunk by chunk until the range is done, the time budget is spent or
    max_chunks chunks ran.  Chunks grow geometrically from 1/256 of the range, each sized to
    ~1/8 of the budget."""
    torch = eng.torch
    if cur.digest != problem_digest(prob):
        raise E.errors_for(prob.jobs[0] if prob.jobs else prob).InvariantViolation(
            "checkpoint", "the checkpoint belongs to a different problem")
    nprob = NativeProblem(prob, cur.idx_bits)
    best = torch.empty(2, dtype=torch.int64, device=eng.device)
    t_start = time.perf_counter()
    size = chunk or max(1, (cur.end - cur.next) // 256)
    ran = 0
    while not cur.done and (max_chunks is None or ran < max_chunks):
        ran += 1
        lo, hi = cur.next, min(cur.end, cur.next + size)
        # the device cell's "nothing yet" is all ones (the kernels test for it), not INT64_MAX
        cell = (1 << 64) - 1 if cur.key == INT64_MAX else cur.key
        st = eng.lib.sat_best_set(_vp(best.data_ptr()), cell, (1 << 64) - 1, _vp(eng.stream()))
        eng._check(st, nprob=nprob)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if cur.kernel == "tree":
            eng.search_tree(nprob, cur.prefix_len, lo, hi, best)
        elif cur.kernel == "bnb":
            eng.search_bnb(nprob, cur.prefix_len, lo, hi, best)
        else:
            eng.search_index(nprob, lo, hi, best)
        e1.record()
        k = int(best[0].item()) & ((1 << 64) - 1)
        dt = e0.elapsed_time(e1) / 1e3
        cur.key = min(cur.key, k if k != (1 << 64) - 1 else INT64_MAX)
        cur.next, cur.chunks, cur.device_seconds = hi, cur.chunks + 1, cur.device_seconds + dt
        if time_budget_s is not None:
            spent = time.perf_counter() - t_start
            if spent >= time_budget_s:
                break
            if chunk is None and dt > 0:       # aim each chunk at ~1/8 of the budget
                size = max(1, min(size * 4, int((hi - lo) * (time_budget_s / 8) / dt)))
        elif chunk is None:
            size *= 2
    return cur


def cursor_result(prob: SearchProblem, cur: SearchCursor):
    """(makespan, index) of the cursor's key, or None while only a seed bound is held."""
    if cur.key == INT64_MAX:
        return None
    idx = cur.key & ((1 << cur.idx_bits) - 1)
    if cur.kernel == "bnb" and idx == (1 << cur.idx_bits) - 1:
        return None                             # the seed bound's placeholder: no candidate yet
    return float(cur.key >> cur.idx_bits), idx


__all__ = ["SearchCursor", "problem_digest", "start_cursor", "run_cursor", "cursor_result", "SAT_OK"]
