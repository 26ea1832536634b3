"""ctypes binding of the CUDA engine (include/saturn_engine.h) plus search orchestration.

PyTorch is plumbing here: device buffers, the current stream, and
``torch.distributed`` (NCCL) for the one cross-GPU exchange -- an all-reduce MIN
of each rank's packed (makespan, index) key.  There is
no CPU path: if the extension or a GPU is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass

import numpy as np

from . import errors as E
from .problem import TIME_FLOAT, TIME_GRID, SearchProblem, SolveOptions

LIB_PATH = os.environ.get("SATURN_ENGINE_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                                  "libsaturn_b200.so")

SAT_OK, SAT_ERR_INVALID, SAT_ERR_NO_OPTIONS, SAT_ERR_TOO_LARGE, SAT_ERR_UNSUPPORTED, SAT_ERR_CUDA = range(6)
SAT_TIME_GRID_I32, SAT_TIME_F64 = 0, 1
SRC_INDEX, SRC_SUBSTREAM, SRC_SEED, SRC_EXPLICIT, SRC_GREEDY = 0, 1, 2, 3, 4
INT64_MAX = (1 << 63) - 1
LS_ROUND_BITS = 13          # SAT_LS_ROUND_BITS: local-search keys are (makespan, rounds, walker)


def ls_key_fields(key: int, idx_bits: int) -> tuple:
    """(makespan, rounds scanned, walker) of a packed local-search key (include/saturn_engine.h)."""
    return (key >> (idx_bits + LS_ROUND_BITS), (key >> idx_bits) & ((1 << LS_ROUND_BITS) - 1),
            key & ((1 << idx_bits) - 1))

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64


class SatProblem(ctypes.Structure):
    _fields_ = [
        ("J", _i32), ("N", _i32), ("G", _i32), ("Cmax", _i32), ("time_mode", _i32), ("idx_bits", _i32),
        ("radix", _vp), ("gpus", _vp), ("node_mask", _vp), ("dur_i32", _vp), ("dur_f64", _vp),
        ("node_gpus", _vp), ("release_i32", _vp), ("release_f64", _vp),
        ("init_free_i32", _vp), ("init_free_f64", _vp),
    ]


class SatDpInfo(ctypes.Structure):
    _fields_ = [("status", _i32), ("levels", _i32), ("states", _u64), ("widest_level", _u64),
                ("makespan", _i32), ("reserved", _i32)]


SAT_DP_INFEASIBLE, SAT_DP_FEASIBLE, SAT_DP_BUDGET = 0, 1, 2
SAT_DP_EXACT = 1                # sat_search_dp_ex flag (ABI v8)
DP_STATUS = {SAT_DP_INFEASIBLE: "infeasible", SAT_DP_FEASIBLE: "feasible", SAT_DP_BUDGET: "budget"}


class SatTreeInfo(ctypes.Structure):
    _fields_ = [("prefix_len", _i32), ("n_sets", _i32), ("n_tasks", _u64),
                ("n_candidates", _u64), ("n_job_steps", _u64), ("pair_packed", _i32), ("reserved", _i32)]


# exported symbols and their signatures (the header is the source of truth;
# tests/test_abi.py checks that every declared function is exported)
_SIGS = {
    "sat_abi_version": ([], _i32),
    "sat_error_string": ([_i32], ctypes.c_char_p),
    "sat_device_info": ([ctypes.c_int, _vp, _vp, _vp], _i32),
    "sat_best_reset": ([_vp, _vp], _i32),
    "sat_workspace_bytes": ([_vp, _vp], _i32),
    "sat_search_index": ([_vp, _u64, _u64, _vp, _vp, ctypes.c_size_t, _vp], _i32),
    "sat_search_sampled": ([_vp, _i32, _u64, _u64, _u64, _vp, _vp, ctypes.c_size_t, _vp], _i32),
    "sat_tree_plan": ([_vp, _i32, _vp], _i32),
    "sat_search_tree": ([_vp, _i32, _u64, _u64, _vp, _vp, ctypes.c_size_t, _vp], _i32),
    "sat_search_bnb": ([_vp, _i32, _u64, _u64, _vp, _vp, ctypes.c_size_t, _vp], _i32),
    "sat_schedule": ([_vp, _i32, _u64, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                      ctypes.c_size_t, _vp], _i32),
    "sat_alu_probe": ([_i32, _i32, _i32, _vp, _vp, _vp], _i32),
    "sat_alu_probe16": ([_i32, _i32, _i32, _vp, _vp, _vp], _i32),
    "sat_tree_param_bytes": ([], ctypes.c_size_t),
    "sat_local_search": ([_vp, _i32, _u64, _u64, _u64, _i32, _i32, _vp, _vp, _vp, ctypes.c_size_t, _vp], _i32),
    "sat_ls_counter_offset": ([_vp, _vp], _i32),
    "sat_tree_shard": ([_vp, _i32, _i32, _i32, _vp, _vp], _i32),
    "sat_dp_workspace_bytes": ([_vp, _i32, _u64, _vp], _i32),
    "sat_best_set": ([_vp, _u64, _u64, _vp], _i32),
    "sat_best_copy": ([_vp, _vp, _vp], _i32),
    "sat_shared_best_alloc": ([_vp, _vp], _i32),
    "sat_shared_best_open": ([_vp, _vp], _i32),
    "sat_shared_best_close": ([_vp, _i32], _i32),
    "sat_peer_atomics": ([_i32, _i32, _vp], _i32),
    "sat_search_dp": ([_vp, _i32, _u64, _vp, _vp, _vp, ctypes.c_size_t, _vp], _i32),
    "sat_key_finish": ([_vp, _i32, _vp, _i32, _vp, _vp, _i32, _u64, _i32, _vp], _i32),
    "sat_dp_workspace_bytes_ex": ([_vp, _i32, _u64, _i32, _vp], _i32),
    "sat_search_dp_ex": ([_vp, _i32, _u64, _i32, _vp, _vp, _vp, ctypes.c_size_t, _vp], _i32),
}

_LIB = None


def load_library(path: str = LIB_PATH):
    """Load libsaturn_b200.so; fails loudly (no fallback) when it is not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise E.PlanFailure(
            f"CUDA engine not built ({path} missing); run `python -m paper_2311_02840_b200.build`")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.sat_abi_version() != 8:
        raise E.PlanFailure("libsaturn_b200.so ABI version mismatch")
    _LIB = lib
    return lib


def _ptr(a) -> int | None:
    return None if a is None else a.ctypes.data


class NativeProblem:
    """sat_problem_t over host numpy arrays (kept alive by this object)."""

    def __init__(self, prob: SearchProblem, idx_bits: int):
        grid = prob.time_mode == TIME_GRID
        J, Cmax, N = prob.J, prob.Cmax, prob.N
        self.radix = np.ascontiguousarray(prob.radix, dtype=np.int32)
        self.gpus = np.ascontiguousarray(prob.gpus, dtype=np.int32)
        self.mask = np.ascontiguousarray(prob.node_mask, dtype=np.uint32)
        self.node_gpus = np.ascontiguousarray(prob.node_gpus, dtype=np.int32)
        if grid:
            self.dur = np.ascontiguousarray(prob.dur_i32, dtype=np.int32)
            self.release = np.ascontiguousarray(prob.release_i32, dtype=np.int32)
            self.init = np.ascontiguousarray(prob.init_free_i32, dtype=np.int32)
        else:
            self.dur = np.ascontiguousarray(prob.runtime, dtype=np.float64)
            self.release = np.ascontiguousarray(prob.release_f64, dtype=np.float64)
            self.init = np.ascontiguousarray(prob.init_free_f64, dtype=np.float64)
        s = SatProblem()
        s.J, s.N, s.G, s.Cmax = J, N, prob.G, Cmax
        s.time_mode = SAT_TIME_GRID_I32 if grid else SAT_TIME_F64
        s.idx_bits = idx_bits
        s.radix, s.gpus, s.node_mask = _ptr(self.radix), _ptr(self.gpus), _ptr(self.mask)
        s.node_gpus = _ptr(self.node_gpus)
        if grid:
            s.dur_i32, s.release_i32, s.init_free_i32 = _ptr(self.dur), _ptr(self.release), _ptr(self.init)
        else:
            s.dur_f64, s.release_f64, s.init_free_f64 = _ptr(self.dur), _ptr(self.release), _ptr(self.init)
        self.struct = s
        self.idx_bits = idx_bits
        self.grid = grid
        self.job_ids = list(prob.job_ids)
        self.err = E.errors_for(prob.jobs[0]) if prob.jobs else E

    def job_without_options(self) -> str:
        """Id of the first job the engine found without a runnable option (SAT_ERR_NO_OPTIONS):
        no option, or an option no node can host."""
        for j, jid in enumerate(self.job_ids):
            R = int(self.radix[j])
            if R < 1:
                return jid
            for o in range(R):
                g = int(self.gpus[j, o]) if self.gpus.ndim == 2 else int(self.gpus[j * self.struct.Cmax + o])
                m = int(self.mask.reshape(len(self.job_ids), -1)[j, o])
                if not any((m >> n) & 1 and int(self.node_gpus[n]) >= g for n in range(len(self.node_gpus))):
                    return jid
        return "<job>"

    @property
    def ref(self):
        return ctypes.byref(self.struct)

    @property
    def param_bytes(self) -> int:
        """Bytes of problem tables that cross to the device per launch."""
        return sum(a.nbytes for a in (self.radix, self.gpus, self.mask, self.node_gpus, self.dur,
                                      self.release, self.init))


class _Cell:
    """A raw device pointer where the search methods expect a best tensor (data_ptr only)."""

    def __init__(self, ptr: int):
        self.ptr = ptr

    def data_ptr(self) -> int:
        return self.ptr


class SharedIncumbent:
    """The cross-rank incumbent: one sat_best_t in rank 0's HBM that every rank's search kernels
    atomicMin into and prune against while they run, reached over NVLink peer memory through a
    CUDA IPC handle (include/saturn_engine.h, sat_shared_best_*).  Bound-and-prune then cuts with
    the best key of ALL ranks, and a local-search walker is abandoned as soon as ANY rank has a
    lower-id walker at the bound -- N-rank pruning matches one rank's.

    Protocol per search: rank 0 resets (or seeds) the cell, every rank waits at a barrier, the
    kernels run, then each rank drains its stream, meets the others at a barrier (all kernels of
    all ranks done: the cell is final) and copies the cell into its local key buffer; the usual
    all-reduce MIN of those copies follows, which also fences the cell's next reset.
    Enabled only when every rank can reach the owner's memory with native peer atomics (NVLink /
    NVSwitch, or the same device); otherwise every rank keeps its own key and the all-reduce
    alone combines them."""

    def __init__(self, eng: "Engine", group):
        import torch.distributed as dist

        self.eng, self.group = eng, group
        rank, world = _rank_world(group)
        self.owner = rank == 0
        self.ptr = ctypes.c_void_p()
        lib = eng.lib
        payload = [None]
        if self.owner:
            handle = (ctypes.c_uint8 * 64)()
            st = lib.sat_shared_best_alloc(ctypes.byref(self.ptr), handle)
            payload = [(st, bytes(handle), eng.device.index)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(payload, src=src, group=group)
        st, hb, owner_dev = payload[0]
        ok = st == SAT_OK
        if ok and not self.owner:
            sup = ctypes.c_int32()
            ok = (lib.sat_peer_atomics(eng.device.index, owner_dev, ctypes.byref(sup)) == SAT_OK and sup.value == 1
                  and lib.sat_shared_best_open((ctypes.c_uint8 * 64).from_buffer_copy(hb), ctypes.byref(self.ptr))
                  == SAT_OK)
        flag = eng.torch.tensor([1 if ok else 0], dtype=eng.torch.int32, device=eng.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        self.enabled = bool(flag.item())
        if not self.enabled and ok and self.ptr.value:
            lib.sat_shared_best_close(self.ptr, 1 if self.owner else 0)
            self.ptr = ctypes.c_void_p()

    @property
    def cell(self) -> _Cell:
        return _Cell(self.ptr.value)

    def begin(self, seed_key: int | None = None):
        """Rank 0 resets (or seeds) the cell; all ranks start their kernels after a barrier."""
        import torch.distributed as dist

        eng = self.eng
        if self.owner:
            if seed_key is None:
                eng._check(eng.lib.sat_best_reset(self.ptr, _vp(eng.stream())))
            else:
                eng._check(eng.lib.sat_best_set(self.ptr, seed_key & ((1 << 64) - 1), (1 << 64) - 1,
                                                _vp(eng.stream())))
        eng.torch.cuda.current_stream(eng.device).synchronize()
        dist.barrier(group=self.group)
        return self.cell

    def collect(self, best):
        """All ranks' kernels done -> the cell is final: copy it into this rank's key buffer."""
        import torch.distributed as dist

        eng = self.eng
        eng.torch.cuda.current_stream(eng.device).synchronize()
        dist.barrier(group=self.group)
        eng._check(eng.lib.sat_best_copy(_vp(best.data_ptr()), self.ptr, _vp(eng.stream())))
        return best


@dataclass
class SearchResult:
    makespan: float            # grid intervals (grid mode) or seconds (float mode)
    index: int                 # winning candidate id (index / sample counter)
    source: int                # SRC_INDEX, SRC_SUBSTREAM, SRC_SEED
    seed: int
    evaluated: int             # candidates evaluated by all ranks
    kernel: str                # "tree", "index", "sampled"
    exhaustive: bool
    launches: int              # engine kernel launches on this rank
    job_steps: int = 0         # list-scheduling placements (tree walk) on all ranks
    device_seconds: float = 0.0
    wall_seconds: float = 0.0
    stats: dict | None = None  # bound-and-prune / local-search counters (this rank)
    idx_bits: int = 0          # bits of the packed key holding the candidate id
    state: tuple | None = None  # local search: the winning walker's final (options, order)
    replay: tuple | None = None  # the winner's schedule (option, node, start, makespan), queued
                                 # behind the search when search(replay=True)
    proven: bool = False       # local search: makespan proven optimal by sat_search_dp


class Engine:
    """One engine per process / CUDA device."""

    def __init__(self, device=None):
        import torch

        if not torch.cuda.is_available():
            raise E.PlanFailure("no CUDA device: the plan-search engine has no CPU fallback")
        self.torch = torch
        self.lib = load_library()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        sm = ctypes.c_int32()
        self._check(self.lib.sat_device_info(self.device.index, ctypes.byref(sm), None, None))
        self.sm_count = sm.value
        self._best = torch.empty(2, dtype=torch.int64, device=self.device)
        self._ws = None
        self._dp_ws = None
        self._shared = {}
        self.launches = 0

    # ---- plumbing ----------------------------------------------------------
    def _check(self, st: int, err=None, what: str = "engine call", nprob=None):
        if st == SAT_OK:
            return
        if err is None:
            err = nprob.err if nprob is not None else E
        msg = f"{what}: {self.lib.sat_error_string(st).decode()}" if hasattr(self, "lib") else what
        if st == SAT_ERR_NO_OPTIONS:
            raise err.NoFeasibleConfig(nprob.job_without_options() if nprob is not None else "<job>")
        if st == SAT_ERR_INVALID:
            raise err.InvariantViolation("problem", msg)
        if st in (SAT_ERR_TOO_LARGE, SAT_ERR_UNSUPPORTED):
            raise err.TooLarge(msg)
        raise err.PlanFailure(msg)

    def stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def workspace(self, nprob: NativeProblem):
        nbytes = ctypes.c_size_t()
        self._check(self.lib.sat_workspace_bytes(nprob.ref, ctypes.byref(nbytes)), nprob=nprob)
        need = int(nbytes.value)
        if self._ws is None or self._ws.numel() < need:
            self._ws = self.torch.empty(max(need, 1 << 16), dtype=self.torch.uint8, device=self.device)
        return self._ws.data_ptr(), self._ws.numel()

    def reset_best(self, best=None):
        best = self._best if best is None else best
        self._check(self.lib.sat_best_reset(_vp(best.data_ptr()), _vp(self.stream())))
        return best

    def shared_incumbent(self, group):
        """The group's SharedIncumbent (created on first use, collectively), or None when peer
        atomics are not available on every rank."""
        key = id(group) if group is not None else 0
        sh = self._shared.get(key)
        if sh is None:
            sh = self._shared[key] = SharedIncumbent(self, group)
        return sh if sh.enabled else None

    # ---- kernels -------------------------------------------------------------
    def tree_plan(self, nprob: NativeProblem, prefix_len: int = 0) -> SatTreeInfo:
        info = SatTreeInfo()
        self._check(self.lib.sat_tree_plan(nprob.ref, prefix_len, ctypes.byref(info)), what="sat_tree_plan", nprob=nprob)
        return info

    def search_tree(self, nprob, prefix_len, task_lo, task_hi, best=None):
        best = self._best if best is None else best
        ws, wsb = self.workspace(nprob)
        self._check(self.lib.sat_search_tree(nprob.ref, prefix_len, task_lo, task_hi, _vp(best.data_ptr()),
                                             _vp(ws), wsb, _vp(self.stream())), what="sat_search_tree", nprob=nprob)
        self.launches += 1

    def search_bnb(self, nprob, prefix_len, task_lo, task_hi, best=None):
        """Bound-and-prune over the tree layout; returns the workspace (counters after the cursor)."""
        best = self._best if best is None else best
        ws, wsb = self.workspace(nprob)
        self._check(self.lib.sat_search_bnb(nprob.ref, prefix_len, task_lo, task_hi, _vp(best.data_ptr()),
                                            _vp(ws), wsb, _vp(self.stream())), what="sat_search_bnb", nprob=nprob)
        self.launches += 1
        return self._ws

    def tree_shard(self, nprob, prefix_len: int, rank: int, world: int) -> tuple:
        """Work-balanced contiguous task range of this rank (sat_tree_shard)."""
        if world == 1:
            info = self.tree_plan(nprob, prefix_len)
            return 0, info.n_tasks
        lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self.lib.sat_tree_shard(nprob.ref, prefix_len, world, rank, ctypes.byref(lo), ctypes.byref(hi)),
                    what="sat_tree_shard", nprob=nprob)
        return lo.value, hi.value

    def full_scan_prefix(self, nprob, world: int) -> int:
        """Lane-prefix length of a sharded full scan: the shortest with ~4 warp tasks per
        resident warp on every rank (40 warps per SM; profiles/r01e_shard_emulation.txt: cfg1
        P = 4 up to 2 ranks, P = 5 from 4).  One rank: the library's choice (0)."""
        return self.tree_prefix(nprob, 160 * self.sm_count * world) if world > 1 else 0

    def tree_prefix(self, nprob, min_tasks: int) -> int:
        """Shortest lane prefix with at least `min_tasks` warp tasks (0 = the library's choice)."""
        return self.bnb_prefix(nprob, min_tasks)

    def bnb_prefix(self, nprob, min_tasks: int = 1 << 15) -> int:
        """Shortest lane prefix giving enough warp tasks to spread the pruned search over the GPU."""
        J = nprob.struct.J
        for P in range(1, J - 1):
            info = SatTreeInfo()
            if self.lib.sat_tree_plan(nprob.ref, P, ctypes.byref(info)) != SAT_OK:
                break
            if info.n_tasks >= min_tasks:
                return P
        return 0

    def seed_bound(self, prob: SearchProblem, budget: int = 1 << 20, seed: int = 7) -> int:
        """Best makespan of a quick sampled search: an achievable upper bound (grid intervals).
        Seeding *best with (U << idx_bits | max index) lets any real candidate with makespan <= U
        replace it while the bound prunes from the start."""
        torch = self.torch
        s_bits = max(1, (budget - 1).bit_length())
        sprob = NativeProblem(prob, s_bits)
        tmp = self.reset_best(torch.empty(2, dtype=torch.int64, device=self.device))
        self.search_sampled(sprob, SRC_SUBSTREAM, seed, 0, budget, tmp)
        k = int(tmp[0].item()) & ((1 << 64) - 1)
        bound = k >> s_bits
        if prob.J >= 10 and prob.time_mode == TIME_GRID:
            # long orders: a local-search wave (~ms) usually reaches the optimum value, which
            # makes the exact search prune far more (seconds saved at 10-12 jobs)
            self.reset_best(tmp)
            self.local_search(sprob, SRC_SUBSTREAM, seed, 0, 4096, 4096, tmp, stop_ms=int(prob.lower_bound()))
            bound = min(bound, ls_key_fields(int(tmp[0].item()) & ((1 << 64) - 1), s_bits)[0])
        return bound

    def seed_upper_bound(self, prob: SearchProblem, nprob: NativeProblem, best, budget: int = 1 << 16,
                         seed: int = 7):
        """Seed *best (device) from seed_bound()."""
        U = self.seed_bound(prob, budget, seed)
        key = (U << nprob.idx_bits) | ((1 << nprob.idx_bits) - 1)
        cur = int(best[0].item())
        if cur == -1 or key < cur:
            best[0:1].fill_(key)

    def local_search(self, nprob, source, seed, lo, hi, max_rounds: int = 4096, best=None, state_out=None,
                     stop_ms: int = -1):
        """Walkers [lo, hi) of the local search; state_out (uint8 device tensor, 2J) receives the
        final (options, order) of walker lo when hi == lo + 1.  stop_ms >= 0 (the problem's lower
        bound) ends a walk at that makespan and abandons walkers that can no longer win."""
        best = self._best if best is None else best
        ws, wsb = self.workspace(nprob)
        self._check(self.lib.sat_local_search(nprob.ref, source, seed & ((1 << 64) - 1), lo, hi, max_rounds,
                                              int(stop_ms), _vp(best.data_ptr()),
                                              _vp(state_out.data_ptr()) if state_out is not None else None,
                                              _vp(ws), wsb, _vp(self.stream())), what="sat_local_search", nprob=nprob)
        self.launches += 1

    def local_search_state(self, nprob, source, seed, walker, max_rounds: int = 4096, stop_ms: int = -1):
        """Replay one walker (same stop_ms as its search): its final (options, order) as lists."""
        torch = self.torch
        J = nprob.struct.J
        out = torch.zeros(2 * J, dtype=torch.uint8, device=self.device)
        tmp = self.reset_best(torch.empty(2, dtype=torch.int64, device=self.device))
        self.local_search(nprob, source, seed, walker, walker + 1, max_rounds, tmp, out, stop_ms=stop_ms)
        v = out.cpu().tolist()
        return v[:J], v[J:]

    def side_stream(self) -> int:
        """A second stream of this engine's device (work overlapped with the current stream's)."""
        if getattr(self, "_side", None) is None:
            self._side = self.torch.cuda.Stream(device=self.device)
        return self._side.cuda_stream

    def dp_search(self, nprob: NativeProblem, target: int, max_states: int = 1 << 22, stream: int | None = None,
                  exact: bool = False):
        """sat_search_dp: does some candidate reach makespan <= target?  Returns (status, info,
        candidate) -- candidate = (options, order) when FEASIBLE.  Synchronous (on ``stream``,
        default the current stream).  ``exact`` (several nodes): labelled states and the list
        scheduler's own node choice, so FEASIBLE carries a candidate (SAT_DP_EXACT, ABI v8)."""
        torch = self.torch
        need = ctypes.c_size_t()
        flags = SAT_DP_EXACT if exact else 0
        self._check(self.lib.sat_dp_workspace_bytes_ex(nprob.ref, int(target), int(max_states), flags,
                                                       ctypes.byref(need)),
                    what="sat_dp_workspace_bytes", nprob=nprob)
        if self._dp_ws is None or self._dp_ws.numel() < need.value:
            self._dp_ws = None
            self._dp_ws = torch.empty(max(need.value, 1 << 16), dtype=torch.uint8, device=self.device)
        J = nprob.struct.J
        cand = (ctypes.c_uint8 * (2 * J))()
        info = SatDpInfo()
        self._check(self.lib.sat_search_dp_ex(nprob.ref, int(target), int(max_states), flags, cand,
                                              ctypes.byref(info), _vp(self._dp_ws.data_ptr()), self._dp_ws.numel(),
                                              _vp(self.stream() if stream is None else stream)),
                    what="sat_search_dp", nprob=nprob)
        self.launches += max(1, info.levels)
        out = None
        if info.status == SAT_DP_FEASIBLE and info.makespan >= 0:      # (the prover rebuilds none)
            v = list(cand)
            out = (v[:J], v[J:])
        return info.status, info, out

    def prove_below(self, prob: SearchProblem, makespan: int, opts: SolveOptions, lb: int | None = None,
                    stats: dict | None = None):
        """Descend from a known candidate makespan with sat_search_dp: target = makespan - 1 until
        no candidate reaches it (the last makespan is then optimal) or the state budget runs out.
        ``lb``: a proven lower bound (default the problem's).  Returns (proven, best makespan,
        improved candidate or None, stats)."""
        nprob = NativeProblem(prob, 1)
        stats = {"attempts": [], "states": 0} if stats is None else stats
        best_ms, cand = int(makespan), None
        lb = int(prob.lower_bound()) if lb is None else int(lb)
        exact = False               # several nodes: the canonical prover first, exact states on demand
        while best_ms > lb:
            st, info, c = self.dp_search(nprob, best_ms - 1, opts.dp_states, exact=exact)
            stats["attempts"].append({"target": best_ms - 1, "status": DP_STATUS[st], "levels": info.levels,
                                      "states": int(info.states), "widest_level": int(info.widest_level),
                                      **({"exact": True} if exact else {})})
            stats["states"] += int(info.states)
            if st == SAT_DP_INFEASIBLE:
                stats["proven"] = True
                return True, best_ms, cand, stats
            if st == SAT_DP_FEASIBLE and c is None and prob.N > 1 and not exact and opts.dp_exact:
                # the multi-node prover's (superset) level is non-empty: ask again on exact
                # states, which either rule the target out or return a candidate reaching it
                exact = True
                continue
            if st == SAT_DP_BUDGET or c is None:
                # out of budget: nothing proven, no shorter candidate in hand
                stats["proven"] = False
                return False, best_ms, cand, stats
            best_ms, cand = int(info.makespan), c
        stats["proven"] = True
        return True, best_ms, cand, stats                  # met the lower bound

    def search_index(self, nprob, lo, hi, best=None):
        best = self._best if best is None else best
        ws, wsb = self.workspace(nprob)
        self._check(self.lib.sat_search_index(nprob.ref, lo, hi, _vp(best.data_ptr()), _vp(ws), wsb,
                                              _vp(self.stream())), what="sat_search_index", nprob=nprob)
        self.launches += 1 if nprob.grid else 2

    def search_sampled(self, nprob, source, seed, lo, hi, best=None):
        best = self._best if best is None else best
        ws, wsb = self.workspace(nprob)
        self._check(self.lib.sat_search_sampled(nprob.ref, source, seed & ((1 << 64) - 1), lo, hi,
                                                _vp(best.data_ptr()), _vp(ws), wsb, _vp(self.stream())),
                    what="sat_search_sampled", nprob=nprob)
        self.launches += 1 if nprob.grid else 2

    def schedule(self, nprob: NativeProblem, source: int, seed: int = 0, ids=None, explicit=None, ids_dev=None):
        """Per-candidate (option, node, start) [n, J] and makespan [n], as numpy arrays.
        ``ids_dev``: candidate ids already on the device (int64 tensor, e.g. the masked winner key)."""
        torch = self.torch
        J = nprob.struct.J
        if ids_dev is not None:
            ids_t, ex = ids_dev, None
            n = ids_t.numel()
        elif source == SRC_EXPLICIT:
            arr = np.ascontiguousarray(explicit, dtype=np.int64).reshape(-1, 2 * J)
            for row in arr:
                if (row[:J] < 0).any() or (row[:J] >= nprob.radix).any() or sorted(row[J:]) != list(range(J)):
                    raise E.InvariantViolation("explicit", "option digit out of range or order not a permutation")
            ex = torch.as_tensor(arr.astype(np.uint8)).to(self.device)
            n = ex.shape[0]
            ids_t = None
        else:
            ids_t = torch.as_tensor(np.asarray(ids, dtype=np.uint64).view(np.int64)).to(self.device)
            n = ids_t.numel()
            ex = None
        # one device buffer for the four outputs -> one device-to-host read after the launch
        # layout: opt [n, J] i32 | node [n, J] i32 | start [n, J] i32/f64 | makespan [n] i64/f64
        st_dt, ms_dt = (np.int32, np.int64) if nprob.grid else (np.float64, np.float64)
        a8 = lambda b: (b + 7) & ~7                                              # noqa: E731
        o_node = a8(4 * n * J)
        o_start = o_node + a8(4 * n * J)
        o_ms = o_start + a8(np.dtype(st_dt).itemsize * n * J)
        out = torch.empty(o_ms + 8 * n, dtype=torch.uint8, device=self.device)
        base = out.data_ptr()
        opt_p, node_p, start_p, ms_p = base, base + o_node, base + o_start, base + o_ms
        ws, wsb = self.workspace(nprob)
        g = nprob.grid
        self._check(self.lib.sat_schedule(
            nprob.ref, source, seed & ((1 << 64) - 1),
            _vp(ids_t.data_ptr()) if ids_t is not None else None,
            _vp(ex.data_ptr()) if ex is not None else None, n,
            _vp(opt_p), _vp(node_p),
            _vp(start_p) if g else None, None if g else _vp(start_p),
            _vp(ms_p) if g else None, None if g else _vp(ms_p),
            _vp(ws), wsb, _vp(self.stream())), what="sat_schedule", nprob=nprob)
        self.launches += 1
        h = out.cpu().numpy()
        return (h[:4 * n * J].view(np.int32).reshape(n, J),
                h[o_node:o_node + 4 * n * J].view(np.int32).reshape(n, J),
                h[o_start:o_start + np.dtype(st_dt).itemsize * n * J].view(st_dt).reshape(n, J),
                h[o_ms:o_ms + 8 * n].view(ms_dt))

    # ---- orchestration ---------------------------------------------------------
    def plan_search(self, prob: SearchProblem, opts: SolveOptions, group=None) -> tuple:
        """Choose kernel + index encoding for a problem: returns (mode, n_indices, prefix)."""
        space = prob.space
        mode = opts.search
        if mode == "auto":
            # exact when the full scan is affordable, or when bound-and-prune applies (one
            # node, grid time) and the packed key still holds the index
            exact = space <= opts.max_exhaustive
            if not exact and opts.kernel in ("auto", "bnb") and self._tree_ok(prob) and space <= opts.max_bnb:
                # the bound-and-prune key holds (makespan <= seed bound) << idx_bits | index:
                # leave at least 7 bits for the makespan (grids of <= 127 intervals)
                exact = (space - 1).bit_length() <= 56
            # otherwise local search from greedy starts (grid time), else plain sampling
            mode = "exhaustive" if exact else ("local" if prob.time_mode == TIME_GRID and prob.J >= 2 else "sampled")
        if mode == "exhaustive":
            if space > (1 << 62):
                raise E.errors_for(prob.jobs[0]).TooLarge(f"exhaustive space {space} exceeds 2^62")
            return mode, space
        if mode == "local":
            return mode, int(opts.walkers)
        return mode, int(opts.budget)

    def search(self, prob: SearchProblem, opts: SolveOptions, group=None, source: int | None = None,
               seed: int | None = None, lo: int | None = None, hi: int | None = None,
               replay: bool = False, on_launched=None) -> SearchResult:
        """Run one solve's search on this rank's shard and combine across ranks (NCCL MIN).
        replay=True (grid time, full-scan / index / sampled searches): the winner's schedule is
        launched on the stream right behind the search, reading its id from the combined
        device key, so the host reads the key and the plan after one wait.
        on_launched(mode): host work run once the first kernels are queued and before the first
        wait on the device (it overlaps the search)."""
        torch = self.torch
        err = E.errors_for(prob.jobs[0]) if prob.jobs else E
        t0 = time.perf_counter()
        mode, n_idx = self.plan_search(prob, opts)
        rank, world = _rank_world(group)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()                       # device time covers every launch of the solve
        use_bnb = (mode == "exhaustive" and opts.kernel in ("auto", "bnb") and self._tree_ok(prob))
        seed_ms = None
        if use_bnb:
            # bound-and-prune: keys only ever hold makespans <= the seed bound
            seed_ms = self.seed_bound(prob)
            idx_bits = max(1, (n_idx - 1).bit_length())
            if idx_bits + max(1, seed_ms.bit_length()) > 63:
                if opts.kernel == "bnb":
                    raise err.TooLarge(f"key needs {idx_bits}+{seed_ms.bit_length()} bits > 63")
                mode, n_idx, use_bnb = "local", int(opts.walkers), False
        if not use_bnb:
            idx_bits, ms_bits = prob.key_bits(n_idx)
            if mode == "local" and idx_bits + LS_ROUND_BITS + ms_bits > 63:
                raise err.TooLarge(f"local-search key needs {idx_bits}+{LS_ROUND_BITS}+{ms_bits} bits > 63")
        nprob = NativeProblem(prob, idx_bits)
        launches0 = self.launches
        best = self.reset_best()
        # several ranks, grid keys, searches that prune (bound-and-prune) or abandon (local
        # search) on the incumbent: the kernels of every rank share one incumbent cell over
        # NVLink.  Full scans / sampled sweeps gain nothing from it and keep rank-local keys.
        shared = (self.shared_incumbent(group)
                  if world > 1 and nprob.grid and opts.share_incumbent and (use_bnb or mode == "local")
                  else None)
        if shared is not None:
            seed_key = (seed_ms << idx_bits) | ((1 << idx_bits) - 1) if use_bnb else None
            kbest = shared.begin(seed_key)
        else:
            kbest = best
        job_steps = 0
        stats, bnb_ws, ls_key = None, None, None
        ls_state = None
        proven_opt = False
        if mode == "exhaustive":
            src = SRC_INDEX
            use_tree = opts.kernel in ("auto", "tree", "bnb") and self._tree_ok(prob)
            if opts.kernel in ("tree", "bnb") and not use_tree and prob.J >= 3:
                raise err.TooLarge("tree / bnb kernels need one node, grid time, 3..20 jobs")
            # (one- and two-job spaces -- the tail of an introspection run -- are scanned by the
            # per-candidate index kernel whatever kernel was asked for)
            if use_bnb:
                # pruning makes task costs uneven but cheap: a short prefix (2^15 tasks over all
                # ranks) beats a longer one at every world size (profiles/r01e_shard_emulation.txt)
                P = self.bnb_prefix(nprob, 1 << 15)
                info = self.tree_plan(nprob, P)
                a, b = self.tree_shard(nprob, info.prefix_len, rank, world)
                if shared is None:
                    best[0:1].fill_((seed_ms << idx_bits) | ((1 << idx_bits) - 1))
                bnb_ws = self.search_bnb(nprob, info.prefix_len, a, b, kbest)
                stats = {"prefix_len": info.prefix_len, "tasks": b - a}
                kernel, evaluated = "bnb", info.n_candidates
            elif use_tree:
                info = self.tree_plan(nprob, self.full_scan_prefix(nprob, world))
                a, b = self.tree_shard(nprob, info.prefix_len, rank, world)
                self.search_tree(nprob, info.prefix_len, a, b, kbest)
                kernel, evaluated, job_steps = "tree", info.n_candidates, info.n_job_steps
            else:
                a, b = _shard(n_idx, rank, world)
                self.search_index(nprob, a, b, kbest)
                kernel, evaluated = "index", n_idx
            seed_used = 0
        elif mode == "local":
            # waves of walkers in walker order; stop after the first wave whose best meets the
            # lower bound (proven optimal).  The stop depends only on completed waves, so the
            # result is deterministic.
            src = (SRC_GREEDY if opts.ls_start == "greedy" else SRC_SUBSTREAM) if source is None else source
            seed_used = opts.seed if seed is None else seed
            target = prob.lower_bound() if nprob.grid else -1.0
            stop_ms = int(target) if (nprob.grid and opts.ls_stop) else -1
            off = ctypes.c_size_t()
            self._check(self.lib.sat_ls_counter_offset(nprob.ref, ctypes.byref(off)), nprob=nprob)
            # geometric waves (wave, 4 x wave, 16 x wave, ...): a small first wave keeps easy
            # problems cheap, larger later waves keep the GPU full when the bound is not met
            # first wave: 2 048 one-warp walkers (< 24 jobs); for 16-warp walkers one resident
            # generation -- two 512-thread blocks per SM (64 registers) -- since with keys
            # (makespan, rounds, walker) every walker of the wave runs until it falls behind
            # the fastest one at the bound (profiles/r02_ls_tiebreak_wave.txt; greedy starts:
            # profiles/r02h_greedy_wave_sweep.txt)
            wave = max(1, int(opts.wave)) if opts.wave else (2048 if prob.J < 24 else 2 * self.sm_count)
            rounds_total, walkers_done, waves = 0, 0, 0
            w0 = 0
            ls_states = []          # (first walker, [walkers][2J] final states) per wave on this rank
            # after a wave that misses the lower bound, the state-space search (one node) either
            # proves the wave's best optimal -- no candidate one interval shorter -- or returns a
            # shorter candidate; it is retried only when a later wave improves the best
            dp_ok = opts.prove and nprob.grid and prob.J <= min(64, opts.dp_max_jobs) and prob.N <= 8
            proof, dp_tried_at, dp_cand = None, None, None
            lb_int = int(target) if nprob.grid else 0
            spec_lb = dp_ok and prob.N == 1 and opts.dp_at_bound
            dp_lb_hit = False
            while w0 < n_idx:
                w1 = min(n_idx, w0 + wave)
                a, b = _shard(w1 - w0, rank, world)
                st_buf = torch.empty(max(1, b - a) * 2 * prob.J, dtype=torch.uint8, device=self.device)
                ls_states.append((w0 + a, w0 + b, st_buf))
                self.local_search(nprob, src, seed_used, w0 + a, w0 + b, opts.max_rounds, kbest, state_out=st_buf,
                                  stop_ms=stop_ms)
                if on_launched is not None:
                    on_launched(mode)
                    on_launched = None
                if spec_lb:
                    # one node: while the first wave runs, the state-space search asks on a side
                    # stream whether anything reaches the lower bound itself.  "No" lifts the
                    # proven bound by one interval, "yes" hands over an optimal candidate.
                    spec_lb = False
                    proof = {"attempts": [], "states": 0}
                    try:
                        st_lb, info_lb, c_lb = self.dp_search(NativeProblem(prob, 1), lb_int, opts.dp_states,
                                                              stream=self.side_stream())
                        proof["attempts"].append({"target": lb_int, "status": DP_STATUS[st_lb],
                                                  "levels": info_lb.levels, "states": int(info_lb.states),
                                                  "widest_level": int(info_lb.widest_level)})
                        proof["states"] += int(info_lb.states)
                        if st_lb == SAT_DP_INFEASIBLE:
                            lb_int += 1
                        elif st_lb == SAT_DP_FEASIBLE and c_lb is not None:
                            dp_cand, dp_lb_hit = (int(info_lb.makespan), c_lb), True
                        else:
                            dp_ok = False            # out of budget at the bound: higher targets too
                    except (E.TooLarge, err.TooLarge, E.InvariantViolation, err.InvariantViolation):
                        dp_ok = False
                walkers_done, waves, w0, wave = w1, waves + 1, w1, wave * 4
                if shared is not None:
                    shared.collect(best)
                # the combined key and this rank's rounds counter: one launch, one read-back
                kw, _ = self._key_finish(best, True, group, world, idx_bits, n_idx,
                                         extra=self._ws[off.value:off.value + 8], extra_words=1)
                kv = kw.cpu().tolist()
                rounds_total += int(kv[2])
                k = int(kv[0])
                ls_key = kv[:2]
                k_ms = ls_key_fields(k, idx_bits)[0]
                if k != INT64_MAX and k_ms <= target:
                    break
                if dp_lb_hit or (k != INT64_MAX and k_ms <= lb_int):
                    # the bound the side search proved (or a candidate at the bound) is met
                    proof["proven"] = True
                    break
                if dp_ok and k != INT64_MAX and dp_tried_at != k_ms:
                    dp_tried_at = k_ms
                    try:
                        proven, dp_ms, cand, proof = self.prove_below(prob, dp_tried_at, opts, lb=lb_int,
                                                                      stats=proof)
                    except (E.TooLarge, err.TooLarge, E.InvariantViolation, err.InvariantViolation):
                        # a shape the state-space search does not take (key width, > 8 nodes):
                        # no proof, the local search's result stands
                        dp_ok, proven, cand = False, False, None
                    if cand is not None:
                        dp_cand = (dp_ms, cand)
                    if proven:
                        break
            stats = {"walkers": walkers_done, "waves": waves, "rounds": rounds_total,
                     "moves_scheduled_max": rounds_total * 32, "lower_bound": target, "stop_ms": stop_ms}
            if proof is not None:
                stats["proof"] = proof
            kernel, evaluated = "local", walkers_done
        else:
            src = SRC_SUBSTREAM if source is None else source
            seed_used = opts.seed if seed is None else seed
            base_lo = 0 if lo is None else lo
            base_hi = n_idx if hi is None else hi
            a, b = _shard(base_hi - base_lo, rank, world)
            self.search_sampled(nprob, src, seed_used, base_lo + a, base_lo + b, kbest)
            kernel, evaluated = "sampled", base_hi - base_lo
        ev1.record()
        if on_launched is not None:
            on_launched(mode)
        if shared is not None:
            shared.collect(best)
        # key hand-off: the combined key, bound-and-prune's counters (they sit at the start of
        # the workspace, which the replay's launch below reuses) and the replay id, in one
        # launch (sat_key_finish) and later one read-back
        do_replay = replay and nprob.grid and mode in ("exhaustive", "sampled")
        # (bound-and-prune replays too: its key always holds a real candidate -- the seed bound
        # comes from a candidate of the same space, which the search itself reaches)
        if mode == "local" and ls_key is not None:
            both, replay_out = ls_key, None         # read back after the last wave already
        else:
            key_dev, ids_dev = self._key_finish(best, nprob.grid, group, world, idx_bits, n_idx,
                                                extra=bnb_ws, want_ids=do_replay,
                                                check_range=mode == "exhaustive")
            replay_out = self.schedule(nprob, src, seed_used, ids_dev=ids_dev) if do_replay else None
            both = key_dev.cpu().tolist()
        key = both[:2]
        if bnb_ws is not None:
            cnt = both[2:]
            stats.update(pruned_tasks=cnt[1], pair_nodes=cnt[2])
        ev1.synchronize()
        dev_s = ev0.elapsed_time(ev1) / 1e3
        if shared is not None:
            stats = {**(stats or {}), "shared_incumbent": True}
        if nprob.grid:
            k = int(key[0])
            if k == INT64_MAX:
                raise err.PlanFailure("search produced no candidate")
            makespan = float(k >> idx_bits)
            index = k & ((1 << idx_bits) - 1)
            if mode == "local":
                ms_, rounds_, index = ls_key_fields(k, idx_bits)
                makespan = float(ms_)
                stats["winner_rounds"] = rounds_
                ls_state = self._walker_state(ls_states, index, prob.J, group, world)
                if dp_cand is not None and dp_cand[0] < makespan:
                    # the state-space search found a shorter candidate than every walker
                    makespan, ls_state = float(dp_cand[0]), (list(dp_cand[1][0]), list(dp_cand[1][1]))
                    stats["winner"] = "sat_search_dp"
                proven_opt = proof is not None and bool(proof.get("proven"))
        else:
            hi_bits, index = int(key[0]), int(key[1])
            if hi_bits == INT64_MAX:
                raise err.PlanFailure("search produced no candidate")
            makespan = float(np.array([hi_bits], dtype=np.int64).view(np.float64)[0])
        return SearchResult(makespan=makespan, index=index, source=src, seed=seed_used, evaluated=evaluated,
                            kernel=kernel, exhaustive=mode == "exhaustive",
                            launches=self.launches - launches0, job_steps=job_steps,
                            device_seconds=dev_s, wall_seconds=time.perf_counter() - t0,
                            stats=stats, idx_bits=idx_bits, state=ls_state, replay=replay_out,
                            proven=mode == "local" and proven_opt)

    def _key_finish(self, best, grid: bool, group, world: int, idx_bits: int, n_idx: int, *, extra=None,
                    extra_words: int = 3, want_ids: bool = False, check_range: bool = False):
        """(key [2 (+ extra_words counters)] int64, replay id [1] or None) on the device:
        `_combine_dev` plus the replay id through one sat_key_finish launch (grid keys; float
        keys combine through `_combine_dev`).  With several ranks the key is all-reduced (MIN)
        in between (the counters stay this rank's)."""
        torch = self.torch
        if not grid:
            return _combine_dev(best, grid, group, world), None
        n_extra = extra_words if extra is not None else 0
        out = torch.empty(2 + n_extra, dtype=torch.int64, device=self.device)
        ids = torch.empty(1, dtype=torch.int64, device=self.device) if want_ids else None
        stream = _vp(self.stream())
        one_launch = world == 1
        self._check(self.lib.sat_key_finish(
            _vp(best.data_ptr()), 2, _vp(extra.data_ptr()) if extra is not None else None, n_extra,
            _vp(out.data_ptr()), _vp(ids.data_ptr()) if (ids is not None and one_launch) else None,
            idx_bits, n_idx & ((1 << 64) - 1), int(check_range), stream), what="sat_key_finish")
        self.launches += 1
        if not one_launch:
            import torch.distributed as dist

            dist.all_reduce(out[:1], op=dist.ReduceOp.MIN, group=group)
            if ids is not None:
                self._check(self.lib.sat_key_finish(None, 2, None, 0, _vp(out.data_ptr()), _vp(ids.data_ptr()),
                                                    idx_bits, n_idx & ((1 << 64) - 1), int(check_range), stream),
                            what="sat_key_finish")
                self.launches += 1
        return out, ids

    def _walker_state(self, ls_states, index: int, J: int, group, world: int):
        """The winning walker's final (options, order), recorded by its search launch (on the
        rank that ran it; other ranks receive it through an all-reduce MAX of zeros)."""
        torch = self.torch
        if world == 1:                  # one rank: the row itself, one copy (no kernels)
            for lo, hi, buf in ls_states:
                if lo <= index < hi:
                    out = buf[(index - lo) * 2 * J:(index - lo + 1) * 2 * J].cpu().tolist()
                    return out[:J], out[J:]
        v = torch.zeros(2 * J, dtype=torch.int32, device=self.device)
        for lo, hi, buf in ls_states:
            if lo <= index < hi:
                v = buf[(index - lo) * 2 * J:(index - lo + 1) * 2 * J].to(torch.int32)
        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(v, op=dist.ReduceOp.MAX, group=group)
        out = v.cpu().tolist()
        return out[:J], out[J:]

    @staticmethod
    def _tree_ok(prob: SearchProblem) -> bool:
        return (prob.N == 1 and prob.time_mode == TIME_GRID and 3 <= prob.J <= 20
                and not prob.release_i32.any() and int(prob.radix.sum()) <= 384)


def _rank_world(group):
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return 0, 1
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _shard(n: int, rank: int, world: int) -> tuple:
    """Contiguous block partition of [0, n)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def _combine(best, grid: bool, group, world: int):
    """All-reduce MIN of the packed key (grid) or of (makespan bits, then index) (float)."""
    return _combine_dev(best, grid, group, world).cpu().tolist()


def _combine_dev(best, grid: bool, group, world: int):
    """`_combine` left on the device (the reduced key tensor)."""
    import torch

    key = best.clone()
    empty = key == -1                                   # all-ones = nothing found on this rank
    key = torch.where(empty, torch.full_like(key, INT64_MAX), key)
    if world > 1:
        import torch.distributed as dist

        if grid:
            dist.all_reduce(key[:1], op=dist.ReduceOp.MIN, group=group)
        else:
            ms = key[:1].clone()
            dist.all_reduce(ms, op=dist.ReduceOp.MIN, group=group)
            idx = torch.where(key[:1] == ms, key[1:], torch.full_like(key[1:], INT64_MAX))
            dist.all_reduce(idx, op=dist.ReduceOp.MIN, group=group)
            key = torch.cat([ms, idx])
    return key
