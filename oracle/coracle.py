"""ctypes wrapper of oracle/oracle.c -- TEST INFRASTRUCTURE ONLY (checker / CPU baseline).

``build()`` compiles oracle.c with gcc into oracle/_build/liboracle.so (git-ignored,
travels to the GPU box with the snapshot).  Problems come from
``saturn_oracle.build`` (the oracle's own restatement), never from the product.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "_build", "liboracle.so")
OMAX_G = 32

_vp = ctypes.c_void_p


class OProblem(ctypes.Structure):
    _fields_ = [("J", ctypes.c_int), ("N", ctypes.c_int), ("Cmax", ctypes.c_int),
                ("radix", _vp), ("gpus", _vp), ("mask", _vp), ("dur", _vp), ("node_gpus", _vp),
                ("release", _vp), ("init_free", _vp)]


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-o", LIB + ".tmp", SRC],
                   check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
        _lib.oracle_search.argtypes = [_vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_int, _vp, _vp]
        _lib.oracle_makespans.argtypes = [_vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          _vp]
        _lib.oracle_eval.argtypes = [_vp, _vp, _vp, _vp, _vp]
        _lib.oracle_eval.restype = ctypes.c_double
        _lib.oracle_decode.argtypes = [_vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _vp, _vp]
        _lib.oracle_local_search.argtypes = [_vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                             ctypes.c_int, _vp, _vp, _vp]
        _lib.oracle_local_search.restype = ctypes.c_double
        _lib.oracle_ls_search.argtypes = [_vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
        _lib.oracle_local_search_from.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]
        _lib.oracle_local_search_from.restype = ctypes.c_double
    return _lib


SOURCES = {"index": 0, "substream": 1, "seed": 2, "greedy": 4}


class CProblem:
    def __init__(self, prob):
        J, N = prob.J, prob.N
        C = max(prob.radix)
        self.J, self.N = J, N
        self.radix = np.array(prob.radix, dtype=np.int32)
        self.gpus = np.zeros((J, C), dtype=np.int32)
        self.mask = np.zeros((J, C), dtype=np.uint32)
        self.dur = np.zeros((J, C, N), dtype=np.float64)
        for j in range(J):
            for o in range(prob.radix[j]):
                self.gpus[j, o] = prob.gpus[j][o]
                for n in range(N):
                    if prob.eligible[j][o][n]:
                        self.mask[j, o] |= np.uint32(1 << n)
                        self.dur[j, o, n] = prob.dur[j][o][n]
        self.node_gpus = np.array(prob.node_gpus, dtype=np.int32)
        self.release = np.array(prob.release, dtype=np.float64)
        self.init = np.zeros((N, OMAX_G), dtype=np.float64)
        for n in range(N):
            self.init[n, : prob.node_gpus[n]] = prob.init_free[n]
        s = OProblem()
        s.J, s.N, s.Cmax = J, N, C
        s.radix, s.gpus, s.mask, s.dur = (self.radix.ctypes.data, self.gpus.ctypes.data, self.mask.ctypes.data,
                                          self.dur.ctypes.data)
        s.node_gpus, s.release, s.init_free = self.node_gpus.ctypes.data, self.release.ctypes.data, self.init.ctypes.data
        self.s = s

    def search(self, source="index", seed=0, lo=0, hi=None, threads=0):
        hi = math.prod(int(r) for r in self.radix) * math.factorial(self.J) if hi is None else hi
        ms = ctypes.c_double()
        ident = ctypes.c_uint64()
        rc = lib().oracle_search(ctypes.byref(self.s), SOURCES[source], seed & ((1 << 64) - 1), lo, hi, threads,
                                 ctypes.byref(ms), ctypes.byref(ident))
        assert rc == 0
        return ms.value, ident.value

    def makespans(self, source="index", seed=0, lo=0, hi=1):
        out = np.empty(hi - lo, dtype=np.float64)
        lib().oracle_makespans(ctypes.byref(self.s), SOURCES[source], seed & ((1 << 64) - 1), lo, hi,
                               out.ctypes.data)
        return out

    def decode(self, ident, source="index", seed=0):
        opt = np.zeros(self.J, dtype=np.int32)
        ordr = np.zeros(self.J, dtype=np.int32)
        lib().oracle_decode(ctypes.byref(self.s), SOURCES[source], seed & ((1 << 64) - 1), ident,
                            opt.ctypes.data, ordr.ctypes.data)
        return opt.tolist(), ordr.tolist()

    def local_search(self, walker, source="substream", seed=0, max_rounds=4096, stop_ms=-1):
        """(makespan, options, order, rounds) of one local-search walker (oracle.c semantics;
        stop_ms >= 0 ends the walk once its makespan is <= stop_ms)."""
        opt = np.zeros(self.J, dtype=np.int32)
        ordr = np.zeros(self.J, dtype=np.int32)
        rounds = ctypes.c_int()
        ms = lib().oracle_local_search(ctypes.byref(self.s), SOURCES[source], seed & ((1 << 64) - 1), walker,
                                       max_rounds, int(stop_ms), opt.ctypes.data, ordr.ctypes.data,
                                       ctypes.byref(rounds))
        return ms, opt.tolist(), ordr.tolist(), rounds.value

    def local_search_from(self, opts, order, max_rounds=4096, stop_ms=-1):
        """(makespan, options, order, rounds) of the walk started at the candidate (opts, order)."""
        opt = np.array(opts, dtype=np.int32)
        ordr = np.array(order, dtype=np.int32)
        rounds = ctypes.c_int()
        ms = lib().oracle_local_search_from(ctypes.byref(self.s), max_rounds, int(stop_ms), opt.ctypes.data,
                                            ordr.ctypes.data, ctypes.byref(rounds))
        return ms, opt.tolist(), ordr.tolist(), rounds.value

    def ls_search(self, source="substream", seed=0, lo=0, hi=1, max_rounds=4096, threads=0, stop_ms=-1):
        ms = ctypes.c_double()
        ident = ctypes.c_uint64()
        lib().oracle_ls_search(ctypes.byref(self.s), SOURCES[source], seed & ((1 << 64) - 1), lo, hi, max_rounds,
                               int(stop_ms), threads, ctypes.byref(ms), ctypes.byref(ident))
        return ms.value, ident.value

    def eval(self, opts, order):
        o = np.array(opts, dtype=np.int32)
        r = np.array(order, dtype=np.int32)
        st = np.zeros(self.J, dtype=np.float64)
        nd = np.zeros(self.J, dtype=np.int32)
        ms = lib().oracle_eval(ctypes.byref(self.s), o.ctypes.data, r.ctypes.data, st.ctypes.data, nd.ctypes.data)
        return ms, st.tolist(), nd.tolist()
