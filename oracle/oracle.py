"""ctypes wrapper of the C oracle (oracle/simrd_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs. The product package
(paper_2006_09616_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "simrd_oracle.c")
LIB = os.path.join(HERE, "libsimrd_oracle.so")

H_DTR, H_DTR_EQ, H_LRU, H_SIZE, H_MSPS, H_LOCAL, H_RANDOM, H_DTR_FULL, H_ESTAR = range(9)
HEURISTICS = {"dtr": H_DTR, "dtr_eq": H_DTR_EQ, "lru": H_LRU, "size": H_SIZE,
              "msps": H_MSPS, "local": H_LOCAL, "random": H_RANDOM, "dtr_full": H_DTR_FULL, "estar": H_ESTAR}
# the D.1 ablation h'(s, m, c) (reading C-23): id = 16 + 4*c + 2*m + s
ABL_C = ("estar", "eqclass", "local", "no")


def abl_id(c: str, m: bool, s: bool) -> int:
    return 16 + 4 * ABL_C.index(c) + 2 * int(bool(m)) + int(bool(s))


for _c in ABL_C:
    for _m in (0, 1):
        for _s in (0, 1):
            HEURISTICS[f"abl_{_c}_{'m' if _m else 'x'}{'s' if _s else 'x'}"] = abl_id(_c, _m, _s)
OK, PRECOND, OOM, THRASH, CAPACITY, STATE, DECISION_CAP = 0, 2, 3, 4, 5, 6, 8

TRACE_DTYPE = np.dtype([("clock", "<u8"), ("id", "<u4"), ("pad", "<u4"), ("num", "<u8"), ("den", "<u8")])
RESULT_DTYPE = np.dtype([("cell_id", "<u4"), ("status", "<u4"), ("records_done", "<u4"), ("n_trace", "<u4"),
                         ("clock", "<u8"), ("base", "<u8"), ("decisions", "<u8"), ("remats", "<u8"),
                         ("computations", "<u8"), ("peak_M", "<u8"), ("trace_hash", "<u8")])

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2). Building the checker is not using it."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-Wno-unused-parameter",
                               "-shared", "-fPIC", "-o", tmp, SRC, "-lpthread"])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(LIB)
            P = C.c_void_p
            u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
            L.oracle_create.restype = P
            L.oracle_create.argtypes = [i32, u64, u64, u32, u64, u64, i32]
            L.oracle_destroy.argtypes = [P]
            L.oracle_make.restype = i32
            L.oracle_make.argtypes = [P, u64, u64, C.POINTER(u32), u32, C.POINTER(u32)]
            for f in ("oracle_get", "oracle_release", "oracle_rematerialize", "oracle_ensure",
                      "oracle_debug_evict"):
                getattr(L, f).restype = i32
                getattr(L, f).argtypes = [P, u32]
            L.oracle_set_budget.argtypes = [P, u64]
            L.oracle_scores.restype = u64
            L.oracle_scores.argtypes = [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(u32), u64]
            L.oracle_neighbourhood.restype = u32
            L.oracle_neighbourhood.argtypes = [P, u32, C.POINTER(u32), u32]
            L.oracle_estar.restype = u32
            L.oracle_estar.argtypes = [P, u32, C.POINTER(u32), u32]
            L.oracle_state.argtypes = [P, C.POINTER(u64)]
            L.oracle_tensors.argtypes = [P, C.POINTER(C.c_uint8), C.POINTER(u64), C.POINTER(u64),
                                         C.POINTER(C.c_int64)]
            L.oracle_uf_root_cost_sum.restype = u64
            L.oracle_uf_root_cost_sum.argtypes = [P]
            L.oracle_uf_roots.argtypes = [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(C.c_int64)]
            L.oracle_result.argtypes = [P, C.c_void_p]
            L.oracle_trace.restype = u64
            L.oracle_trace.argtypes = [P, C.c_void_p, u64]
            L.oracle_replay.restype = i32
            L.oracle_replay.argtypes = [C.POINTER(u32), u64, i32, u64, u64, u32, u64, i32, i32,
                                        C.c_void_p, C.c_void_p, u64]
            L.oracle_set_dealloc.argtypes = [P, i32]
            _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


DEALLOC = {"v2": 0, "v1": 1, "eager": 2, "ignore": 3}


def replay(words: np.ndarray, heuristic: int, budget: int, *, seed: int = 0, thrash_kill: int = 16,
           max_decisions: int = 0, e_mode: int = 0, trace_cap: int = 0, dealloc: int = 0):
    """Replay a whole log. Returns (result_row: np.void, trace: np.ndarray)."""
    L = lib()
    w = np.ascontiguousarray(words, dtype=np.uint32)
    res = np.zeros(1, dtype=RESULT_DTYPE)
    tr = np.zeros(max(trace_cap, 1), dtype=TRACE_DTYPE)
    L.oracle_replay(_ptr(w, C.c_uint32), len(w), int(heuristic), int(budget), int(seed),
                    int(thrash_kill), int(max_decisions), int(e_mode), int(dealloc),
                    res.ctypes.data_as(C.c_void_p), tr.ctypes.data_as(C.c_void_p), int(trace_cap))
    r = res[0]
    return r, tr[: min(int(r["decisions"]), trace_cap)]


class Runtime:
    """Per-call oracle runtime mirroring the boundary's dtr_* calls (fixtures, tests)."""

    def __init__(self, heuristic=H_DTR, budget=(1 << 62), seed=0, thrash_kill=0, max_decisions=0,
                 trace_cap=1 << 16, e_mode=0, dealloc=0):
        self.L = lib()
        self.h = self.L.oracle_create(int(heuristic), int(budget), int(seed), int(thrash_kill),
                                      int(max_decisions), int(trace_cap), int(e_mode))
        self.L.oracle_set_dealloc(self.h, int(dealloc))
        self.trace_cap = trace_cap

    def __del__(self):
        try:
            if self.h:
                self.L.oracle_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def compute(self, mem, cost, parents=()):
        ps = np.asarray(list(parents), dtype=np.uint32)
        out = C.c_uint32(0)
        rc = self.L.oracle_make(self.h, int(mem), int(cost), _ptr(ps, C.c_uint32) if len(ps) else None,
                                len(ps), C.byref(out))
        return rc, out.value

    def get(self, t):
        return self.L.oracle_get(self.h, int(t))

    def release(self, t):
        return self.L.oracle_release(self.h, int(t))

    def rematerialize(self, t):
        return self.L.oracle_rematerialize(self.h, int(t))

    def ensure(self, t):
        return self.L.oracle_ensure(self.h, int(t))

    def debug_evict(self, t):
        return self.L.oracle_debug_evict(self.h, int(t))

    def set_budget(self, B):
        self.L.oracle_set_budget(self.h, int(B))

    def scores(self):
        cap = 1 << 16
        num = np.zeros(cap, np.uint64)
        den = np.zeros(cap, np.uint64)
        ids = np.zeros(cap, np.uint32)
        k = self.L.oracle_scores(self.h, _ptr(num, C.c_uint64), _ptr(den, C.c_uint64), _ptr(ids, C.c_uint32), cap)
        return {int(ids[i]): (int(num[i]), int(den[i])) for i in range(k)}

    def neighbourhood(self, t):
        cap = 1 << 16
        out = np.zeros(cap, np.uint32)
        k = self.L.oracle_neighbourhood(self.h, int(t), _ptr(out, C.c_uint32), cap)
        return sorted(int(x) for x in out[:k])

    def estar(self, t):
        cap = 1 << 16
        out = np.zeros(cap, np.uint32)
        k = self.L.oracle_estar(self.h, int(t), _ptr(out, C.c_uint32), cap)
        return sorted(int(x) for x in out[:k])

    def state(self):
        s = np.zeros(8, np.uint64)
        self.L.oracle_state(self.h, _ptr(s, C.c_uint64))
        keys = ("clock", "M", "B", "n", "decisions", "remats", "computations", "status")
        return {k: int(v) for k, v in zip(keys, s)}

    def tensors(self):
        n = self.state()["n"]
        fl = np.zeros(max(n, 1), np.uint8)
        rho = np.zeros(max(n, 1), np.uint64)
        ell = np.zeros(max(n, 1), np.uint64)
        la = np.zeros(max(n, 1), np.int64)
        self.L.oracle_tensors(self.h, _ptr(fl, C.c_uint8), _ptr(rho, C.c_uint64), _ptr(ell, C.c_uint64),
                              _ptr(la, C.c_int64))
        return fl[:n], rho[:n], ell[:n], la[:n]

    def uf_root_cost_sum(self):
        return int(self.L.oracle_uf_root_cost_sum(self.h))

    def uf_roots(self):
        n = self.state()["n"]
        r = np.zeros(max(n, 1), np.uint64)
        c = np.zeros(max(n, 1), np.uint64)
        m = np.zeros(max(n, 1), np.int64)
        self.L.oracle_uf_roots(self.h, _ptr(r, C.c_uint64), _ptr(c, C.c_uint64), _ptr(m, C.c_int64))
        return r[:n], c[:n], m[:n]

    def result(self):
        res = np.zeros(1, dtype=RESULT_DTYPE)
        self.L.oracle_result(self.h, res.ctypes.data_as(C.c_void_p))
        return res[0]

    def trace(self):
        tr = np.zeros(max(self.trace_cap, 1), dtype=TRACE_DTYPE)
        k = self.L.oracle_trace(self.h, tr.ctypes.data_as(C.c_void_p), self.trace_cap)
        return tr[: min(k, self.trace_cap)]


NEG_INF = -(1 << 63)
