"""Thin ctypes binding of libdtr.so (include/dtr.h). Argument marshalling only:
every step of a replay runs in the library's CUDA kernels. There is no CPU
fallback -- if the extension is missing the import fails loudly.

PyTorch supplies device memory (torch.empty(..., device='cuda')) and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTR_LIB") or os.path.join(HERE, "libdtr.so")   # DTR_LIB: probes only

DTR_OK, DTR_E_INVAL, DTR_E_PRECOND, DTR_E_OOM, DTR_E_THRASH = 0, 1, 2, 3, 4
DTR_E_CAPACITY, DTR_E_STATE, DTR_E_CUDA, DTR_E_DECISION_CAP = 5, 6, 7, 8
H_DTR, H_DTR_EQ, H_LRU, H_SIZE, H_MSPS, H_LOCAL, H_RANDOM, H_DTR_FULL, H_ESTAR = range(9)
HEURISTICS = {"dtr": H_DTR, "dtr_eq": H_DTR_EQ, "lru": H_LRU, "size": H_SIZE, "msps": H_MSPS,
              "local": H_LOCAL, "random": H_RANDOM, "dtr_full": H_DTR_FULL, "estar": H_ESTAR}
# the D.1 ablation h'(s, m, c) (include/dtr.h DTR_H_ABLATION): id = 16 + 4*c + 2*m + s
ABL_C = ("estar", "eqclass", "local", "no")


def abl_id(c, m, s):
    return 16 + 4 * ABL_C.index(c) + 2 * int(bool(m)) + int(bool(s))


for _c in ABL_C:
    for _m in (0, 1):
        for _s in (0, 1):
            HEURISTICS[f"abl_{_c}_{'m' if _m else 'x'}{'s' if _s else 'x'}"] = abl_id(_c, _m, _s)
ENGINE_CTA, ENGINE_GRID = 1, 2
GRID_MIN_TENSORS = 65536   # include/dtr.h DTR_GRID_MIN_TENSORS: logs this large replay on the whole-GPU engine
DEALLOC = {"v2": 0, "v1": 1, "eager": 2, "ignore": 3}
STATUS_NAMES = {0: "ok", 1: "inval", 2: "precond", 3: "oom", 4: "thrash_killed", 5: "capacity",
                6: "state", 7: "cuda", 8: "decision_cap"}

TRACE_DTYPE = np.dtype([("clock", "<u8"), ("id", "<u4"), ("pad", "<u4"), ("num", "<u8"), ("den", "<u8")])
RESULT_DTYPE = np.dtype([("cell_id", "<u4"), ("status", "<u4"), ("records_done", "<u4"), ("n_trace", "<u4"),
                         ("clock", "<u8"), ("base", "<u8"), ("decisions", "<u8"), ("remats", "<u8"),
                         ("computations", "<u8"), ("peak_M", "<u8"), ("trace_hash", "<u8"),
                         ("cand_evals", "<u8"), ("score_bytes", "<u8"), ("wall_ns", "<u8")])
CELL_DTYPE = np.dtype([("log_offset", "<u8"), ("budget", "<u8"), ("seed", "<u8"), ("max_decisions", "<u8"),
                       ("trace_offset", "<u8"), ("trace_cap", "<u8"), ("heuristic", "<u4"),
                       ("thrash_kill", "<u4"), ("cell_id", "<u4"), ("dealloc", "<u4")])
ADV_DTYPE = np.dtype([("n", "<u4"), ("budget", "<u4"), ("heuristic", "<u4"), ("cell_id", "<u4"),
                      ("seed", "<u8"), ("trace_offset", "<u8"), ("trace_cap", "<u4"), ("reserved", "<u4")])
assert TRACE_DTYPE.itemsize == 32 and RESULT_DTYPE.itemsize == 96 and CELL_DTYPE.itemsize == 64
assert ADV_DTYPE.itemsize == 40

# every symbol include/dtr.h declares
EXPORTS = ["dtr_strerror", "dtr_last_cuda_error", "dtr_version", "dtr_batch_workspace_bytes", "dtr_cta_class",
           "dtr_replay_batch", "dtr_replay_batch_host", "dtr_create", "dtr_destroy", "dtr_compute", "dtr_get",
           "dtr_release", "dtr_rematerialize", "dtr_ensure", "dtr_stats", "dtr_trace", "dtr_debug_evict",
           "dtr_debug_set_budget", "dtr_debug_scores", "dtr_debug_state", "dtr_pool_argmin", "dtr_adversary_workspace_bytes",
           "dtr_adversary_batch"]


class DtrError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        super().__init__(f"{what}: {STATUS_NAMES.get(code, code)} ({code})")


class _Config(C.Structure):
    _fields_ = [("budget", C.c_uint64), ("seed", C.c_uint64), ("max_decisions", C.c_uint64),
                ("trace_cap", C.c_uint64), ("heuristic", C.c_uint32), ("thrash_kill", C.c_uint32),
                ("cap_tensors", C.c_uint32), ("cap_edges", C.c_uint32), ("device", C.c_int),
                ("dealloc", C.c_uint32), ("stream", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libdtr.so not built ({LIB_PATH}); run __graft_entry__.build() -- "
                          "there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    L.dtr_strerror.restype = C.c_char_p
    L.dtr_strerror.argtypes = [i32]
    L.dtr_last_cuda_error.restype = C.c_char_p
    L.dtr_version.restype = i32
    L.dtr_batch_workspace_bytes.restype = i32
    L.dtr_batch_workspace_bytes.argtypes = [P, u32, u32, C.POINTER(u64)]
    L.dtr_cta_class.restype = i32
    L.dtr_cta_class.argtypes = [u32, u32, u32, C.POINTER(u32)]
    L.dtr_replay_batch.restype = i32
    L.dtr_replay_batch.argtypes = [P, P, P, u32, u32, P, u64, P, P, P]
    L.dtr_pool_argmin.restype = i32
    L.dtr_pool_argmin.argtypes = [P, u32, P, P, P]
    L.dtr_adversary_workspace_bytes.restype = i32
    L.dtr_adversary_workspace_bytes.argtypes = [P, u32, C.POINTER(u64)]
    L.dtr_adversary_batch.restype = i32
    L.dtr_adversary_batch.argtypes = [P, P, u32, P, u64, P, P, P, P]
    L.dtr_replay_batch_host.restype = i32
    L.dtr_replay_batch_host.argtypes = [P, u64, P, u32, u32, P, P, u64, P]
    L.dtr_create.restype = i32
    L.dtr_create.argtypes = [C.POINTER(_Config), C.POINTER(P)]
    L.dtr_destroy.restype = i32
    L.dtr_destroy.argtypes = [P]
    L.dtr_compute.restype = i32
    L.dtr_compute.argtypes = [P, u32, u32, P, u32, C.POINTER(u32)]
    for f in ("dtr_get", "dtr_release", "dtr_rematerialize", "dtr_ensure", "dtr_debug_evict"):
        getattr(L, f).restype = i32
        getattr(L, f).argtypes = [P, u32]
    L.dtr_stats.restype = i32
    L.dtr_stats.argtypes = [P, P]
    L.dtr_trace.restype = i32
    L.dtr_trace.argtypes = [P, P, u64, C.POINTER(u64)]
    L.dtr_debug_set_budget.restype = i32
    L.dtr_debug_set_budget.argtypes = [P, u64]
    L.dtr_debug_scores.restype = i32
    L.dtr_debug_scores.argtypes = [P, P, P, P, u64, C.POINTER(u64)]
    L.dtr_debug_state.restype = i32
    L.dtr_debug_state.argtypes = [P, P, u64, C.POINTER(u64)]
    return L


lib = _load()


def _check(rc, what):
    if rc != DTR_OK:
        if rc == DTR_E_CUDA:
            raise DtrError(rc, f"{what} [{lib.dtr_last_cuda_error().decode()}]")
        raise DtrError(rc, what)


def _np_ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


# ---------------------------------------------------------------------------
# Batches
# ---------------------------------------------------------------------------

def pack_logs(logs):
    """Concatenate encoded logs; returns (words, offsets)."""
    offs, cur = [], 0
    for w in logs:
        offs.append(cur)
        cur += len(w)
    words = np.concatenate([np.asarray(w, dtype=np.uint32) for w in logs]) if logs else np.zeros(0, np.uint32)
    return words, offs


def make_cells(log_offsets, specs, trace_caps=None):
    """specs: list of dicts {log (index), budget, heuristic, seed=0, thrash_kill=16,
    max_decisions=0}. Returns (cells array, total trace records)."""
    cells = np.zeros(len(specs), dtype=CELL_DTYPE)
    tcur = 0
    for i, s in enumerate(specs):
        cells[i]["log_offset"] = log_offsets[s["log"]]
        cells[i]["budget"] = int(s["budget"])
        cells[i]["seed"] = int(s.get("seed", 0))
        cells[i]["max_decisions"] = int(s.get("max_decisions", 0))
        cap = int(trace_caps[i]) if trace_caps is not None else 0
        cells[i]["trace_offset"] = tcur
        cells[i]["trace_cap"] = cap
        tcur += cap
        cells[i]["heuristic"] = int(s["heuristic"])
        cells[i]["thrash_kill"] = int(s.get("thrash_kill", 16))
        cells[i]["cell_id"] = int(s.get("cell_id", i))
        cells[i]["dealloc"] = int(s.get("dealloc", 0))
    return cells, tcur


def cell_dims(words, cells):
    dims = np.zeros(3 * len(cells), dtype=np.uint32)
    for i, c in enumerate(cells):
        o = int(c["log_offset"])
        dims[3 * i] = words[o + 2]
        dims[3 * i + 1] = words[o + 3]
        dims[3 * i + 2] = c["heuristic"]
    return dims


def workspace_bytes(dims, engine):
    out = C.c_uint64(0)
    _check(lib.dtr_batch_workspace_bytes(_np_ptr(dims), len(dims) // 3, engine, C.byref(out)),
           "dtr_batch_workspace_bytes")
    return out.value


def cta_class(n_tensors, n_edges, heuristic):
    """Shared-memory class (0 small, 1 staged, 2 global) of a CTA-engine cell."""
    out = C.c_uint32(0)
    _check(lib.dtr_cta_class(int(n_tensors), int(n_edges), int(heuristic), C.byref(out)), "dtr_cta_class")
    return out.value


def replay_batch(d_words, d_cells, h_dims, n_cells, engine, d_ws, ws_bytes, d_rows, d_trace, stream):
    """dtr_replay_batch on device pointers (ints) with host dims (np.uint32),
    asynchronous on `stream` (int handle)."""
    _check(lib.dtr_replay_batch(d_words, d_cells, _np_ptr(h_dims), n_cells, engine, d_ws, ws_bytes, d_rows,
                                d_trace, stream), "dtr_replay_batch")


def replay_batch_host(words, cells, engine=0, trace_total=0, stream=None):
    """dtr_replay_batch_host: host arrays in, host rows (+ traces) out."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    cells = np.ascontiguousarray(cells, dtype=CELL_DTYPE)
    rows = np.zeros(len(cells), dtype=RESULT_DTYPE)
    tr = np.zeros(max(trace_total, 1), dtype=TRACE_DTYPE) if trace_total else None
    _check(lib.dtr_replay_batch_host(_np_ptr(words), len(words), _np_ptr(cells), len(cells), engine,
                                     _np_ptr(rows), _np_ptr(tr), trace_total, stream),
           "dtr_replay_batch_host")
    return rows, tr


class DeviceBatch:
    """A batch whose inputs are resident in HBM (torch-allocated), replayed by
    dtr_replay_batch with one call per step."""

    def __init__(self, logs, specs, engine=ENGINE_CTA, trace_caps=None, device=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        words, offs = pack_logs(logs)
        cells, ttot = make_cells(offs, specs, trace_caps)
        dims = cell_dims(words, cells)
        self.engine = engine
        self.n_cells = len(cells)
        self.ws_bytes = workspace_bytes(dims, engine)
        dev = self.device
        self.words = torch.from_numpy(words.view(np.int32)).to(dev)
        self.cells = torch.from_numpy(cells.view(np.uint8)).to(dev)
        self.h_dims = dims
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.rows = torch.zeros(self.n_cells * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.trace_total = ttot
        self.trace = torch.zeros(max(ttot, 1) * TRACE_DTYPE.itemsize, dtype=torch.uint8, device=dev) if ttot else None
        self.h_cells = cells
        self.h_words = words
        self.specs = specs

    def launches_per_run(self):
        """Kernel launches one run() makes: grid engine one per cell; CTA engine one
        per run of consecutive cells of one shared-memory class (dtr.cu)."""
        if self.engine == ENGINE_GRID:
            return self.n_cells
        d = self.h_dims.reshape(-1, 3)
        cls = [cta_class(int(a), int(b), int(c)) for a, b, c in d]
        return sum(1 for i in range(len(cls)) if i == 0 or cls[i] != cls[i - 1])

    def run(self, stream=None):
        # every dtr_* entry point works on the current device: make it the one that owns the buffers
        with self.torch.cuda.device(self.device):
            s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
            replay_batch(self.words.data_ptr(), self.cells.data_ptr(), self.h_dims, self.n_cells, self.engine,
                         self.ws.data_ptr(), self.ws_bytes, self.rows.data_ptr(),
                         self.trace.data_ptr() if self.trace is not None else None, s.cuda_stream)

    def pool_argmin(self, cell=0, stream=None):
        """dtr_pool_argmin over the grid-engine workspace (call after run()).
        Returns (num, den, id, score_bytes, cand_evals) as a device tensor of 5 int64."""
        torch = self.torch
        assert self.engine == ENGINE_GRID
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if not hasattr(self, "_pa_out"):
            self._pa_out = torch.zeros(5, dtype=torch.int64, device=self.device)
        log_ptr = self.words.data_ptr() + 4 * int(self.h_cells[cell]["log_offset"])
        _check(lib.dtr_pool_argmin(log_ptr, int(self.h_cells[cell]["heuristic"]), self.ws.data_ptr(),
                                   self._pa_out.data_ptr(), s.cuda_stream), "dtr_pool_argmin")
        return self._pa_out

    def result_rows(self):
        return self.rows.cpu().numpy().view(RESULT_DTYPE).copy()

    def traces(self):
        if self.trace is None:
            return None
        return self.trace.cpu().numpy().view(TRACE_DTYPE).copy()

    def cell_trace(self, i, tr=None):
        tr = self.traces() if tr is None else tr
        c = self.h_cells[i]
        return tr[int(c["trace_offset"]): int(c["trace_offset"]) + int(c["trace_cap"])]


# ---------------------------------------------------------------------------
# Theorem 2 adversary batches (App. B; include/dtr.h dtr_adversary_batch)
# ---------------------------------------------------------------------------

class AdversaryBatch:
    """Runs of the online adversary, one CTA each, one launch per run() call.
    runs: dicts {n, budget, heuristic, seed=0, trace_cap=0, cell_id=i}."""

    def __init__(self, runs, device=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        a = np.zeros(len(runs), dtype=ADV_DTYPE)
        toff = 0
        for i, r in enumerate(runs):
            a[i]["n"] = int(r["n"])
            a[i]["budget"] = int(r["budget"])
            a[i]["heuristic"] = int(r["heuristic"])
            a[i]["cell_id"] = int(r.get("cell_id", i))
            a[i]["seed"] = int(r.get("seed", 0))
            a[i]["trace_cap"] = int(r.get("trace_cap", 0))
            a[i]["trace_offset"] = toff
            toff += int(a[i]["trace_cap"])
        self.h_runs = a
        self.n_runs = len(runs)
        self.p_off = np.concatenate([[0], np.cumsum(a["n"].astype(np.int64))])
        nb = C.c_uint64(0)
        _check(lib.dtr_adversary_workspace_bytes(_np_ptr(a), len(a), C.byref(nb)), "dtr_adversary_workspace_bytes")
        dev = self.device
        self.ws_bytes = int(nb.value)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.d_runs = torch.from_numpy(a.view(np.uint8).copy()).to(dev)
        self.rows = torch.zeros(len(a) * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.parents = torch.zeros(int(self.p_off[-1]), dtype=torch.int32, device=dev)
        self.trace_total = toff
        self.trace = torch.zeros(max(toff, 1) * TRACE_DTYPE.itemsize, dtype=torch.uint8, device=dev) if toff else None

    def run(self, stream=None):
        with self.torch.cuda.device(self.device):
            s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
            _check(lib.dtr_adversary_batch(self.d_runs.data_ptr(), _np_ptr(self.h_runs), self.n_runs,
                                           self.ws.data_ptr(), self.ws_bytes, self.rows.data_ptr(),
                                           self.parents.data_ptr(),
                                           self.trace.data_ptr() if self.trace is not None else None, s.cuda_stream),
                   "dtr_adversary_batch")

    def result_rows(self):
        return self.rows.cpu().numpy().view(RESULT_DTYPE).copy()

    def run_parents(self, i, all_parents=None):
        p = self.parents.cpu().numpy().view(np.uint32) if all_parents is None else all_parents
        return p[int(self.p_off[i]): int(self.p_off[i + 1])].copy()

    def run_trace(self, i):
        if self.trace is None:
            return None
        tr = self.trace.cpu().numpy().view(TRACE_DTYPE)
        o, c = int(self.h_runs[i]["trace_offset"]), int(self.h_runs[i]["trace_cap"])
        return tr[o: o + c].copy()


# ---------------------------------------------------------------------------
# Per-call runtime (simrd external API)
# ---------------------------------------------------------------------------

class Runtime:
    def __init__(self, heuristic=H_DTR, budget=(1 << 62), seed=0, thrash_kill=0, max_decisions=0,
                 trace_cap=1 << 16, cap_tensors=1 << 12, cap_edges=1 << 14, device=0, stream=None, dealloc=0):
        cfg = _Config(budget, seed, max_decisions, trace_cap, heuristic, thrash_kill, cap_tensors, cap_edges,
                      device, dealloc, stream)
        h = C.c_void_p()
        _check(lib.dtr_create(C.byref(cfg), C.byref(h)), "dtr_create")
        self.h = h
        self.cap_tensors = cap_tensors

    def close(self):
        if getattr(self, "h", None):
            lib.dtr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def compute(self, mem, cost, parents=()):
        ps = np.asarray(list(parents), dtype=np.uint32)
        out = C.c_uint32(0)
        rc = lib.dtr_compute(self.h, int(mem), int(cost), _np_ptr(ps), len(ps), C.byref(out))
        return rc, out.value

    def get(self, t):
        return lib.dtr_get(self.h, int(t))

    def release(self, t):
        return lib.dtr_release(self.h, int(t))

    def rematerialize(self, t):
        return lib.dtr_rematerialize(self.h, int(t))

    def ensure(self, t):
        return lib.dtr_ensure(self.h, int(t))

    def debug_evict(self, t):
        return lib.dtr_debug_evict(self.h, int(t))

    def set_budget(self, B):
        _check(lib.dtr_debug_set_budget(self.h, int(B)), "dtr_debug_set_budget")

    def scores(self):
        cap = self.cap_tensors + 1
        num = np.zeros(cap, np.uint64)
        den = np.zeros(cap, np.uint64)
        ids = np.zeros(cap, np.uint32)
        n = C.c_uint64(0)
        _check(lib.dtr_debug_scores(self.h, _np_ptr(num), _np_ptr(den), _np_ptr(ids), cap, C.byref(n)),
               "dtr_debug_scores")
        return {int(ids[i]): (int(num[i]), int(den[i])) for i in range(n.value)}

    def state(self):
        """Residency of every created tensor: 0 uncomputed, 1 resident, 2 evicted, 3 banished."""
        cap = self.cap_tensors + 1
        out = np.zeros(cap, np.uint8)
        n = C.c_uint64(0)
        _check(lib.dtr_debug_state(self.h, _np_ptr(out), cap, C.byref(n)), "dtr_debug_state")
        return out[: min(n.value, cap)].copy()

    def stats(self):
        r = np.zeros(1, dtype=RESULT_DTYPE)
        _check(lib.dtr_stats(self.h, _np_ptr(r)), "dtr_stats")
        return r[0]

    def trace(self, cap=1 << 20):
        buf = np.zeros(cap, dtype=TRACE_DTYPE)
        n = C.c_uint64(0)
        _check(lib.dtr_trace(self.h, _np_ptr(buf), cap, C.byref(n)), "dtr_trace")
        return buf[: min(n.value, cap)]
