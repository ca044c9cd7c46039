"""Binary op-log format shared by the oracle and the CUDA path (input only).

This module holds NO arithmetic of the method: it only records simrd API calls
(PAPER.md Doc A §4.2: make_tensor / get / release / rematerialize)
plus the output-condition ENSURE record (reading C-11) into a flat little-endian
u32 array, and performs program-level liveness bookkeeping (how much memory the
*program itself* holds live) so a budget can be expressed as a fraction of the
program's own peak (reading C-16).

Layout (all u32 words):

    header[16]:
      0 magic 'DTRL' (0x4C525444)   1 version (1)
      2 n_tensors                   3 n_edges (sum of parent-list lengths)
      4 n_ops                       5 model_id
      6,7   base_compute (u64: sum of MAKE compute costs)
      8,9   peak_live    (u64: max over MAKE of sum mem of tensors with rho>0)
      10,11 peak_total   (u64: sum of all mem)
      12,13 seed (u64)              14 max_parents    15 reserved (0)
    mem[n_tensors]                  (memory units, >= 1)
    cost[n_tensors]                 (compute units, >= 1)
    par_off[n_tensors + 1]          (CSR offsets into par)
    par[n_edges]                    (parent ids, deduplicated, first-occurrence order, < child id)
    ops[n_ops]                      (op << 29 | id)

Opcodes: MAKE=1 (id = the new tensor, must equal the running count),
GET=2, RELEASE=3, REMAT=4, ENSURE=5, DEBUG_EVICT=6 (test fixtures only).
"""
from __future__ import annotations

import numpy as np

MAGIC = 0x4C525444
VERSION = 1
HEADER_WORDS = 16

OP_MAKE = 1
OP_GET = 2
OP_RELEASE = 3
OP_REMAT = 4
OP_ENSURE = 5
OP_DEBUG_EVICT = 6
OP_SHIFT = 29
ID_MASK = (1 << OP_SHIFT) - 1

OP_NAMES = {OP_MAKE: "MAKE", OP_GET: "GET", OP_RELEASE: "RELEASE",
            OP_REMAT: "REMAT", OP_ENSURE: "ENSURE", OP_DEBUG_EVICT: "DEBUG_EVICT"}

# Input-domain limits (reading C-14): keep every product of the exact score
# comparison inside 128 bits and the clock inside u32 with a 16x thrash kill.
MAX_MEM = (1 << 32) - 1
MAX_COST = (1 << 31) - 1
MAX_BASE = 1 << 27


class LogBuilder:
    """Records a simrd call sequence. Validates the preconditions P:149-156."""

    def __init__(self, model_id: int = 0, seed: int = 0):
        self.model_id = model_id
        self.seed = seed
        self.mem: list[int] = []
        self.cost: list[int] = []
        self.par_off: list[int] = [0]
        self.par: list[int] = []
        self.ops: list[int] = []
        self.rho: list[int] = []
        self.live_mem = 0
        self.peak_live = 0
        self.max_parents = 0

    @property
    def n(self) -> int:
        return len(self.mem)

    def make(self, mem: int, cost: int, parents=()) -> int:
        mem = int(mem)
        cost = int(cost)
        if not (1 <= mem <= MAX_MEM) or not (1 <= cost <= MAX_COST):
            raise ValueError(f"mem/cost out of range: {mem}, {cost}")
        seen = set()
        plist = []
        for p in parents:
            p = int(p)
            if p in seen:
                continue  # P is a set: keep the first occurrence
            if not (0 <= p < self.n):
                raise ValueError(f"unknown parent {p}")
            if self.rho[p] <= 0:
                raise ValueError(f"parent {p} has no external reference")
            seen.add(p)
            plist.append(p)
        t = self.n
        self.mem.append(mem)
        self.cost.append(cost)
        self.par.extend(plist)
        self.par_off.append(len(self.par))
        self.max_parents = max(self.max_parents, len(plist))
        self.rho.append(1)
        self.ops.append((OP_MAKE << OP_SHIFT) | t)
        self.live_mem += mem
        self.peak_live = max(self.peak_live, self.live_mem)
        return t

    def get(self, t: int) -> None:
        if self.rho[t] <= 0:
            raise ValueError("get on a released tensor")
        self.rho[t] += 1
        self.ops.append((OP_GET << OP_SHIFT) | t)

    def release(self, t: int) -> None:
        if self.rho[t] <= 0:
            raise ValueError("release on a released tensor")
        self.rho[t] -= 1
        if self.rho[t] == 0:
            self.live_mem -= self.mem[t]
        self.ops.append((OP_RELEASE << OP_SHIFT) | t)

    def remat(self, t: int) -> None:
        self.ops.append((OP_REMAT << OP_SHIFT) | t)

    def ensure(self, t: int) -> None:
        self.ops.append((OP_ENSURE << OP_SHIFT) | t)

    def debug_evict(self, t: int) -> None:
        self.ops.append((OP_DEBUG_EVICT << OP_SHIFT) | t)

    def build(self) -> np.ndarray:
        n = self.n
        base = sum(self.cost)
        if base > MAX_BASE:
            raise ValueError(f"base compute {base} exceeds {MAX_BASE}")
        hdr = np.zeros(HEADER_WORDS, dtype=np.uint32)
        hdr[0] = MAGIC
        hdr[1] = VERSION
        hdr[2] = n
        hdr[3] = len(self.par)
        hdr[4] = len(self.ops)
        hdr[5] = self.model_id
        for k, v in ((6, base), (8, self.peak_live), (10, sum(self.mem)), (12, self.seed)):
            hdr[k] = v & 0xFFFFFFFF
            hdr[k + 1] = (v >> 32) & 0xFFFFFFFF
        hdr[14] = self.max_parents
        return np.concatenate([
            hdr,
            np.asarray(self.mem, dtype=np.uint32),
            np.asarray(self.cost, dtype=np.uint32),
            np.asarray(self.par_off, dtype=np.uint32),
            np.asarray(self.par, dtype=np.uint32),
            np.asarray(self.ops, dtype=np.uint32),
        ]).astype(np.uint32)


def assemble(mem, cost, par_off, par, ops, *, model_id=0, seed=0, peak_live=None) -> np.ndarray:
    """Vectorised assembly for very large generated logs (stress configs)."""
    mem = np.asarray(mem, dtype=np.uint32)
    cost = np.asarray(cost, dtype=np.uint32)
    par_off = np.asarray(par_off, dtype=np.uint32)
    par = np.asarray(par, dtype=np.uint32)
    ops = np.asarray(ops, dtype=np.uint32)
    n = len(mem)
    base = int(cost.astype(np.uint64).sum())
    if base > MAX_BASE:
        raise ValueError(f"base compute {base} exceeds {MAX_BASE}")
    total = int(mem.astype(np.uint64).sum())
    if peak_live is None:
        peak_live = total
    hdr = np.zeros(HEADER_WORDS, dtype=np.uint32)
    hdr[0] = MAGIC
    hdr[1] = VERSION
    hdr[2] = n
    hdr[3] = len(par)
    hdr[4] = len(ops)
    hdr[5] = model_id
    for k, v in ((6, base), (8, int(peak_live)), (10, total), (12, seed)):
        hdr[k] = v & 0xFFFFFFFF
        hdr[k + 1] = (v >> 32) & 0xFFFFFFFF
    deg = np.diff(par_off.astype(np.int64))
    hdr[14] = int(deg.max()) if n else 0
    return np.concatenate([hdr, mem, cost, par_off, par, ops]).astype(np.uint32)


class LogView:
    """Read-only view of an encoded log (header fields + sections)."""

    def __init__(self, words: np.ndarray):
        w = np.asarray(words, dtype=np.uint32)
        if int(w[0]) != MAGIC or int(w[1]) != VERSION:
            raise ValueError("not a DTR log")
        self.words = w
        self.n = int(w[2])
        self.n_edges = int(w[3])
        self.n_ops = int(w[4])
        self.model_id = int(w[5])
        u64 = lambda k: int(w[k]) | (int(w[k + 1]) << 32)
        self.base = u64(6)
        self.peak_live = u64(8)
        self.peak_total = u64(10)
        self.seed = u64(12)
        self.max_parents = int(w[14])
        o = HEADER_WORDS
        n, e = self.n, self.n_edges
        self.mem = w[o:o + n]; o += n
        self.cost = w[o:o + n]; o += n
        self.par_off = w[o:o + n + 1]; o += n + 1
        self.par = w[o:o + e]; o += e
        self.ops = w[o:o + self.n_ops]; o += self.n_ops
        if o != len(w):
            raise ValueError("log length mismatch")

    def parents(self, t: int):
        return [int(x) for x in self.par[self.par_off[t]:self.par_off[t + 1]]]

    def budget(self, permille: int) -> int:
        """B = floor(peak_live * permille / 1000) (reading C-16)."""
        return self.peak_live * int(permille) // 1000


def log_words_len(words) -> int:
    return len(words)
