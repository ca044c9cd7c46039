// dtr.cu -- kernels and C ABI of libdtr.so (see include/dtr.h).
//
// Engines:
//   K6 cta_engine   one CTA per simulation: leader thread 0 runs the control,
//                   the CTA scores the pool and reduces the argmin (bar.sync).
//   K7 grid_engine  one cooperative persistent grid per simulation: leader is
//                   block 0 / thread 0; every SM scores a slice of the pool,
//                   per-block partial argmins are reduced by block 0.
//   percall_engine  the per-call API: one CTA applies one record to persistent
//                   device state (children kept as linked lists because future
//                   children are unknown).
// K1/K2 (component maintenance + aggregation) run inside the leader
// (leader.cuh); K3+K4 (score + argmin) are team_argmin() below; K5 (MSPS
// closure) is the warp-cooperative msps_closure().
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>
#include <algorithm>

#include "engine.cuh"
#include "leader.cuh"
#include "../../include/dtr.h"

namespace cg = cooperative_groups;
using namespace dtr;

#define CTA_THREADS 256
#define GRID_THREADS 512
#define GRID_MSPS_WARPS 1024

// ---------------------------------------------------------------------------
// K5: warp-cooperative MSPS closure e_R(t): evicted ancestors reached through
// evicted parents.  Per-warp visited bitmap + queue in global
// memory; returns the sum of c0 over e_R(t) in every lane.
// ---------------------------------------------------------------------------
__device__ u64 msps_closure(const Graph &g, const Work &w, u32 t, u32 *bm, u32 *q, volatile u32 *tail,
                            u64 &bytes) {
  u32 lane = threadIdx.x & 31;
  if (lane == 0) *tail = 0;
  __syncwarp();
  u64 sum = 0;
  auto visit = [&](u32 p) {
    bytes += 8;   // parent id + its state word
    if (!is_evicted(w.state[p])) return;
    bytes += 12;  // cost + its parent CSR offsets
    u32 bit = 1u << (p & 31);
    u32 old = atomicOr(&bm[p >> 5], bit);
    if (old & bit) return;
    sum += __ldg(&g.cost[p]);
    u32 pos = atomicAdd((u32 *)tail, 1u);
    q[pos] = p;
  };
  u32 b = __ldg(&g.par_off[t]), e = __ldg(&g.par_off[t + 1]);
  for (u32 j = b + lane; j < e; j += 32) visit(__ldg(&g.par[j]));
  __syncwarp();
  u32 head = 0, tl = *tail;
  __syncwarp();
  while (head < tl) {
    for (u32 i = head + lane; i < tl; i += 32) {
      u32 x = q[i];
      u32 xb = __ldg(&g.par_off[x]), xe = __ldg(&g.par_off[x + 1]);
      for (u32 j = xb; j < xe; j++) visit(__ldg(&g.par[j]));
    }
    __syncwarp();
    head = tl;
    tl = *tail;
    __syncwarp();
  }
  for (u32 i = lane; i < tl; i += 32) bm[q[i] >> 5] = 0;
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  return sum;
}

// ---------------------------------------------------------------------------
// K3 + K4: score every pool member of a slice and return the slice argmin.
// rank/size: this thread's index in the team; wrank/wsize: warp index (MSPS).
// ---------------------------------------------------------------------------
__device__ Cand team_score(const Graph &g, const Work &w, const Cmd &cmd, u32 rank, u32 size, u32 wrank,
                           u32 wsize, u32 msps_warps, volatile u32 *msps_tail, u64 &bytes, u64 &evals) {
  Cand best = cand_none();
  const u32 P = cmd.pool_size;
  if (cmd.heur == H_MSPS) {
    if (wrank >= msps_warps) return best;
    u32 *bm = w.msps_bm + (size_t)wrank * w.msps_words;
    u32 *q = w.msps_q + (size_t)wrank * (g.n + 1);
    u32 lane = threadIdx.x & 31;
    u32 nw = wsize < msps_warps ? wsize : msps_warps;
    for (u32 i = wrank; i < P; i += nw) {
      u32 t = w.pool_ids[i];
      u64 sum = msps_closure(g, w, t, bm, q, msps_tail + ((threadIdx.x >> 5)), bytes);
      if (lane == 0) {
        bytes += 4 + 8 + 8;   // pool id; mem, cost; parent CSR offsets
        evals++;
        Cand c;
        c.num = (u64)__ldg(&g.cost[t]) + sum;
        c.den = __ldg(&g.mem[t]);
        c.id = t;
        if (cand_less(c, best)) best = c;
      }
    }
    return best;
  }
  for (u32 i = rank; i < P; i += size) {
    u32 t = w.pool_ids[i];
    Cand c;
    score_one(g, w, cmd.heur, cmd.clock, cmd.seed, cmd.decisions, t, c.num, c.den, bytes);
    evals++;
    c.id = t;
    if (cand_less(c, best)) best = c;
  }
  return best;
}

// per-call OP_SCORES: write every pool member's score (MSPS included)
__device__ void team_scores_out(const Graph &g, const Work &w, const Cmd &cmd, u32 rank, u32 size,
                                volatile u32 *msps_tail, u64 *onum, u64 *oden, u32 *oid) {
  const u32 P = cmd.pool_size;
  if (cmd.heur == H_MSPS) {
    u32 wr = rank >> 5, ws = (size + 31) >> 5, lane = threadIdx.x & 31;
    u32 *bm = w.msps_bm + (size_t)wr * w.msps_words;
    u32 *q = w.msps_q + (size_t)wr * (g.n + 1);
    for (u32 i = wr; i < P; i += ws) {
      u32 t = w.pool_ids[i];
      u64 junk = 0;
      u64 sum = msps_closure(g, w, t, bm, q, msps_tail + (threadIdx.x >> 5), junk);
      if (lane == 0) { onum[i] = (u64)g.cost[t] + sum; oden[i] = g.mem[t]; oid[i] = t; }
    }
    return;
  }
  for (u32 i = rank; i < P; i += size) {
    u32 t = w.pool_ids[i];
    u64 num, den, junk = 0;
    score_one(g, w, cmd.heur, cmd.clock, cmd.seed, cmd.decisions, t, num, den, junk);
    onum[i] = num; oden[i] = den; oid[i] = t;
  }
}

// ---------------------------------------------------------------------------
// Initialisation (team-parallel): zero per-tensor state, free lists, and the
// children CSR of the log (count, scan, fill).
// ---------------------------------------------------------------------------
struct ScanSmem {
  u32 warp_tot[32];
  u32 carry;
};

// exclusive scan of cnt[0..n) into off[0..n], off[n] = total; cnt reset to 0.
// Executed by ONE block.
__device__ void block_scan_excl(u32 *cnt, u32 *off, u32 n, ScanSmem &sm) {
  u32 T = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = (T + 31) >> 5;
  u32 chunk = (n + T - 1) / T;
  u32 lo = tid * chunk, hi = lo + chunk < n ? lo + chunk : n;
  u32 local = 0;
  for (u32 i = lo; i < hi; i++) local += cnt[i];
  // inclusive warp scan
  u32 v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (u32)o) v += y;
  }
  if (lane == 31) sm.warp_tot[wid] = v;
  __syncthreads();
  if (wid == 0) {
    u32 x = lane < nw ? sm.warp_tot[lane] : 0;
    u32 y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= (u32)o) y += z;
    }
    if (lane < nw) sm.warp_tot[lane] = y - x;   // exclusive warp offsets
    if (lane == nw - 1) sm.carry = y;
  }
  __syncthreads();
  u32 run = sm.warp_tot[wid] + v - local;
  for (u32 i = lo; i < hi; i++) { u32 c = cnt[i]; off[i] = run; run += c; cnt[i] = 0; }
  if (tid == 0) off[n] = sm.carry;
  __syncthreads();
}

template <class Sync>
__device__ void init_sim(const Graph &g, const Work &w, u32 heur, u32 msps_warps, u32 rank, u32 size,
                         bool scan_block, ScanSmem &ssm, Sync sync) {
  const u32 n = g.n;
  for (u32 i = rank; i <= n; i += size) {
    w.state[i] = 0; w.la[i] = 0; w.rho[i] = 0; w.ell[i] = 0; w.pool_pos[i] = NONE;
    if (heur == H_DTR) { w.stamp[i] = 0; w.comp_free[i] = n - i; }   // pops 0, 1, 2, ...
    if (heur == H_DTR_EQ) w.node_of[i] = NONE;
    if (!g.linked) w.ch_fill[i] = 0;
    else w.ch_head[i] = NONE;
  }
  if (heur == H_DTR_EQ) {
    u64 cap = 2 * (u64)n + 64;
    for (u64 i = rank; i < cap; i += size) w.uf_remap[i] = NONE;
  }
  if (heur == H_MSPS) {
    u64 words = (u64)w.msps_words * msps_warps;
    for (u64 i = rank; i < words; i += size) w.msps_bm[i] = 0;
  }
  sync();
  if (g.linked) return;
  for (u32 c = rank; c < n; c += size) {
    u32 b = __ldg(&g.par_off[c]), e = __ldg(&g.par_off[c + 1]);
    for (u32 j = b; j < e; j++) atomicAdd(&w.ch_fill[__ldg(&g.par[j])], 1u);
  }
  sync();
  if (scan_block) block_scan_excl(w.ch_fill, w.ch_off, n, ssm);
  sync();
  for (u32 c = rank; c < n; c += size) {
    u32 b = __ldg(&g.par_off[c]), e = __ldg(&g.par_off[c + 1]);
    for (u32 j = b; j < e; j++) {
      u32 p = __ldg(&g.par[j]);
      u32 k = atomicAdd(&w.ch_fill[p], 1u);
      w.ch[w.ch_off[p] + k] = c;
    }
  }
  sync();
  // deterministic child order (ascending id): results never depend on it, but
  // union-find tree shapes (and so the byte accounting) do
  for (u32 p = rank; p < n; p += size) {
    u32 b = w.ch_off[p], e = w.ch_off[p + 1];
    for (u32 i = b + 1; i < e; i++) {
      u32 x = w.ch[i], j = i;
      while (j > b && w.ch[j - 1] > x) { w.ch[j] = w.ch[j - 1]; j--; }
      w.ch[j] = x;
    }
  }
  sync();
}

// block-wide sum of two counters; result valid in thread 0
__device__ void block_sum2(u64 &a, u64 &b, RedSmem &sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { a += __shfl_xor_sync(0xffffffffu, a, o); b += __shfl_xor_sync(0xffffffffu, b, o); }
  u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) { sm.warp[wid].num = a; sm.warp[wid].den = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0; b = 0;
    for (u32 i = 0; i < nw; i++) { a += sm.warp[i].num; b += sm.warp[i].den; }
  }
}

__device__ void init_scalars(Scalars &s, const dtr_cell &cell, u32 n) {
  memset(&s, 0, sizeof(Scalars));
  s.B = cell.budget;
  s.seed = cell.seed;
  s.max_decisions = cell.max_decisions;
  s.trace_cap = cell.trace_cap;
  s.trace_off = cell.trace_offset;
  s.heuristic = cell.heuristic;
  s.thrash_kill = cell.thrash_kill;
  s.cell_id = cell.cell_id;
  s.comp_free_top = n + 1;
  s.uf_cap = 2 * n + 64;
  s.trace_hash = 14695981039346656037ull;
}

__device__ void write_row(dtr_result &r, const Scalars &s) {
  r.cell_id = s.cell_id;
  r.status = s.status;
  r.records_done = s.records_done;
  r.n_trace = (u32)s.trace_n;
  r.clock = s.clock;
  r.base = s.base_so_far;
  r.decisions = s.decisions;
  r.remats = s.remats;
  r.computations = s.computations;
  r.peak_M = s.peak_M;
  r.trace_hash = s.trace_hash;
  r.cand_evals = 0;
  r.score_bytes = 0;
}

// ---------------------------------------------------------------------------
// Plan: per-cell workspace offsets (exclusive scan of carve() sizes).
// ws layout: [u64 off[n_cells]] [pad] [cells ...]
// ---------------------------------------------------------------------------
__host__ __device__ inline u64 cell_bytes(u32 n, u32 E, u32 heur, u32 engine) {
  Work w;
  u32 mw = engine == DTR_ENGINE_GRID ? GRID_MSPS_WARPS : CTA_THREADS / 32;
  return (carve(w, 0, n, E, heur, 0, mw) + 255) & ~255ull;
}

__host__ __device__ inline u64 ws_header_bytes(u32 n_cells) {
  // offsets + grid command + per-block partials
  return ((u64)n_cells * 8 + 256 + 4096 * sizeof(Cand) + 255) & ~255ull;
}

__global__ void plan_kernel(const u32 *dims, u32 n_cells, u32 engine, u64 ws_bytes, u64 *off, u32 *ok) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  u64 cur = ws_header_bytes(n_cells), mx = 0;
  for (u32 i = 0; i < n_cells; i++) {
    u64 b = cell_bytes(dims[3 * i], dims[3 * i + 1], dims[3 * i + 2], engine);
    if (engine == DTR_ENGINE_GRID) { off[i] = cur; mx = b > mx ? b : mx; }
    else { off[i] = cur; cur += b; }
  }
  u64 need = engine == DTR_ENGINE_GRID ? cur + mx : cur;
  *ok = need <= ws_bytes;
}

// ---------------------------------------------------------------------------
// K6: one CTA per simulation.
// ---------------------------------------------------------------------------
struct __align__(16) CtaShared {
  Graph g;
  Work w;
  Scalars s;
  Leader L;
  Cmd cmd;
  RedSmem red;
  ScanSmem scan;
  u32 msps_tail[CTA_THREADS / 32];
};

struct CtaSync {
  __device__ void operator()() const { __syncthreads(); }
};

__global__ void __launch_bounds__(CTA_THREADS) cta_engine(const u32 *words, const dtr_cell *cells, u32 n_cells,
                                                          char *ws, dtr_result *rows, dtr_evict_rec *trace) {
  __shared__ CtaShared sh;
  const u32 tid = threadIdx.x;
  const u64 *off = (const u64 *)ws;
  const u32 ci = blockIdx.x;
  if (ci >= n_cells) return;
  const u32 *ok = (const u32 *)(ws + (u64)n_cells * 8);
  if (!*ok) {
    if (tid == 0) {
      dtr_result r; memset(&r, 0, sizeof r);
      r.cell_id = cells[ci].cell_id; r.status = ST_CAPACITY;
      rows[ci] = r;
    }
    return;
  }
  if (tid == 0) {
    const dtr_cell cell = cells[ci];
    graph_from_log(sh.g, words + cell.log_offset);
    carve(sh.w, (uintptr_t)(ws + off[ci]), sh.g.n, sh.g.E, cell.heuristic, 0, CTA_THREADS / 32);
    sh.g.ch_off = sh.w.ch_off;
    sh.g.ch = sh.w.ch;
    init_scalars(sh.s, cell, sh.g.n);
    sh.L.g = &sh.g; sh.L.w = &sh.w; sh.L.s = &sh.s;
    sh.L.trace = (trace && cell.trace_cap) ? trace + cell.trace_offset : nullptr;
    sh.L.op_idx = 0; sh.L.op_end = sh.g.nops;
    sh.L.phase = PH_OP; sh.L.post = 0; sh.L.root = 0; sh.L.percall = 0; sh.L.free_size = 0;
  }
  __syncthreads();
  init_sim(sh.g, sh.w, sh.s.heuristic, CTA_THREADS / 32, tid, blockDim.x, true, sh.scan, CtaSync());
  Cand res = cand_none();
  bool have = false;
  u64 bytes = 0, evals = 0;
  for (;;) {
    if (tid == 0) {
      u32 kind = sh.L.resume(have, res);
      have = false;
      sh.cmd.kind = kind;
      sh.cmd.pool_size = sh.s.pool_size;
      sh.cmd.clock = sh.s.clock;
      sh.cmd.decisions = sh.s.decisions;
      sh.cmd.seed = sh.s.seed;
      sh.cmd.heur = sh.s.heuristic;
    }
    __syncthreads();
    if (sh.cmd.kind != CMD_ARGMIN) break;
    Cand best = team_score(sh.g, sh.w, sh.cmd, tid, blockDim.x, tid >> 5, blockDim.x >> 5, CTA_THREADS / 32,
                           sh.msps_tail, bytes, evals);
    best = block_argmin(best, sh.red);
    if (tid == 0) { res = best; have = true; }
  }
  block_sum2(bytes, evals, sh.red);
  if (tid == 0) {
    write_row(rows[ci], sh.s);
    rows[ci].score_bytes = bytes;
    rows[ci].cand_evals = evals;
  }
}

// ---------------------------------------------------------------------------
// K7: the whole GPU on one simulation (cooperative launch).
// ---------------------------------------------------------------------------
struct __align__(16) GridShared {
  Graph g;
  Work w;
  Scalars s;
  Leader L;
  Cmd cmd;
  RedSmem red;
  ScanSmem scan;
  u32 msps_tail[GRID_THREADS / 32];
};

struct GridSync {
  __device__ void operator()() const { cg::this_grid().sync(); }
};

__global__ void __launch_bounds__(GRID_THREADS) grid_engine(const u32 *words, const dtr_cell *cells, u32 n_cells,
                                                            u32 ci, char *ws, dtr_result *rows,
                                                            dtr_evict_rec *trace) {
  __shared__ GridShared sh;
  cg::grid_group grid = cg::this_grid();
  const u32 tid = threadIdx.x;
  const u64 *off = (const u64 *)ws;
  const u32 *ok = (const u32 *)(ws + (u64)n_cells * 8);
  Cmd *gcmd = (Cmd *)(ws + (u64)n_cells * 8 + 64);
  Cand *partials = (Cand *)(ws + (u64)n_cells * 8 + 256);
  if (!*ok) {
    if (blockIdx.x == 0 && tid == 0) {
      dtr_result r; memset(&r, 0, sizeof r);
      r.cell_id = cells[ci].cell_id; r.status = ST_CAPACITY;
      rows[ci] = r;
    }
    return;
  }
  const dtr_cell cell = cells[ci];
  if (tid == 0) {
    graph_from_log(sh.g, words + cell.log_offset);
    carve(sh.w, (uintptr_t)(ws + off[ci]), sh.g.n, sh.g.E, cell.heuristic, 0, GRID_MSPS_WARPS);
    sh.g.ch_off = sh.w.ch_off;
    sh.g.ch = sh.w.ch;
    if (blockIdx.x == 0) {
      init_scalars(sh.s, cell, sh.g.n);
      sh.L.g = &sh.g; sh.L.w = &sh.w; sh.L.s = &sh.s;
      sh.L.trace = (trace && cell.trace_cap) ? trace + cell.trace_offset : nullptr;
      sh.L.op_idx = 0; sh.L.op_end = sh.g.nops;
      sh.L.phase = PH_OP; sh.L.post = 0; sh.L.root = 0; sh.L.percall = 0; sh.L.free_size = 0;
    }
  }
  __syncthreads();
  const u32 rank = blockIdx.x * blockDim.x + tid, size = gridDim.x * blockDim.x;
  const u32 wrank = rank >> 5, wsize = size >> 5;
  u64 *gstats = (u64 *)(ws + (u64)n_cells * 8 + 128);   // [bytes, evals]
  if (rank == 0) { gstats[0] = 0; gstats[1] = 0; }
  init_sim(sh.g, sh.w, cell.heuristic, GRID_MSPS_WARPS, rank, size, blockIdx.x == 0, sh.scan, GridSync());
  Cand res = cand_none();
  bool have = false;
  u64 bytes = 0, evals = 0;
  for (;;) {
    if (blockIdx.x == 0 && tid == 0) {
      u32 kind = sh.L.resume(have, res);
      have = false;
      Cmd c;
      c.kind = kind; c.pool_size = sh.s.pool_size; c.clock = sh.s.clock; c.decisions = sh.s.decisions;
      c.seed = sh.s.seed; c.heur = sh.s.heuristic; c.pad = 0;
      *gcmd = c;
    }
    grid.sync();
    if (tid == 0) {
      Cmd c;
      c.kind = __ldcg(&gcmd->kind); c.pool_size = __ldcg(&gcmd->pool_size); c.clock = __ldcg(&gcmd->clock);
      c.decisions = __ldcg(&gcmd->decisions); c.seed = __ldcg(&gcmd->seed); c.heur = __ldcg(&gcmd->heur);
      sh.cmd = c;
    }
    __syncthreads();
    if (sh.cmd.kind != CMD_ARGMIN) break;
    Cand best = team_score(sh.g, sh.w, sh.cmd, rank, size, wrank, wsize, GRID_MSPS_WARPS, sh.msps_tail,
                           bytes, evals);
    best = block_argmin(best, sh.red);
    if (tid == 0) partials[blockIdx.x] = best;
    grid.sync();
    if (blockIdx.x == 0 && tid < 32) {
      Cand c = cand_none();
      for (u32 b = tid; b < gridDim.x; b += 32) {
        Cand d;
        d.num = __ldcg(&partials[b].num); d.den = __ldcg(&partials[b].den); d.id = __ldcg(&partials[b].id);
        if (cand_less(d, c)) c = d;
      }
      c = warp_argmin(c);
      if (tid == 0) { res = c; have = true; }
    }
  }
  block_sum2(bytes, evals, sh.red);
  if (tid == 0) { atomicAdd(&gstats[0], bytes); atomicAdd(&gstats[1], evals); }
  grid.sync();
  if (blockIdx.x == 0 && tid == 0) {
    write_row(rows[ci], sh.s);
    rows[ci].score_bytes = __ldcg(&gstats[0]);
    rows[ci].cand_evals = __ldcg(&gstats[1]);
  }
}

// ---------------------------------------------------------------------------
// Per-call engine: apply ONE record to the persistent state of a runtime.
// ---------------------------------------------------------------------------
struct PercallArgs {
  Graph g;          // tensor table arrays of the runtime (linked children)
  Work w;
  dtr_evict_rec *trace;
  u64 *onum, *oden;
  u32 *oid;
  u32 init;         // first launch: initialise state
};

__global__ void __launch_bounds__(CTA_THREADS) percall_engine(PercallArgs a) {
  __shared__ CtaShared sh;
  const u32 tid = threadIdx.x;
  if (tid == 0) {
    sh.g = a.g;
    sh.w = a.w;
    sh.g.ch_head = sh.w.ch_head; sh.g.e_next = sh.w.e_next; sh.g.e_child = sh.w.e_child;
    sh.s = *a.w.sc;
  }
  __syncthreads();
  if (a.init) {
    init_sim(sh.g, sh.w, sh.s.heuristic, CTA_THREADS / 32, tid, blockDim.x, true, sh.scan, CtaSync());
    if (tid == 0) *a.w.sc = sh.s;
    return;
  }
  if (tid == 0) {
    sh.L.g = &sh.g; sh.L.w = &sh.w; sh.L.s = &sh.s;
    sh.L.trace = a.trace;
    sh.L.op_idx = 0; sh.L.op_end = 1;
    sh.L.phase = PH_OP; sh.L.post = 0; sh.L.root = 0; sh.L.percall = 1; sh.L.free_size = 0;
    sh.s.last_rc = ST_OK;
  }
  __syncthreads();
  Cand res = cand_none();
  bool have = false;
  for (;;) {
    if (tid == 0) {
      u32 kind = sh.L.resume(have, res);
      have = false;
      sh.cmd.kind = kind; sh.cmd.pool_size = sh.s.pool_size; sh.cmd.clock = sh.s.clock;
      sh.cmd.decisions = sh.s.decisions; sh.cmd.seed = sh.s.seed; sh.cmd.heur = sh.s.heuristic;
    }
    __syncthreads();
    if (sh.cmd.kind == CMD_DONE) break;
    if (sh.cmd.kind == CMD_SCORES) {
      team_scores_out(sh.g, sh.w, sh.cmd, tid, blockDim.x, sh.msps_tail, a.onum, a.oden, a.oid);
      if (tid == 0) sh.s.n_scores = sh.cmd.pool_size;
      __syncthreads();
      continue;
    }
    u64 junk = 0, junk2 = 0;
    Cand best = team_score(sh.g, sh.w, sh.cmd, tid, blockDim.x, tid >> 5, blockDim.x >> 5, CTA_THREADS / 32,
                           sh.msps_tail, junk, junk2);
    best = block_argmin(best, sh.red);
    if (tid == 0) { res = best; have = true; }
  }
  if (tid == 0) *a.w.sc = sh.s;
}

// ===========================================================================
// Host ABI
// ===========================================================================
static thread_local char g_cuda_err[256] = "";

static int cuda_fail(cudaError_t e) {
  snprintf(g_cuda_err, sizeof g_cuda_err, "%s", cudaGetErrorString(e));
  return DTR_E_CUDA;
}
#define CK(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return cuda_fail(_e); } while (0)

extern "C" {

const char *dtr_strerror(int code) {
  switch (code) {
    case DTR_OK: return "ok";
    case DTR_E_INVAL: return "invalid argument";
    case DTR_E_PRECOND: return "precondition violated";
    case DTR_E_OOM: return "out of memory (pool empty while over budget)";
    case DTR_E_THRASH: return "thrash kill-switch";
    case DTR_E_CAPACITY: return "capacity exceeded";
    case DTR_E_STATE: return "runtime stopped by an earlier error";
    case DTR_E_CUDA: return "CUDA error";
    case DTR_E_DECISION_CAP: return "decision cap reached";
  }
  return "unknown";
}

const char *dtr_last_cuda_error(void) { return g_cuda_err; }

int dtr_version(void) { return 1; }

int dtr_batch_workspace_bytes(const uint32_t *dims, uint32_t n_cells, uint32_t engine, uint64_t *bytes_out) {
  if (!bytes_out || (n_cells && !dims) || (engine != DTR_ENGINE_CTA && engine != DTR_ENGINE_GRID)) return DTR_E_INVAL;
  u64 cur = ws_header_bytes(n_cells), mx = 0;
  for (u32 i = 0; i < n_cells; i++) {
    if (dims[3 * i + 2] > H_RANDOM) return DTR_E_INVAL;
    u64 b = cell_bytes(dims[3 * i], dims[3 * i + 1], dims[3 * i + 2], engine);
    if (engine == DTR_ENGINE_GRID) mx = b > mx ? b : mx;
    else cur += b;
  }
  *bytes_out = engine == DTR_ENGINE_GRID ? cur + mx : cur;
  return DTR_OK;
}

static int grid_blocks(int *blocks) {
  int dev, sms, per_sm = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grid_engine, GRID_THREADS, 0));
  if (per_sm < 1) return DTR_E_CUDA;
  *blocks = sms * (per_sm > 2 ? 2 : per_sm);
  if (*blocks > 4096) *blocks = 4096;
  return DTR_OK;
}

int dtr_replay_batch(const uint32_t *d_words, const dtr_cell *d_cells, const uint32_t *d_dims, uint32_t n_cells,
                     uint32_t engine, void *d_ws, uint64_t ws_bytes, dtr_result *d_rows, dtr_evict_rec *d_trace,
                     void *stream) {
  if (!n_cells) return DTR_OK;
  if (!d_words || !d_cells || !d_dims || !d_ws || !d_rows) return DTR_E_INVAL;
  if (engine != DTR_ENGINE_CTA && engine != DTR_ENGINE_GRID) return DTR_E_INVAL;
  if (ws_bytes < ws_header_bytes(n_cells)) return DTR_E_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)d_ws;
  plan_kernel<<<1, 32, 0, st>>>(d_dims, n_cells, engine, ws_bytes, (u64 *)ws, (u32 *)(ws + (u64)n_cells * 8));
  CK(cudaGetLastError());
  if (engine == DTR_ENGINE_CTA) {
    cta_engine<<<n_cells, CTA_THREADS, 0, st>>>(d_words, d_cells, n_cells, ws, d_rows, d_trace);
    CK(cudaGetLastError());
  } else {
    int blocks;
    int rc = grid_blocks(&blocks);
    if (rc) return rc;
    for (u32 i = 0; i < n_cells; i++) {
      u32 ci = i;
      void *args[] = {(void *)&d_words, (void *)&d_cells, (void *)&n_cells, (void *)&ci, (void *)&ws,
                      (void *)&d_rows, (void *)&d_trace};
      CK(cudaLaunchCooperativeKernel((void *)grid_engine, dim3(blocks), dim3(GRID_THREADS), args, 0, st));
    }
  }
  return DTR_OK;
}

int dtr_replay_batch_host(const uint32_t *h_words, uint64_t n_words, const dtr_cell *h_cells, uint32_t n_cells,
                          uint32_t engine, dtr_result *h_rows, dtr_evict_rec *h_trace, uint64_t trace_total,
                          void *stream) {
  if (!n_cells) return DTR_OK;
  if (!h_words || !h_cells || !h_rows) return DTR_E_INVAL;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<u32> dims(3 * (size_t)n_cells);
  u32 max_n = 0;
  for (u32 i = 0; i < n_cells; i++) {
    u64 o = h_cells[i].log_offset;
    if (o + DTR_LOG_HEADER_WORDS > n_words || h_words[o] != DTR_LOG_MAGIC) return DTR_E_INVAL;
    dims[3 * i] = h_words[o + 2];
    dims[3 * i + 1] = h_words[o + 3];
    dims[3 * i + 2] = h_cells[i].heuristic;
    max_n = std::max(max_n, h_words[o + 2]);
  }
  if (engine == 0) engine = max_n > 65536 ? DTR_ENGINE_GRID : DTR_ENGINE_CTA;
  uint64_t ws_bytes = 0;
  int rc = dtr_batch_workspace_bytes(dims.data(), n_cells, engine, &ws_bytes);
  if (rc) return rc;
  u32 *d_words = nullptr, *d_dims = nullptr;
  dtr_cell *d_cells = nullptr;
  dtr_result *d_rows = nullptr;
  dtr_evict_rec *d_trace = nullptr;
  void *d_ws = nullptr;
  CK(cudaMallocAsync((void **)&d_words, n_words * 4, st));
  CK(cudaMallocAsync((void **)&d_dims, dims.size() * 4, st));
  CK(cudaMallocAsync((void **)&d_cells, (size_t)n_cells * sizeof(dtr_cell), st));
  CK(cudaMallocAsync((void **)&d_rows, (size_t)n_cells * sizeof(dtr_result), st));
  if (h_trace && trace_total) CK(cudaMallocAsync((void **)&d_trace, trace_total * sizeof(dtr_evict_rec), st));
  CK(cudaMallocAsync(&d_ws, ws_bytes, st));
  CK(cudaMemcpyAsync(d_words, h_words, n_words * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_dims, dims.data(), dims.size() * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_cells, h_cells, (size_t)n_cells * sizeof(dtr_cell), cudaMemcpyHostToDevice, st));
  rc = dtr_replay_batch(d_words, d_cells, d_dims, n_cells, engine, d_ws, ws_bytes, d_rows, d_trace, st);
  if (rc == DTR_OK) {
    CK(cudaMemcpyAsync(h_rows, d_rows, (size_t)n_cells * sizeof(dtr_result), cudaMemcpyDeviceToHost, st));
    if (d_trace) CK(cudaMemcpyAsync(h_trace, d_trace, trace_total * sizeof(dtr_evict_rec), cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(d_words, st);
  cudaFreeAsync(d_dims, st);
  cudaFreeAsync(d_cells, st);
  cudaFreeAsync(d_rows, st);
  if (d_trace) cudaFreeAsync(d_trace, st);
  cudaFreeAsync(d_ws, st);
  CK(cudaStreamSynchronize(st));
  return rc;
}

// ---------------------------------------------------------------------------
// per-call runtime
// ---------------------------------------------------------------------------
struct dtr_runtime {
  dtr_config cfg;
  cudaStream_t st;
  u32 *d_mem, *d_cost, *d_par_off, *d_par;
  void *d_ws;
  dtr_evict_rec *d_trace;
  u64 *d_num, *d_den;
  u32 *d_ids;
  u64 score_cap;
  Graph g;
  Work w;
  std::vector<u32> h_par_off;
  Scalars hs;   // mirror of the device scalars after the last call
};

static int rt_sync_scalars(dtr_runtime *rt) {
  CK(cudaMemcpyAsync(&rt->hs, rt->w.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, rt->st));
  CK(cudaStreamSynchronize(rt->st));
  return DTR_OK;
}

static int rt_launch(dtr_runtime *rt, u32 init, u32 op_word) {
  PercallArgs a;
  a.g = rt->g; a.w = rt->w; a.trace = rt->d_trace; a.onum = rt->d_num; a.oden = rt->d_den; a.oid = rt->d_ids;
  a.init = init;
  if (!init) {
    CK(cudaMemcpyAsync((char *)rt->w.sc + offsetof(Scalars, pending_op), &op_word, 4, cudaMemcpyHostToDevice,
                       rt->st));
  }
  percall_engine<<<1, CTA_THREADS, 0, rt->st>>>(a);
  CK(cudaGetLastError());
  return rt_sync_scalars(rt);
}

int dtr_create(const dtr_config *cfg, dtr_runtime **out) {
  if (!cfg || !out || cfg->cap_tensors == 0 || cfg->heuristic > H_RANDOM) return DTR_E_INVAL;
  if (cfg->cap_tensors >= (1u << 29) || cfg->cap_tensors > COMP_MASK) return DTR_E_INVAL;
  dtr_runtime *rt = new dtr_runtime();
  rt->cfg = *cfg;
  rt->st = (cudaStream_t)cfg->stream;
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) { delete rt; return cuda_fail(e); }
  u32 n = cfg->cap_tensors, E = cfg->cap_edges;
  u64 ws = carve(rt->w, 0, n, E, cfg->heuristic, 1, CTA_THREADS / 32);
  rt->score_cap = (u64)n + 1;
#define AL(p, bytes) do { e = cudaMalloc((void **)&(p), (bytes)); if (e != cudaSuccess) { dtr_destroy(rt); return cuda_fail(e); } } while (0)
  AL(rt->d_mem, 4 * ((u64)n + 1));
  AL(rt->d_cost, 4 * ((u64)n + 1));
  AL(rt->d_par_off, 4 * ((u64)n + 2));
  AL(rt->d_par, 4 * ((u64)E + 1));
  AL(rt->d_ws, ws);
  AL(rt->d_num, 8 * rt->score_cap);
  AL(rt->d_den, 8 * rt->score_cap);
  AL(rt->d_ids, 4 * rt->score_cap);
  if (cfg->trace_cap) AL(rt->d_trace, cfg->trace_cap * sizeof(dtr_evict_rec));
#undef AL
  carve(rt->w, (uintptr_t)rt->d_ws, n, E, cfg->heuristic, 1, CTA_THREADS / 32);
  memset(&rt->g, 0, sizeof(Graph));
  rt->g.n = n; rt->g.E = E; rt->g.nops = 1;
  rt->g.mem = rt->d_mem; rt->g.cost = rt->d_cost; rt->g.par_off = rt->d_par_off; rt->g.par = rt->d_par;
  rt->g.ops = nullptr;
  rt->g.linked = 1;
  rt->h_par_off.assign(1, 0);
  u32 zero = 0;
  e = cudaMemcpyAsync(rt->d_par_off, &zero, 4, cudaMemcpyHostToDevice, rt->st);
  if (e != cudaSuccess) { dtr_destroy(rt); return cuda_fail(e); }
  // scalars
  Scalars s;
  memset(&s, 0, sizeof s);
  s.B = cfg->budget; s.seed = cfg->seed; s.max_decisions = cfg->max_decisions; s.trace_cap = cfg->trace_cap;
  s.heuristic = cfg->heuristic; s.thrash_kill = cfg->thrash_kill; s.comp_free_top = n + 1;
  s.uf_cap = 2 * n + 64; s.trace_hash = 14695981039346656037ull;
  e = cudaMemcpyAsync(rt->w.sc, &s, sizeof s, cudaMemcpyHostToDevice, rt->st);
  if (e != cudaSuccess) { dtr_destroy(rt); return cuda_fail(e); }
  int rc = rt_launch(rt, 1, 0);
  if (rc) { dtr_destroy(rt); return rc; }
  *out = rt;
  return DTR_OK;
}

int dtr_destroy(dtr_runtime *rt) {
  if (!rt) return DTR_OK;
  cudaFree(rt->d_mem); cudaFree(rt->d_cost); cudaFree(rt->d_par_off); cudaFree(rt->d_par);
  cudaFree(rt->d_ws); cudaFree(rt->d_num); cudaFree(rt->d_den); cudaFree(rt->d_ids);
  if (rt->d_trace) cudaFree(rt->d_trace);
  delete rt;
  return DTR_OK;
}

static bool sticky(const dtr_runtime *rt) { return rt->hs.status != ST_OK && rt->hs.status != ST_PRECOND; }

static int rt_op(dtr_runtime *rt, u32 op, u32 id) {
  if (!rt) return DTR_E_INVAL;
  if (sticky(rt)) return DTR_E_STATE;
  if (id >= (1u << 29)) return DTR_E_PRECOND;   // unknown tensor (device checks id < n_alloc)
  int rc = rt_launch(rt, 0, (op << 29) | id);
  if (rc) return rc;
  return (int)rt->hs.last_rc;
}

int dtr_compute(dtr_runtime *rt, uint32_t mem, uint32_t compute, const uint32_t *parents, uint32_t n_parents,
                uint32_t *out_id) {
  if (!rt || mem == 0 || compute == 0 || compute > 0x7FFFFFFFu || (n_parents && !parents)) return DTR_E_INVAL;
  if (sticky(rt)) return DTR_E_STATE;
  u32 t = rt->hs.n_alloc;
  std::vector<u32> ps;
  ps.reserve(n_parents);
  for (u32 j = 0; j < n_parents; j++) {
    if (parents[j] >= t) return DTR_E_INVAL;
    if (std::find(ps.begin(), ps.end(), parents[j]) == ps.end()) ps.push_back(parents[j]);
  }
  if (t >= rt->cfg.cap_tensors) return DTR_E_CAPACITY;
  u32 base = rt->h_par_off[t];
  if ((u64)base + ps.size() > rt->cfg.cap_edges) return DTR_E_CAPACITY;
  u32 end = base + (u32)ps.size();
  CK(cudaMemcpyAsync(rt->d_mem + t, &mem, 4, cudaMemcpyHostToDevice, rt->st));
  CK(cudaMemcpyAsync(rt->d_cost + t, &compute, 4, cudaMemcpyHostToDevice, rt->st));
  CK(cudaMemcpyAsync(rt->d_par_off + t + 1, &end, 4, cudaMemcpyHostToDevice, rt->st));
  if (!ps.empty()) CK(cudaMemcpyAsync(rt->d_par + base, ps.data(), 4 * ps.size(), cudaMemcpyHostToDevice, rt->st));
  int rc = rt_launch(rt, 0, (OP_MAKE << 29) | t);
  if (rc) return rc;
  if (rt->hs.n_alloc == t + 1) {
    rt->h_par_off.resize(t + 2);
    rt->h_par_off[t + 1] = end;
    if (out_id) *out_id = t;
  }
  return (int)rt->hs.last_rc;
}

int dtr_get(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_GET, id); }
int dtr_release(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_RELEASE, id); }
int dtr_rematerialize(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_REMAT, id); }
int dtr_ensure(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_ENSURE, id); }
int dtr_debug_evict(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_DEBUG_EVICT, id); }

int dtr_debug_set_budget(dtr_runtime *rt, uint64_t budget) {
  if (!rt) return DTR_E_INVAL;
  CK(cudaMemcpyAsync((char *)rt->w.sc + offsetof(Scalars, B), &budget, 8, cudaMemcpyHostToDevice, rt->st));
  return rt_sync_scalars(rt);
}

int dtr_debug_scores(dtr_runtime *rt, uint64_t *num, uint64_t *den, uint32_t *ids, uint64_t cap, uint64_t *n_out) {
  if (!rt || !n_out) return DTR_E_INVAL;
  int rc = rt_launch(rt, 0, (u32)OP_SCORES << 29);
  if (rc) return rc;
  u64 k = rt->hs.n_scores;
  *n_out = k;
  u64 m = std::min<u64>(k, (u64)cap);
  if (m) {
    CK(cudaMemcpyAsync(num, rt->d_num, 8 * m, cudaMemcpyDeviceToHost, rt->st));
    CK(cudaMemcpyAsync(den, rt->d_den, 8 * m, cudaMemcpyDeviceToHost, rt->st));
    CK(cudaMemcpyAsync(ids, rt->d_ids, 4 * m, cudaMemcpyDeviceToHost, rt->st));
    CK(cudaStreamSynchronize(rt->st));
  }
  return DTR_OK;
}

int dtr_stats(dtr_runtime *rt, dtr_result *out) {
  if (!rt || !out) return DTR_E_INVAL;
  int rc = rt_sync_scalars(rt);
  if (rc) return rc;
  const Scalars &s = rt->hs;
  memset(out, 0, sizeof *out);
  out->status = s.status; out->records_done = s.records_done; out->n_trace = (u32)s.trace_n;
  out->clock = s.clock; out->base = s.base_so_far; out->decisions = s.decisions; out->remats = s.remats;
  out->computations = s.computations; out->peak_M = s.peak_M; out->trace_hash = s.trace_hash;
  return DTR_OK;
}

int dtr_trace(dtr_runtime *rt, dtr_evict_rec *buf, uint64_t cap, uint64_t *n_out) {
  if (!rt || !n_out) return DTR_E_INVAL;
  u64 k = rt->hs.trace_n;
  *n_out = k;
  u64 m = std::min<u64>(k, (u64)cap);
  if (m && rt->d_trace) {
    CK(cudaMemcpyAsync(buf, rt->d_trace, m * sizeof(dtr_evict_rec), cudaMemcpyDeviceToHost, rt->st));
    CK(cudaStreamSynchronize(rt->st));
  }
  return DTR_OK;
}

}  // extern "C"
