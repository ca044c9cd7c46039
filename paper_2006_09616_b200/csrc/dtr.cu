// dtr.cu -- kernels and C ABI of libdtr.so (see include/dtr.h).
//
// Engines:
//   K6 cta_engine   one CTA per simulation: leader thread 0 runs the control
//                   (leader.cuh), the CTA scores the pool and reduces the argmin
//                   (team.cuh).  The whole simulation -- log tables and state --
//                   lives in shared memory when it fits (SM = true).
//   K7 grid_engine  one cooperative persistent grid per simulation: leader is
//                   block 0 / thread 0; every SM scores a slice of the pool,
//                   per-block partial argmins are reduced by block 0.
//   percall_engine  the per-call API: one CTA applies one record to persistent
//                   device state (children kept as linked lists because future
//                   children are unknown).
// K1/K2 (component maintenance + aggregation) run inside the leader; K3+K4
// (score + argmin) and K5 (MSPS closure) are team.cuh.
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>
#include <algorithm>

#include "engine.cuh"
#include "leader.cuh"
#include "team.cuh"
#include "../../include/dtr.h"

namespace cg = cooperative_groups;
using namespace dtr;

#define CTA_THREADS 256
#define GRID_THREADS 512
#define GRID_MSPS_WARPS 1024
#define WS_HEADER 164352ull  /* 512 + 4096 * (sizeof(Cand) + 16), multiple of 256 */
#define WS_BSTATS 98816      /* per-block {bytes, evals} for dtr_pool_argmin */
#define WS_SCALARS 128       /* grid engine: final Scalars of the last cell */
#define WS_PARTIALS 512
#define WS_SLOWN 124         /* whole-GPU team: slow-queue length (u32) */
#define CTA_SMEM_MAX (225u * 1024u)  /* + ~1 KB static CtaShared <= 227 KB per block */

// ---------------------------------------------------------------------------
// Initialisation (team-parallel): static records and parents from the log,
// zeroed dynamic state, children CSR (count, scan, fill, sort).
// ---------------------------------------------------------------------------
struct ScanSmem {
  u32 warp_tot[32];
  u32 carry;
};

// exclusive scan of the child counts crec[p].y into offsets crec[p].x; run by ONE block.
template <bool SM>
__device__ void block_scan_children(const Sim<SM> &g, u32 n, ScanSmem &sm) {
  const u32 T = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = (T + 31) >> 5;
  const u32 chunk = (n + T - 1) / T;
  const u32 lo = tid * chunk < n ? tid * chunk : n, hi = lo + chunk < n ? lo + chunk : n;
  u32 local = 0;
  for (u32 i = lo; i < hi; i++) local += g.crec(i).y;
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
    if (lane < nw) sm.warp_tot[lane] = y - x;
  }
  __syncthreads();
  u32 run = sm.warp_tot[wid] + v - local;
  for (u32 i = lo; i < hi; i++) { uint2 c = g.crec(i); g.crec(i).x = run; run += c.y; }
  __syncthreads();
}

template <bool SM, class Sync>
__device__ void init_sim(const Sim<SM> &g, const u32 *logw, u32 rank, u32 size, bool scan_block, ScanSmem &ssm,
                         Sync sync) {
  const u32 n = g.L.n, E = g.L.E, heur = g.L.heur;
  const u32 *lmem = logw + 16, *lcost = lmem + n, *loff = lcost + n, *lpar = loff + n + 1;
  for (u32 t = rank; t < n; t += size) {
    const u32 b = loff[t], e = loff[t + 1];
    g.srec(t) = make_uint4(lmem[t], lcost[t], 0, 0);     // la = -inf, nev = 0
    g.arec(t) = make_uint4(b, e - b, 0, 0);               // children counted below
    g.state(t) = 0; g.rho(t) = 0; g.ell(t) = 0;
    g.pool_pos(t) = NONE;
    g.m.w(g.L.fr + t) = 0;                      // fill cursor (the stack is unused until the leader starts)
    if (heur == H_DTR) g.m.w(g.L.stamp + t) = 0;
    if (uses_uf(heur)) g.m.w(g.L.node_of + t) = NONE;
  }
  for (u32 j = rank; j < E; j += size) g.par(j) = lpar[j];
  for (u32 w = rank; w < g.L.pool_words; w += size) g.pool_word(w) = 0;
  if (uses_closure(heur)) {
    const u32 words = g.L.msps_words * g.L.msps_warps;
    for (u32 i = rank; i < words; i += size) g.m.w(g.L.msps_bm + i) = 0;
  }
  sync();
  for (u32 c = rank; c < n; c += size) {
    const u32 b = loff[c], e = loff[c + 1];
    for (u32 j = b; j < e; j++) atomicAdd(&g.crec(lpar[j]).y, 1u);
  }
  sync();
  if (scan_block) block_scan_children(g, n, ssm);
  sync();
  for (u32 c = rank; c < n; c += size) {
    const u32 b = loff[c], e = loff[c + 1];
    for (u32 j = b; j < e; j++) {
      const u32 p = lpar[j];
      const u32 k = atomicAdd(&g.m.w(g.L.fr + p), 1u);
      g.m.w(g.L.ch + g.crec(p).x + k) = c;
    }
  }
  sync();
  // deterministic child order (ascending id): results never depend on it, but
  // union-find tree shapes (and so the byte accounting) do
  for (u32 p = rank; p < n; p += size) {
    const uint2 cr = g.crec(p);
    const u32 b = g.L.ch + cr.x, e = b + cr.y;
    for (u32 i = b + 1; i < e; i++) {
      u32 x = g.m.w(i), j = i;
      while (j > b && g.m.w(j - 1) > x) { g.m.w(j) = g.m.w(j - 1); j--; }
      g.m.w(j) = x;
    }
  }
  sync();
}

__device__ void init_scalars(Scalars &s, const dtr_cell &cell) {
  memset(&s, 0, sizeof(Scalars));
  s.B = cell.budget;
  s.seed = cell.seed;
  s.max_decisions = cell.max_decisions;
  s.trace_cap = cell.trace_cap;
  s.trace_off = cell.trace_offset;
  s.heuristic = cell.heuristic;
  s.thrash_kill = cell.thrash_kill;
  s.cell_id = cell.cell_id;
  s.dealloc = cell.dealloc;
  s.trace_hash = 14695981039346656037ull;
  norm_scalars(s);
}

__device__ void write_row(dtr_result &r, const Scalars &s, u64 bytes, u64 evals) {
  dtr_result x;
  x.cell_id = s.cell_id;
  x.status = s.status;
  x.records_done = s.records_done;
  x.n_trace = (u32)s.trace_n;
  x.clock = s.clock;
  x.base = s.base_so_far;
  x.decisions = s.decisions;
  x.remats = s.remats;
  x.computations = s.computations;
  x.peak_M = s.peak_M;
  x.trace_hash = s.trace_hash;
  x.cand_evals = evals;
  x.score_bytes = bytes;
  r = x;
}

__device__ __forceinline__ void publish(Cmd &c, u32 kind, const Scalars &s) {
  c.kind = kind; c.pool_size = s.pool_size; c.clock = s.clock; c.decisions = s.decisions;
  c.seed = s.seed; c.heur = s.heuristic; c.n_ids = s.n_alloc;
}

template <bool SM, bool BM>
__device__ __forceinline__ void leader_init(Leader<SM, BM> &L, const Sim<SM> &g, const u32 *logw, const dtr_cell &cell,
                                            dtr_evict_rec *trace) {
  L.g = g;
  init_scalars(L.s, cell);
  const u32 n = g.L.n, E = g.L.E;
  L.ops = logw + 16 + 3 * n + 1 + E;
  L.trace = (trace && cell.trace_cap) ? trace + cell.trace_offset : nullptr;
  L.op_idx = 0; L.op_end = logw[4];
  L.phase = PH_OP; L.post = 0; L.root = 0; L.percall = 0; L.free_size = 0;
}

// ---------------------------------------------------------------------------
// Workspace: header ([0,64) grid command, [64,128) grid stats, [256, ...) grid
// per-block partials), then one region per cell (CTA engine, in cell order) or
// one region reused by every cell (grid engine).
// ---------------------------------------------------------------------------
__host__ __device__ inline u64 cell_bytes(u32 n, u32 E, u32 heur, u32 engine) {
  Lay L;
  make_layout(L, n, E, heur, 0, engine == DTR_ENGINE_GRID ? GRID_MSPS_WARPS : CTA_THREADS / 32,
              engine == DTR_ENGINE_GRID);
  return ((u64)L.words * 4 + 255) & ~255ull;
}

__host__ __device__ inline u64 cta_smem_need(u32 n, u32 E, u32 heur) {
  Lay L;
  make_layout(L, n, E, heur, 0, CTA_THREADS / 32);
  return (u64)L.words * 4;
}

// ---------------------------------------------------------------------------
// K6: one CTA per simulation.
// ---------------------------------------------------------------------------
struct __align__(16) CtaShared {
  Cmd cmd;
  RedSmem red;
  ScanSmem scan;
  u32 msps_tail[CTA_THREADS / 32];
};

struct CtaSync {
  __device__ void operator()() const { __syncthreads(); }
};

// Hybrid team: warp 0 holds the leader (lane 0); a decision over a pool of at
// most WARP_TEAM_MAX candidates is scored by warp 0 alone (no CTA barrier, one
// warp-shuffle reduction); larger pools wake the whole CTA through the barrier.
#define WARP_TEAM_MAX 192

__device__ __forceinline__ Cmd shfl_cmd(const Cmd &c) {
  Cmd r;
  r.kind = __shfl_sync(0xffffffffu, c.kind, 0);
  r.pool_size = __shfl_sync(0xffffffffu, c.pool_size, 0);
  r.clock = __shfl_sync(0xffffffffu, c.clock, 0);
  r.decisions = __shfl_sync(0xffffffffu, c.decisions, 0);
  r.seed = __shfl_sync(0xffffffffu, c.seed, 0);
  r.heur = __shfl_sync(0xffffffffu, c.heur, 0);
  r.n_ids = __shfl_sync(0xffffffffu, c.n_ids, 0);
  return r;
}

// CL = false: compiled without the K5 closure pass (batches whose cells use
// no closure heuristic): the leader's hot path then shares its kernel with
// less cold code (measured 3.5 % faster on the bench's critical cells).
template <bool SM, bool CL>
__device__ void run_cta(const u32 *logw, const dtr_cell &cell, u32 *gbase, dtr_result *row, dtr_evict_rec *trace,
                        CtaShared &sh) {
  const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Sim<SM> g;
  g.m.gbase = gbase;
  make_layout(g.L, logw[2], logw[3], cell.heuristic, 0, CTA_THREADS / 32);
  PROF_T(ti0);
  init_sim(g, logw, tid, blockDim.x, true, sh.scan, CtaSync());
  PROF_T(ti1);
  if (tid == 0) PROF_ADD(6, ti1 - ti0);
  u64 bytes = 0, evals = 0;
  if (warp == 0) {
    Leader<SM, false> L;
    if (lane == 0) leader_init(L, g, logw, cell, trace);
    Cand res = cand_none();
    bool have = false;
    for (;;) {
      Cmd c;
      if (lane == 0) {
        PROF_T(t0);
        const u32 kind = L.resume(have, res);
        have = false;
        publish(c, kind, L.s);
        PROF_T(t1);
        PROF_ADD(0, t1 - t0);
      }
      c = shfl_cmd(c);
      if (c.kind == CMD_ARGMIN && c.pool_size <= WARP_TEAM_MAX && g.L.pool_key) {   // size / LRU: 64-bit keys
        PROF_T(t2);
        const u64 k = warp_min64(team_intkey_min(g, c, lane, 32, bytes, evals));
        PROF_T(t3);
        if (lane == 0) { res = intkey_cand(g, c, k); have = true; PROF_ADD(1, t3 - t2); PROF_ADD(3, 1); }
        continue;
      }
      if (c.kind == CMD_ARGMIN && c.pool_size <= WARP_TEAM_MAX) {
        PROF_T(t2);
        u32 bk;
        Cand best = team_score<SM, false, false, CL>(g, c, lane, 32, 0, 1, sh.msps_tail, bytes, evals, bk);
        PROF_T(t3);
        best = warp_argmin_fast(best, bk, int_key_heur(c.heur));
        PROF_T(t4);
        if (lane == 0) { res = best; have = true; PROF_ADD(1, t3 - t2); PROF_ADD(2, t4 - t3); PROF_ADD(3, 1); }
        continue;
      }
      PROF_T(t5);
      if (lane == 0) sh.cmd = c;
      __syncthreads();
      if (c.kind != CMD_ARGMIN) break;
      u32 bk;
      Cand best = team_score<SM, false, false, CL>(g, c, tid, blockDim.x, warp, blockDim.x >> 5, sh.msps_tail, bytes, evals, bk);
      best = block_argmin(best, bk, sh.red, int_key_heur(c.heur));
      PROF_T(t6);
      if (lane == 0) { res = best; have = true; PROF_ADD(4, t6 - t5); PROF_ADD(5, 1); }
    }
    if (lane == 0) write_row(*row, L.s, 0, 0);
  } else {
    for (;;) {
      __syncthreads();
      const Cmd c = sh.cmd;
      if (c.kind != CMD_ARGMIN) break;
      u32 bk;
      Cand best = team_score<SM, false, false, CL>(g, c, tid, blockDim.x, warp, blockDim.x >> 5, sh.msps_tail, bytes, evals, bk);
      block_argmin(best, bk, sh.red, int_key_heur(c.heur));
    }
  }
  block_sum2(bytes, evals, sh.red);
  if (tid == 0) { row->score_bytes = bytes; row->cand_evals = evals; }
}

template <bool CL>
__global__ void __launch_bounds__(CTA_THREADS, 1) cta_engine(const u32 *words, const dtr_cell *cells, u32 c0, u32 n_run,
                                                          char *ws, u64 ws_bytes, dtr_result *rows,
                                                          dtr_evict_rec *trace, u32 smem_bytes) {
  __shared__ CtaShared sh;
  const u32 tid = threadIdx.x;
  if (blockIdx.x >= n_run) return;
  const u32 ci = c0 + blockIdx.x;
  // this cell's global region: header + sizes of all cells before it
  u64 part = 0, junk = 0;
  for (u32 j = tid; j < ci; j += blockDim.x) {
    const dtr_cell c = cells[j];
    const u32 *h = words + c.log_offset;
    part += cell_bytes(h[2], h[3], c.heuristic, DTR_ENGINE_CTA);
  }
  block_sum2(part, junk, sh.red);
  if (tid == 0) sh.red.warp[0].num = part;
  __syncthreads();
  part = sh.red.warp[0].num;
  const dtr_cell cell = cells[ci];
  const u32 *logw = words + cell.log_offset;
  const u64 off = WS_HEADER + part;
  if (off + cell_bytes(logw[2], logw[3], cell.heuristic, DTR_ENGINE_CTA) > ws_bytes) {
    if (tid == 0) {
      dtr_result r; memset(&r, 0, sizeof r);
      r.cell_id = cell.cell_id; r.status = ST_CAPACITY;
      rows[ci] = r;
    }
    return;
  }
  if (cta_smem_need(logw[2], logw[3], cell.heuristic) <= smem_bytes)
    run_cta<true, CL>(logw, cell, nullptr, &rows[ci], trace, sh);
  else
    run_cta<false, CL>(logw, cell, (u32 *)(ws + off), &rows[ci], trace, sh);
}

// ---------------------------------------------------------------------------
// K7: the whole GPU on one simulation (cooperative launch).
// ---------------------------------------------------------------------------
struct __align__(16) GridShared {
  Cmd cmd;
  RedSmem red;
  ScanSmem scan;
  u32 msps_tail[GRID_THREADS / 32];
};

struct GridSync {
  __device__ void operator()() const { cg::this_grid().sync(); }
};

__global__ void __launch_bounds__(GRID_THREADS, 1) grid_engine(const u32 *words, const dtr_cell *cells, u32 ci,
                                                            char *ws, u64 ws_bytes, dtr_result *rows,
                                                            dtr_evict_rec *trace) {
  __shared__ GridShared sh;
  cg::grid_group grid = cg::this_grid();
  const u32 tid = threadIdx.x;
  Cmd *gcmd = (Cmd *)ws;
  u64 *gstats = (u64 *)(ws + 64);   // [bytes, evals]
  Cand *partials = (Cand *)(ws + WS_PARTIALS);
  const dtr_cell cell = cells[ci];
  const u32 *logw = words + cell.log_offset;
  if (WS_HEADER + cell_bytes(logw[2], logw[3], cell.heuristic, DTR_ENGINE_GRID) > ws_bytes) {
    if (blockIdx.x == 0 && tid == 0) {
      dtr_result r; memset(&r, 0, sizeof r);
      r.cell_id = cell.cell_id; r.status = ST_CAPACITY;
      rows[ci] = r;
    }
    return;
  }
  Sim<false> g;
  g.m.gbase = (u32 *)(ws + WS_HEADER);
  make_layout(g.L, logw[2], logw[3], cell.heuristic, 0, GRID_MSPS_WARPS, 1);
  const u32 rank = blockIdx.x * blockDim.x + tid, size = gridDim.x * blockDim.x;
  const u32 wrank = rank >> 5, wsize = size >> 5;
  u32 *slown = (u32 *)(ws + WS_SLOWN);
  if (rank == 0) { gstats[0] = 0; gstats[1] = 0; *slown = 0; }
  init_sim(g, logw, rank, size, blockIdx.x == 0, sh.scan, GridSync());
  Leader<false, true> L;
  if (rank == 0) leader_init(L, g, logw, cell, trace);
  Cand res = cand_none();
  bool have = false;
  u64 bytes = 0, evals = 0;
  PROF_T(tg0);
  for (;;) {
    if (rank == 0) {
      PROF_T(a0);
      const u32 kind = L.resume(have, res);
      have = false;
      Cmd c;
      publish(c, kind, L.s);
      *gcmd = c;
      *slown = 0;                   // every warp has finished reading it (grid barrier since)
      PROF_T(a1);
      PROF_ADD(0, a1 - a0);
    }
    PROF_T(b0);
    grid.sync();
    PROF_T(b1);
    if (rank == 0) PROF_ADD(1, b1 - b0);
    if (tid == 0) {
      Cmd c;
      c.kind = __ldcg(&gcmd->kind); c.pool_size = __ldcg(&gcmd->pool_size); c.clock = __ldcg(&gcmd->clock);
      c.decisions = __ldcg(&gcmd->decisions); c.seed = __ldcg(&gcmd->seed); c.heur = __ldcg(&gcmd->heur);
      c.n_ids = __ldcg(&gcmd->n_ids);
      sh.cmd = c;
    }
    __syncthreads();
    if (sh.cmd.kind != CMD_ARGMIN) break;
    u32 bk;
    PROF_T(c0);
    Cand best = team_score<false, true, true>(g, sh.cmd, rank, size, wrank, wsize, sh.msps_tail, bytes, evals, bk,
                                              slown);
    PROF_T(c1);
    const bool ik = int_key_heur(sh.cmd.heur);
    best = block_argmin(best, bk, sh.red, ik);
    if (tid == 0) partials[blockIdx.x] = best;
    PROF_T(c2);
    grid.sync();
    PROF_T(c3);
    if (rank == 0) { PROF_ADD(2, c1 - c0); PROF_ADD(3, c2 - c1); PROF_ADD(4, c3 - c2); PROF_ADD(5, 1); }
    if (blockIdx.x == 0) {          // block 0 reduces the per-block partials (one load per thread)
      Cand c = cand_none();
      u32 ck = KEY_NONE;
      for (u32 b = tid; b < gridDim.x; b += blockDim.x) {
        Cand d;
        d.num = __ldcg(&partials[b].num); d.den = __ldcg(&partials[b].den); d.id = __ldcg(&partials[b].id);
        cand_take(c, ck, d, ik);
      }
      c = block_argmin(c, ck, sh.red, ik);
      if (tid == 0) { res = c; have = true; }
    }
  }
  PROF_T(tg1);
  if (rank == 0) PROF_ADD(6, tg1 - tg0);
  block_sum2(bytes, evals, sh.red);
  if (tid == 0) { atomicAdd(&gstats[0], bytes); atomicAdd(&gstats[1], evals); }
  grid.sync();
  if (rank == 0) {
    write_row(rows[ci], L.s, __ldcg(&gstats[0]), __ldcg(&gstats[1]));
    *(Scalars *)(ws + WS_SCALARS) = L.s;   // kept for dtr_pool_argmin
  }
}

// ---------------------------------------------------------------------------
// K3+K4 alone: score the current pool of the simulation left in a grid-engine
// workspace and reduce its argmin (last-block reduction, no cooperative sync).
// Used to time the score pass in isolation (bench roofline_large_pool).
// ---------------------------------------------------------------------------
#define PA_THREADS 256
struct __align__(16) PaShared {
  RedSmem red;
  u32 msps_tail[PA_THREADS / 32];
};

__global__ void __launch_bounds__(PA_THREADS, 4) pool_argmin_kernel(const u32 *logw, u32 heur, char *ws,
                                                                    u64 *out /* num, den, id, bytes, evals */) {
  __shared__ PaShared sh;
  const u32 tid = threadIdx.x;
  Cand *partials = (Cand *)(ws + WS_PARTIALS);
  u32 *slown = (u32 *)(ws + WS_SLOWN);
  Sim<false> g;
  g.m.gbase = (u32 *)(ws + WS_HEADER);
  make_layout(g.L, logw[2], logw[3], heur, 0, GRID_MSPS_WARPS, 1);
  const Scalars *sc = (const Scalars *)(ws + WS_SCALARS);
  Cmd cmd;
  cmd.kind = CMD_ARGMIN; cmd.pool_size = sc->pool_size; cmd.clock = sc->clock; cmd.decisions = sc->decisions;
  cmd.seed = sc->seed; cmd.heur = heur; cmd.n_ids = sc->n_alloc;
  const u32 rank = blockIdx.x * blockDim.x + tid, size = gridDim.x * blockDim.x;
  u64 bytes = 0, evals = 0;
  u32 bk;
  Cand best = team_score<false, true, true>(g, cmd, rank, size, rank >> 5, size >> 5, sh.msps_tail, bytes, evals, bk,
                                            slown);
  const bool ik = int_key_heur(heur);
  best = block_argmin(best, bk, sh.red, ik);
  block_sum2(bytes, evals, sh.red);
  u64 *bstats = (u64 *)(ws + WS_BSTATS);
  if (tid == 0) {
    partials[blockIdx.x] = best;
    bstats[2 * blockIdx.x] = bytes;
    bstats[2 * blockIdx.x + 1] = evals;
  }
  cg::this_grid().sync();
  if (blockIdx.x == 0) {      // block 0 reduces the partials (all loads in flight)
    Cand c = cand_none();
    u32 ck = KEY_NONE;
    u64 tb = 0, te = 0;
    for (u32 b = tid; b < gridDim.x; b += blockDim.x) {
      Cand d;
      d.num = __ldcg(&partials[b].num); d.den = __ldcg(&partials[b].den); d.id = __ldcg(&partials[b].id);
      cand_take(c, ck, d, ik);
      tb += __ldcg(&bstats[2 * b]);
      te += __ldcg(&bstats[2 * b + 1]);
    }
    c = block_argmin(c, ck, sh.red, ik);
    Cand w = c;
    block_sum2(tb, te, sh.red);
    if (tid == 0) { out[0] = w.num; out[1] = w.den; out[2] = w.id; out[3] = tb; out[4] = te; *slown = 0; }
  }
}

// ---------------------------------------------------------------------------
// Per-call engine: apply ONE record to the persistent state of a runtime
// (global memory, linked children; the host writes srec[t] and the parent ids
// of each new tensor before the MAKE launch).
// ---------------------------------------------------------------------------
struct PercallArgs {
  Lay L;
  u32 *base;
  Scalars *sc;
  dtr_evict_rec *trace;
  u64 *onum, *oden;
  u32 *oid;
  u32 init;         // first launch: initialise state
};

__global__ void __launch_bounds__(CTA_THREADS) percall_engine(PercallArgs a) {
  __shared__ CtaShared sh;
  const u32 tid = threadIdx.x;
  Sim<false> g;
  g.m.gbase = a.base;
  g.L = a.L;
  if (a.init) {
    for (u32 w = tid; w < g.L.pool_words; w += blockDim.x) g.pool_word(w) = 0;
    for (u32 t = tid; t <= g.L.n; t += blockDim.x) {
      g.srec(t) = make_uint4(0, 0, 0, 0);
      g.state(t) = 0; g.rho(t) = 0; g.ell(t) = 0;
      g.pool_pos(t) = NONE;
      g.crec(t) = make_uint2(NONE, 0);
      if (g.L.heur == H_DTR) g.m.w(g.L.stamp + t) = 0;
      if (uses_uf(g.L.heur)) g.m.w(g.L.node_of + t) = NONE;
    }
    if (uses_closure(g.L.heur)) {
      const u32 words = g.L.msps_words * g.L.msps_warps;
      for (u32 i = tid; i < words; i += blockDim.x) g.m.w(g.L.msps_bm + i) = 0;
    }
    return;
  }
  Leader<false, false> L;
  if (tid == 0) {
    L.g = g;
    L.s = *a.sc;
    L.ops = nullptr;
    L.trace = a.trace;
    L.op_idx = 0; L.op_end = 1;
    L.phase = PH_OP; L.post = 0; L.root = 0; L.percall = 1; L.free_size = 0;
    L.s.last_rc = ST_OK;
  }
  Cand res = cand_none();
  bool have = false;
  for (;;) {
    if (tid == 0) {
      const u32 kind = L.resume(have, res);
      have = false;
      publish(sh.cmd, kind, L.s);
    }
    __syncthreads();
    if (sh.cmd.kind == CMD_DONE) break;
    if (sh.cmd.kind == CMD_SCORES) {
      team_scores_out(g, sh.cmd, tid, blockDim.x, sh.msps_tail, a.onum, a.oden, a.oid);
      if (tid == 0) L.s.n_scores = sh.cmd.pool_size;
      __syncthreads();
      continue;
    }
    u64 junk = 0, junk2 = 0;
    u32 bk;
    Cand best = team_score<false, false>(g, sh.cmd, tid, blockDim.x, tid >> 5, blockDim.x >> 5, sh.msps_tail, junk, junk2,
                                         bk);
    best = block_argmin(best, bk, sh.red, int_key_heur(sh.cmd.heur));
    if (tid == 0) { res = best; have = true; }
  }
  if (tid == 0) *a.sc = L.s;
}

// ---------------------------------------------------------------------------
// K8: the Theorem 2 adversary (App. B; reading C-24), one CTA per
// run.  The graph is revealed online from the runtime's own residency: t0
// (locked resident by one ENSURE) gets B children, the B paths; afterwards
// the whole CTA scans the state words, marks the paths that hold a resident
// node, and the next node is appended to the lowest-indexed path with none.
// Each reveal is one MAKE applied by the per-call leader (linked children),
// its evictions scored by the CTA team.  State lives in shared memory when
// it fits, else in this run's workspace region.
// ---------------------------------------------------------------------------
struct AdvLay {
  u32 path_of, tail, rp, words;
};

__host__ __device__ inline bool adv_layout(Lay &L, AdvLay &A, u32 N, u32 B, u32 heur) {
  if (!make_layout(L, N, N, heur, 1, CTA_THREADS / 32)) return false;
  A.path_of = L.words;
  A.tail = A.path_of + N;
  A.rp = A.tail + B;
  A.words = A.rp + (B + 31) / 32;
  return true;
}

__host__ __device__ inline u64 adv_bytes(const dtr_adversary &r) {
  Lay L;
  AdvLay A;
  adv_layout(L, A, r.n, r.budget, r.heuristic);
  return ((u64)A.words * 4 + 255) & ~255ull;
}

struct __align__(16) AdvShared {
  Cmd cmd;
  RedSmem red;
  u32 msps_tail[CTA_THREADS / 32];
  u32 next;        // ADV_*
  u32 pick;        // the chosen path
  u32 parent;      // its last node (the new node's parent)
};
enum { ADV_DONE = 0, ADV_T0 = 1, ADV_ENSURE = 2, ADV_CHILD = 3, ADV_SCAN = 4 };

// run the leader / team protocol until the pending op is applied (all threads)
template <bool SM>
__device__ void adv_apply(Leader<SM, false> &L, const Sim<SM> &g, AdvShared &sh, u64 &bytes, u64 &evals) {
  const u32 tid = threadIdx.x;
  Cand res = cand_none();
  bool have = false;
  for (;;) {
    if (tid == 0) {
      const u32 kind = L.resume(have, res);
      have = false;
      publish(sh.cmd, kind, L.s);
    }
    __syncthreads();
    if (sh.cmd.kind != CMD_ARGMIN) break;
    u32 bk;
    Cand best = team_score<SM, false>(g, sh.cmd, tid, blockDim.x, tid >> 5, blockDim.x >> 5, sh.msps_tail, bytes,
                                      evals, bk);
    best = block_argmin(best, bk, sh.red, int_key_heur(sh.cmd.heur));
    if (tid == 0) { res = best; have = true; }
  }
  __syncthreads();
}

template <bool SM>
__device__ void run_adversary(const dtr_adversary &run, u32 *gbase, dtr_result *row, u32 *parents,
                              dtr_evict_rec *trace, AdvShared &sh) {
  const u32 tid = threadIdx.x;
  const u32 N = run.n, B = run.budget;
  Sim<SM> g;
  g.m.gbase = gbase;
  AdvLay A;
  adv_layout(g.L, A, N, B, run.heuristic);
  for (u32 w = tid; w < g.L.pool_words; w += blockDim.x) g.pool_word(w) = 0;
  for (u32 t = tid; t <= N; t += blockDim.x) {
    g.srec(t) = make_uint4(0, 0, 0, 0);
    g.state(t) = 0; g.rho(t) = 0; g.ell(t) = 0;
    g.pool_pos(t) = NONE;
    g.crec(t) = make_uint2(NONE, 0);
    if (g.L.heur == H_DTR) g.m.w(g.L.stamp + t) = 0;
    if (uses_uf(g.L.heur)) g.m.w(g.L.node_of + t) = NONE;
    if (t < N) { parents[t] = NONE; g.m.w(A.path_of + t) = NONE; }
  }
  if (uses_closure(g.L.heur))
    for (u32 i = tid; i < g.L.msps_words * g.L.msps_warps; i += blockDim.x) g.m.w(g.L.msps_bm + i) = 0;
  __syncthreads();
  Leader<SM, false> L;
  u32 edges = 0, ensured = 0;
  if (tid == 0) {
    L.g = g;
    memset(&L.s, 0, sizeof(Scalars));
    L.s.B = B; L.s.seed = run.seed; L.s.trace_cap = run.trace_cap; L.s.trace_off = run.trace_offset;
    L.s.heuristic = run.heuristic; L.s.cell_id = run.cell_id;
    L.s.trace_hash = 14695981039346656037ull;
    norm_scalars(L.s);
    L.ops = nullptr;
    L.trace = (trace && run.trace_cap) ? trace + run.trace_offset : nullptr;
    L.post = 0; L.root = 0; L.percall = 1; L.free_size = 0;
  }
  const u32 n_first = B < N - 1 ? B : N - 1;      // t0's children
  const u32 rp_words = (B + 31) / 32;
  u64 bytes = 0, evals = 0;
  for (;;) {
    if (tid == 0) {
      const u32 n = L.s.n_alloc;
      u32 nx;
      if (L.s.status != ST_OK || (n >= N && ensured)) nx = ADV_DONE;
      else if (n == 0) nx = ADV_T0;
      else if (!ensured) nx = ADV_ENSURE;
      else if (n - 1 < n_first) nx = ADV_CHILD;
      else nx = ADV_SCAN;
      sh.next = nx;
    }
    __syncthreads();
    const u32 nx = sh.next;
    if (nx == ADV_DONE) break;
    if (nx == ADV_SCAN) {                         // which paths hold a resident node?
      const u32 n = sh.cmd.n_ids;                 // n_alloc as of the last publish
      for (u32 w = tid; w < rp_words; w += blockDim.x) g.m.w(A.rp + w) = 0;
      __syncthreads();
      for (u32 t = 1 + tid; t < n; t += blockDim.x)
        if (is_material(g.state(t))) {
          const u32 j = g.m.w(A.path_of + t);
          atomicOr(&g.m.w(A.rp + (j >> 5)), 1u << (j & 31));
        }
      __syncthreads();
    }
    if (tid == 0) {
      const u32 t = L.s.n_alloc;
      u32 p = NONE, j = NONE;
      if (nx == ADV_T0) {
        g.srec(0) = make_uint4(1, 1, 0, 0);
        g.prec(0) = make_uint2(edges, 0);
      } else if (nx == ADV_CHILD || nx == ADV_SCAN) {
        if (nx == ADV_CHILD) {
          j = t - 1;
        } else {
          for (u32 w = 0; w < rp_words && j == NONE; w++) {
            u32 free_bits = ~g.m.w(A.rp + w);
            if (w == rp_words - 1 && (B & 31)) free_bits &= (1u << (B & 31)) - 1;
            if (free_bits) j = w * 32 + __ffs(free_bits) - 1;
          }
          // B paths share B - 1 units, so j exists; if not, stop
          if (j == NONE) { L.s.status = ST_STATE; }
        }
        if (j != NONE) {
          p = nx == ADV_CHILD ? 0u : g.m.w(A.tail + j);
          g.srec(t) = make_uint4(1, 1, 0, 0);
          g.prec(t) = make_uint2(edges, 1);
          g.par(edges) = p;
        }
      }
      L.s.pending_op = nx == ADV_ENSURE ? ((u32)OP_ENSURE << 29) : (((u32)OP_MAKE << 29) | t);
      L.op_idx = 0; L.op_end = (L.s.status == ST_OK) ? 1 : 0;
      L.phase = PH_OP;
      sh.pick = j;
      sh.parent = p;
    }
    __syncthreads();
    adv_apply(L, g, sh, bytes, evals);
    if (tid == 0) {
      if (nx == ADV_ENSURE) ensured = 1;
      else if (L.s.status == ST_OK && L.s.last_rc == ST_OK) {
        const u32 t = L.s.n_alloc - 1, j = sh.pick;
        if (nx != ADV_T0) {
          edges++;
          parents[t] = sh.parent;
          g.m.w(A.path_of + t) = j;
          g.m.w(A.tail + j) = t;
        }
      } else if (L.s.status == ST_OK) {
        L.s.status = L.s.last_rc;                  // a precondition failure cannot happen here
      }
    }
    __syncthreads();
  }
  block_sum2(bytes, evals, sh.red);
  if (tid == 0) write_row(*row, L.s, bytes, evals);
}

__global__ void __launch_bounds__(CTA_THREADS, 1) adversary_engine(const dtr_adversary *runs, u32 n_runs, char *ws,
                                                                u64 ws_bytes, dtr_result *rows, u32 *parents,
                                                                dtr_evict_rec *trace, u32 smem_bytes) {
  __shared__ AdvShared sh;
  const u32 tid = threadIdx.x, ri = blockIdx.x;
  if (ri >= n_runs) return;
  u64 off = 0, poff = 0;
  for (u32 j = tid; j < ri; j += blockDim.x) {
    const dtr_adversary r = runs[j];
    off += adv_bytes(r);
    poff += r.n;
  }
  block_sum2(off, poff, sh.red);
  if (tid == 0) { sh.red.warp[0].num = off; sh.red.warp[0].den = poff; }
  __syncthreads();
  off = sh.red.warp[0].num;
  poff = sh.red.warp[0].den;
  __syncthreads();
  const dtr_adversary run = runs[ri];
  Lay L;
  AdvLay A;
  if (run.n == 0 || run.budget < 3 || !valid_heuristic(run.heuristic) || !adv_layout(L, A, run.n, run.budget, run.heuristic) ||
      off + adv_bytes(run) > ws_bytes) {
    if (tid == 0) {
      dtr_result r; memset(&r, 0, sizeof r);
      r.cell_id = run.cell_id; r.status = run.n == 0 || run.budget < 3 ? ST_INVAL : ST_CAPACITY;
      rows[ri] = r;
    }
    return;
  }
  if ((u64)A.words * 4 <= smem_bytes)
    run_adversary<true>(run, nullptr, &rows[ri], parents + poff, trace, sh);
  else
    run_adversary<false>(run, (u32 *)(ws + off), &rows[ri], parents + poff, trace, sh);
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

#ifdef DTR_PROFILE
int dtr_debug_profile(unsigned long long *out, int reset) {
  CK(cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 16));
  if (reset) { unsigned long long z[16] = {0}; CK(cudaMemcpyToSymbol(g_prof, z, sizeof z)); }
  return DTR_OK;
}
#endif

int dtr_batch_workspace_bytes(const uint32_t *dims, uint32_t n_cells, uint32_t engine, uint64_t *bytes_out) {
  if (!bytes_out || (n_cells && !dims) || (engine != DTR_ENGINE_CTA && engine != DTR_ENGINE_GRID)) return DTR_E_INVAL;
  u64 cur = WS_HEADER, mx = 0;
  for (u32 i = 0; i < n_cells; i++) {
    if (!valid_heuristic(dims[3 * i + 2])) return DTR_E_INVAL;
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
  if (const char *e = getenv("DTR_GRID_BLOCKS")) {   // probes only
    int b = atoi(e);
    if (b > 0 && b < *blocks) *blocks = b;
  }
  if (*blocks > 4096) *blocks = 4096;
  return DTR_OK;
}

int dtr_replay_batch(const uint32_t *d_words, const dtr_cell *d_cells, const uint32_t *h_dims, uint32_t n_cells,
                     uint32_t engine, void *d_ws, uint64_t ws_bytes, dtr_result *d_rows, dtr_evict_rec *d_trace,
                     void *stream) {
  if (!n_cells) return DTR_OK;
  if (!d_words || !d_cells || !h_dims || !d_ws || !d_rows) return DTR_E_INVAL;
  if (engine != DTR_ENGINE_CTA && engine != DTR_ENGINE_GRID) return DTR_E_INVAL;
  uint64_t need = 0;
  int rc = dtr_batch_workspace_bytes(h_dims, n_cells, engine, &need);
  if (rc) return rc;
  if (ws_bytes < need) return DTR_E_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)d_ws;
  if (engine == DTR_ENGINE_CTA) {
    // Consecutive cells of the same shared-memory class form one launch: small
    // (<= 48 KiB: several CTAs per SM), large (<= 225 KiB staged), global (state
    // stays in the workspace).  Classes run concurrently on forked streams.
    static cudaStream_t cls_st[3];
    static cudaEvent_t fork_ev, join_ev[3];
    static bool init = false;
    static int sm_count = 0;
    if (!init) {
      int dev;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
      CK(cudaFuncSetAttribute(cta_engine<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX));
      CK(cudaFuncSetAttribute(cta_engine<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX));
      for (int k = 0; k < 3; k++) {
        CK(cudaStreamCreateWithFlags(&cls_st[k], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&join_ev[k], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
      init = true;
    }
    auto cls_of = [&](u32 i, u64 *need) -> int {
      u64 s = cta_smem_need(h_dims[3 * i], h_dims[3 * i + 1], h_dims[3 * i + 2]);
      *need = s;
      return s <= 48 * 1024 - 1024 ? 0 : (s <= CTA_SMEM_MAX ? 1 : 2);
    };
    bool used[3] = {false, false, false};
    u64 first_need;
    const int c_first = cls_of(0, &first_need);
    bool single = true;
    for (u32 i = 1; i < n_cells && single; i++) { u64 nd; single = cls_of(i, &nd) == c_first; }
    if (!single) CK(cudaEventRecord(fork_ev, st));
    u32 i = 0;
    while (i < n_cells) {
      u64 need;
      const int c = cls_of(i, &need);
      u64 smem = c == 2 ? 0 : need;
      u32 j = i + 1;
      bool cl = uses_closure(h_dims[3 * i + 2]);
      for (; j < n_cells; j++) {
        u64 nd;
        if (cls_of(j, &nd) != c) break;
        if (c != 2 && nd > smem) smem = nd;
        cl = cl || uses_closure(h_dims[3 * j + 2]);
      }
      smem = (smem + 15) & ~15ull;
      // at most one cell per SM: reserve more than half an SM's shared memory so
      // no two CTAs (each a latency-bound single-leader simulation) share an SM
      if (c != 2 && n_cells <= (u32)sm_count && !getenv("DTR_PACK_CTAS")) smem = std::max<u64>(smem, 116u * 1024u);
      cudaStream_t ls = st;
      if (!single) {
        ls = cls_st[c];
        if (!used[c]) { CK(cudaStreamWaitEvent(ls, fork_ev, 0)); used[c] = true; }
      }
      if (getenv("DTR_DEBUG")) fprintf(stderr, "dtr: cta launch cells [%u,%u) class %d smem %llu\n", i, j, c, smem);
      if (cl)   // the K5 closure pass is compiled only into this instantiation
        cta_engine<true><<<j - i, CTA_THREADS, smem, ls>>>(d_words, d_cells, i, j - i, ws, ws_bytes, d_rows, d_trace,
                                                         (u32)smem);
      else
        cta_engine<false><<<j - i, CTA_THREADS, smem, ls>>>(d_words, d_cells, i, j - i, ws, ws_bytes, d_rows,
                                                          d_trace, (u32)smem);
      CK(cudaGetLastError());
      i = j;
    }
    if (!single) {
      for (int k = 0; k < 3; k++) {
        if (!used[k]) continue;
        CK(cudaEventRecord(join_ev[k], cls_st[k]));
        CK(cudaStreamWaitEvent(st, join_ev[k], 0));
      }
    }
  } else {
    int blocks;
    rc = grid_blocks(&blocks);
    if (rc) return rc;
    for (u32 i = 0; i < n_cells; i++) {
      u32 ci = i;
      void *args[] = {(void *)&d_words, (void *)&d_cells, (void *)&ci, (void *)&ws, (void *)&ws_bytes,
                      (void *)&d_rows, (void *)&d_trace};
      CK(cudaLaunchCooperativeKernel((void *)grid_engine, dim3(blocks), dim3(GRID_THREADS), args, 0, st));
    }
  }
  return DTR_OK;
}

int dtr_pool_argmin(const uint32_t *d_log, uint32_t heuristic, void *d_ws, uint64_t *d_out, void *stream) {
  if (!d_log || !d_ws || !d_out || !valid_heuristic(heuristic)) return DTR_E_INVAL;
  int dev, sms, per_sm = 0, blocks;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pool_argmin_kernel, PA_THREADS, 0));
  blocks = sms * (per_sm < 1 ? 1 : per_sm);
  if (blocks > 4096) blocks = 4096;
  cudaStream_t st = (cudaStream_t)stream;
  void *args[] = {(void *)&d_log, (void *)&heuristic, (void *)&d_ws, (void *)&d_out};
  CK(cudaLaunchCooperativeKernel((void *)pool_argmin_kernel, dim3(blocks), dim3(PA_THREADS), args, 0, st));
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
  static bool pool_set = false;
  if (!pool_set) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set = true;
  }
  u32 *d_words = nullptr;
  dtr_cell *d_cells = nullptr;
  dtr_result *d_rows = nullptr;
  dtr_evict_rec *d_trace = nullptr;
  void *d_ws = nullptr;
  CK(cudaMallocAsync((void **)&d_words, n_words * 4, st));
  CK(cudaMallocAsync((void **)&d_cells, (size_t)n_cells * sizeof(dtr_cell), st));
  CK(cudaMallocAsync((void **)&d_rows, (size_t)n_cells * sizeof(dtr_result), st));
  if (h_trace && trace_total) CK(cudaMallocAsync((void **)&d_trace, trace_total * sizeof(dtr_evict_rec), st));
  CK(cudaMallocAsync(&d_ws, ws_bytes, st));
  CK(cudaMemcpyAsync(d_words, h_words, n_words * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_cells, h_cells, (size_t)n_cells * sizeof(dtr_cell), cudaMemcpyHostToDevice, st));
  rc = dtr_replay_batch(d_words, d_cells, dims.data(), n_cells, engine, d_ws, ws_bytes, d_rows, d_trace, st);
  if (rc == DTR_OK) {
    CK(cudaMemcpyAsync(h_rows, d_rows, (size_t)n_cells * sizeof(dtr_result), cudaMemcpyDeviceToHost, st));
    if (d_trace) CK(cudaMemcpyAsync(h_trace, d_trace, trace_total * sizeof(dtr_evict_rec), cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(d_words, st);
  cudaFreeAsync(d_cells, st);
  cudaFreeAsync(d_rows, st);
  if (d_trace) cudaFreeAsync(d_trace, st);
  cudaFreeAsync(d_ws, st);
  CK(cudaStreamSynchronize(st));
  return rc;
}

// ---------------------------------------------------------------------------
// Theorem 2 adversary batches
// ---------------------------------------------------------------------------
int dtr_adversary_workspace_bytes(const dtr_adversary *h_runs, uint32_t n_runs, uint64_t *bytes) {
  if (!bytes || (n_runs && !h_runs)) return DTR_E_INVAL;
  u64 total = 256;
  for (u32 i = 0; i < n_runs; i++) {
    const dtr_adversary &r = h_runs[i];
    if (r.n == 0 || r.n >= (1u << 27) || r.budget < 3 || !valid_heuristic(r.heuristic)) return DTR_E_INVAL;
    total += adv_bytes(r);
  }
  *bytes = total;
  return DTR_OK;
}

int dtr_adversary_batch(const dtr_adversary *d_runs, const dtr_adversary *h_runs, uint32_t n_runs, void *d_ws,
                        uint64_t ws_bytes, dtr_result *d_rows, uint32_t *d_parents, dtr_evict_rec *d_trace,
                        void *stream) {
  if (!d_runs || !h_runs || !d_rows || !d_parents || (n_runs && !d_ws)) return DTR_E_INVAL;
  if (n_runs == 0) return DTR_OK;
  uint64_t need = 0;
  int rc = dtr_adversary_workspace_bytes(h_runs, n_runs, &need);
  if (rc) return rc;
  if (ws_bytes < need) return DTR_E_CAPACITY;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(adversary_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX));
    attr = true;
  }
  u64 smem = 0;
  for (u32 i = 0; i < n_runs; i++) {
    Lay L;
    AdvLay A;
    adv_layout(L, A, h_runs[i].n, h_runs[i].budget, h_runs[i].heuristic);
    const u64 b = (u64)A.words * 4;
    if (b <= CTA_SMEM_MAX && b > smem) smem = b;
  }
  smem = (smem + 15) & ~15ull;
  adversary_engine<<<n_runs, CTA_THREADS, smem, (cudaStream_t)stream>>>(d_runs, n_runs, (char *)d_ws, ws_bytes,
                                                                       d_rows, d_parents, d_trace, (u32)smem);
  CK(cudaGetLastError());
  return DTR_OK;
}

// ---------------------------------------------------------------------------
// per-call runtime
// ---------------------------------------------------------------------------
struct dtr_runtime {
  dtr_config cfg;
  cudaStream_t st;
  Lay L;
  u32 *d_ws;
  Scalars *d_sc;
  dtr_evict_rec *d_trace;
  u64 *d_num, *d_den;
  u32 *d_ids;
  u64 score_cap;
  u32 edges;      // parent edges written so far
  Scalars hs;     // mirror of the device scalars after the last call
};

static int rt_sync_scalars(dtr_runtime *rt) {
  CK(cudaMemcpyAsync(&rt->hs, rt->d_sc, sizeof(Scalars), cudaMemcpyDeviceToHost, rt->st));
  CK(cudaStreamSynchronize(rt->st));
  return DTR_OK;
}

static int rt_launch(dtr_runtime *rt, u32 init, u32 op_word) {
  PercallArgs a;
  a.L = rt->L; a.base = rt->d_ws; a.sc = rt->d_sc;
  a.trace = rt->d_trace; a.onum = rt->d_num; a.oden = rt->d_den; a.oid = rt->d_ids;
  a.init = init;
  if (!init) {
    CK(cudaMemcpyAsync((char *)rt->d_sc + offsetof(Scalars, pending_op), &op_word, 4, cudaMemcpyHostToDevice,
                       rt->st));
  }
  percall_engine<<<1, CTA_THREADS, 0, rt->st>>>(a);
  CK(cudaGetLastError());
  return rt_sync_scalars(rt);
}

int dtr_create(const dtr_config *cfg, dtr_runtime **out) {
  if (!cfg || !out || cfg->cap_tensors == 0 || !valid_heuristic(cfg->heuristic) || cfg->dealloc > DEALLOC_IGNORE)
    return DTR_E_INVAL;
  if (cfg->cap_tensors >= (1u << 29)) return DTR_E_INVAL;
  dtr_runtime *rt = new dtr_runtime();
  rt->cfg = *cfg;
  rt->st = (cudaStream_t)cfg->stream;
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) { delete rt; return cuda_fail(e); }
  const u32 n = cfg->cap_tensors, E = cfg->cap_edges;
  if (!make_layout(rt->L, n, E, cfg->heuristic, 1, CTA_THREADS / 32)) { delete rt; return DTR_E_INVAL; }
  rt->score_cap = (u64)n + 1;
#define AL(p, bytes) do { e = cudaMalloc((void **)&(p), (bytes)); if (e != cudaSuccess) { dtr_destroy(rt); return cuda_fail(e); } } while (0)
  AL(rt->d_ws, (u64)rt->L.words * 4);
  AL(rt->d_sc, sizeof(Scalars));
  AL(rt->d_num, 8 * rt->score_cap);
  AL(rt->d_den, 8 * rt->score_cap);
  AL(rt->d_ids, 4 * rt->score_cap);
  if (cfg->trace_cap) AL(rt->d_trace, cfg->trace_cap * sizeof(dtr_evict_rec));
#undef AL
  rt->edges = 0;
  Scalars s;
  memset(&s, 0, sizeof s);
  s.B = cfg->budget; s.seed = cfg->seed; s.max_decisions = cfg->max_decisions; s.trace_cap = cfg->trace_cap;
  s.heuristic = cfg->heuristic; s.thrash_kill = cfg->thrash_kill; s.dealloc = cfg->dealloc;
  s.trace_hash = 14695981039346656037ull;
  norm_scalars(s);
  e = cudaMemcpyAsync(rt->d_sc, &s, sizeof s, cudaMemcpyHostToDevice, rt->st);
  if (e != cudaSuccess) { dtr_destroy(rt); return cuda_fail(e); }
  int rc = rt_launch(rt, 1, 0);
  if (rc) { dtr_destroy(rt); return rc; }
  *out = rt;
  return DTR_OK;
}

int dtr_destroy(dtr_runtime *rt) {
  if (!rt) return DTR_OK;
  cudaFree(rt->d_ws); cudaFree(rt->d_sc); cudaFree(rt->d_num); cudaFree(rt->d_den); cudaFree(rt->d_ids);
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
  const u32 t = rt->hs.n_alloc;
  std::vector<u32> ps;
  ps.reserve(n_parents);
  for (u32 j = 0; j < n_parents; j++) {
    if (parents[j] >= t) return DTR_E_INVAL;
    if (std::find(ps.begin(), ps.end(), parents[j]) == ps.end()) ps.push_back(parents[j]);
  }
  if (t >= rt->cfg.cap_tensors) return DTR_E_CAPACITY;
  if ((u64)rt->edges + ps.size() > rt->cfg.cap_edges) return DTR_E_CAPACITY;
  const uint4 sr = make_uint4(mem, compute, 0, 0);            // {mem, cost, la, nev}
  const uint2 pr = make_uint2(rt->edges, (u32)ps.size());     // {par_off, npar}
  CK(cudaMemcpyAsync(rt->d_ws + rt->L.srec + 4 * (u64)t, &sr, 16, cudaMemcpyHostToDevice, rt->st));
  CK(cudaMemcpyAsync(rt->d_ws + rt->L.arec + 4 * (u64)t, &pr, 8, cudaMemcpyHostToDevice, rt->st));
  if (!ps.empty())
    CK(cudaMemcpyAsync(rt->d_ws + rt->L.par + rt->edges, ps.data(), 4 * ps.size(), cudaMemcpyHostToDevice, rt->st));
  int rc = rt_launch(rt, 0, (OP_MAKE << 29) | t);
  if (rc) return rc;
  if (rt->hs.n_alloc == t + 1) {
    rt->edges += (u32)ps.size();
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
  CK(cudaMemcpyAsync((char *)rt->d_sc + offsetof(Scalars, B), &budget, 8, cudaMemcpyHostToDevice, rt->st));
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
