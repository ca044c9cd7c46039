#pragma once
// kcommon.cuh -- what the kernel translation units (k_*.cu) and the host ABI
// (dtr.cu) of libdtr.so share: constants, workspace layout, the team-parallel
// initialisation, and the launchers each k_*.cu defines.
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
#include <mutex>

#include "engine.cuh"
#include "leader.cuh"
#include "team.cuh"
#include "../../include/dtr.h"

namespace cg = cooperative_groups;
using namespace dtr;

#define CTA_THREADS 256
#define GRID_THREADS 512
#define WS_HEADER 164352ull  /* 512 + 4096 * (sizeof(Cand) + 16), multiple of 256 */
#define WS_BSTATS 98816      /* per-block {bytes, evals} for dtr_pool_argmin */
#define WS_SCALARS 128       /* grid engine: final Scalars of the last cell */
#define WS_PARTIALS 512
#define WS_PA_DONE 124       /* dtr_pool_argmin: blocks finished (u32; zeroed by the grid engine) */
#define CTA_SMEM_MAX (225u * 1024u)
#define CTA_WQ_PAIRS 384u    /* global-state cells: per-warp stack of deferred candidates (team.cuh SlowStack) */
#define CTA_WQ_BYTES (CTA_G_THREADS / 32 * (CTA_WQ_PAIRS * 8 + 32 * 8))   /* stacks + multi-walk sums: the
                                                                          dynamic shared memory of those launches */
// walk mirror of a global-state closure cell (engine.cuh Lay.mirror): u16 parent
// offsets and ids + the evicted bitmap, after the stacks in the dynamic smem
__host__ __device__ inline u64 mirror_bytes(u32 n, u32 E) {
  return (((u64)2 * (n + 1) + 3) & ~3ull) + (((u64)2 * E + 3) & ~3ull) + 4ull * ((n + 31) / 32 + 1);
}
__host__ __device__ inline bool mirror_ok(u32 n, u32 E, u32 heur) {
  return uses_closure(heur) && n < 65535 && E < 65535;
}
#define GRID_WQ_PAIRS 192u   /* whole-GPU teams: per-warp stack (>= 32 * 4 steps + 32) */  /* + ~1 KB static CtaShared <= 227 KB per block */

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
    if (g.L.ccache) g.ccache(t) = make_uint2(0, 0);
    if (g.L.lcache) g.m.w(g.L.lcache + t) = 0;
  }
  for (u32 j = rank; j < E; j += size) g.par(j) = lpar[j];
  for (u32 w = rank; w < g.L.pool_words; w += size) g.pool_word(w) = 0;
  if (uses_closure(heur)) {
    const u32 words = g.L.msps_words * g.L.msps_warps;
    for (u32 i = rank; i < words; i += size) g.m.w(g.L.msps_bm + i) = 0;
    if (g.L.msps_lock)
      for (u32 i = rank; i < g.L.msps_warps; i += size) g.m.w(g.L.msps_lock + i) = 0;
    if (g.L.msps_d) {
      const u32 dw = (g.L.n + 1) * g.L.msps_warps;
      for (u32 i = rank; i < dw; i += size) g.m.w(g.L.msps_d + i) = 0;
    }
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

static __device__ void init_scalars(Scalars &s, const dtr_cell &cell) {
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

static __device__ __forceinline__ u64 gtimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// t0: gtimer() at the start of the run (0: wall_ns = 0)
static __device__ void write_row(dtr_result &r, const Scalars &s, u64 bytes, u64 evals, u64 t0 = 0) {
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
  x.wall_ns = t0 ? gtimer() - t0 : 0;
  r = x;
}

// the closure-cache events travel with an ARGMIN command (the team processes
// them before scoring) and are consumed by it
__device__ __forceinline__ void publish(Cmd &c, u32 kind, Scalars &s) {
  c.kind = kind; c.pool_size = s.pool_size; c.clock = s.clock; c.decisions = s.decisions;
  c.seed = s.seed; c.heur = s.heuristic; c.n_ids = s.n_alloc;
  c.n_ev = s.ev_n;
  if (kind == CMD_ARGMIN) s.ev_n = 0;
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
// 0 = the layout does not fit 32-bit word offsets (DTR_E_CAPACITY)
__host__ __device__ inline bool cell_layout(Lay &L, u32 n, u32 E, u32 heur, u32 engine) {
  const bool grid = engine == DTR_ENGINE_GRID;
  return make_layout(L, n, E, heur, 0, grid ? grid_closure_slots(n) : CTA_THREADS / 32, grid, 1);
}
__host__ __device__ inline u64 cell_bytes(u32 n, u32 E, u32 heur, u32 engine) {
  Lay L;
  if (!cell_layout(L, n, E, heur, engine)) return 0;
  return ((u64)L.words * 4 + 255) & ~255ull;
}

__host__ __device__ inline u64 cta_smem_need(u32 n, u32 E, u32 heur) {
  Lay L;
  make_layout(L, n, E, heur, 0, CTA_THREADS / 32);
  return (u64)L.words * 4;
}

#define PA_THREADS 256

#define CTA_G_THREADS 512   /* K6 for cells whose state stays in global memory (cta_engine_g) */

struct __align__(16) CtaShared {
  Cmd cmd;
  RedSmem red;
  ScanSmem scan;
  u32 msps_tail[CTA_G_THREADS / 32];
  u32 best;                          // the CTA team's best pass-1 key (score_stream pruning)
};

struct PercallArgs {
  Lay L;
  u32 *base;
  Scalars *sc;
  dtr_evict_rec *trace;
  u64 *onum, *oden;
  u32 *oid;
  u32 init;         // first launch: initialise state
};

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


// ---------------------------------------------------------------------------
// Launchers (host side of each kernel translation unit).  Each returns the
// CUDA error of its attribute call or launch.
// ---------------------------------------------------------------------------
namespace dtr {
// k_cta_cl.cu / k_cta_nocl.cu: K6 with / without the K5 closure pass
cudaError_t cta_set_attrs_cl();
cudaError_t cta_set_attrs_nocl();
cudaError_t launch_cta_cl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 c0,
                          char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace);
cudaError_t launch_cta_nocl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 c0,
                            char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace);
// the same for cells whose state stays in global memory (CTA_G_THREADS threads, smem = CTA_WQ_BYTES)
cudaError_t launch_cta_g_cl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 c0,
                            char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace);
cudaError_t launch_cta_g_nocl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 c0,
                              char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace);
// k_grid.cu: K7 and the standalone K3+K4
cudaError_t grid_occupancy(int *grid_per_sm, int *pa_per_sm);
cudaError_t launch_grid(int blocks, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 ci, char *ws,
                        u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace);
cudaError_t launch_pool_argmin(int blocks, cudaStream_t st, const u32 *logw, u32 heur, char *ws, u64 *out);
// k_percall.cu
cudaError_t launch_percall(const PercallArgs &a, cudaStream_t st);
// k_adv.cu: K8
cudaError_t adv_set_attrs();
cudaError_t launch_adv(u32 n_runs, u32 smem, cudaStream_t st, const dtr_adversary *runs, char *ws, u64 ws_bytes,
                       dtr_result *rows, u32 *parents, dtr_evict_rec *trace);
#ifdef DTR_PROFILE
// clock64 phase counters: every translation unit has its own copy; summed into out
cudaError_t prof_read_cta_cl(unsigned long long *out, int reset);
cudaError_t prof_read_cta_nocl(unsigned long long *out, int reset);
cudaError_t prof_read_grid(unsigned long long *out, int reset);
cudaError_t prof_read_percall(unsigned long long *out, int reset);
cudaError_t prof_read_adv(unsigned long long *out, int reset);
#endif
}  // namespace dtr
