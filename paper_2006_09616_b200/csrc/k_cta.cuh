#pragma once
// k_cta.cuh -- K6, one CTA per simulation (many small runs of a sweep).
// Included by k_cta_cl.cu (the instantiation with the K5 closure pass) and
// k_cta_nocl.cu (without it), two translation units compiled in parallel.
#include "kcommon.cuh"

namespace cg = cooperative_groups;
using namespace dtr;

// ---------------------------------------------------------------------------
// K6: one CTA per simulation.
// ---------------------------------------------------------------------------

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
  r.n_ev = __shfl_sync(0xffffffffu, c.n_ev, 0);
  return r;
}

// CL = false: compiled without the K5 closure pass (batches whose cells use
// no closure heuristic): the leader's hot path then shares its kernel with
// less cold code (measured 3.5 % faster on the bench's critical cells).
template <bool SM, bool CL>
__device__ void run_cta(const u32 *logw, const dtr_cell &cell, u32 *gbase, dtr_result *row, dtr_evict_rec *trace,
                        CtaShared &sh, u32 smem_bytes) {
  const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Sim<SM> g;
  g.m.gbase = gbase;
  make_layout(g.L, logw[2], logw[3], cell.heuristic, 0, CTA_THREADS / 32, 0, SM ? 0 : 1);
  g.m.lim = g.L.words;
  PROF_T(ti0);
  const u64 t_start = gtimer();
  init_sim(g, logw, tid, blockDim.x, true, sh.scan, CtaSync());
  if constexpr (!SM) {
    // closure heuristics: the walk mirror after the stacks, when the launch reserved room for it
    const u32 n = g.L.n, E = g.L.E;
    const u32 base = (blockDim.x >> 5) * (CTA_WQ_PAIRS * 8 + 32 * 8);
    if (mirror_ok(n, E, cell.heuristic) && base + mirror_bytes(n, E) <= smem_bytes) {
      g.L.mirror = 1;
      g.L.mo_off = base;
      g.L.mo_par = base + (u32)(((u64)2 * (n + 1) + 3) & ~3ull);
      g.L.mo_ev = g.L.mo_par + (u32)(((u64)2 * E + 3) & ~3ull);
      const u32 *loff = logw + 16 + 2 * n, *lpar = loff + n + 1;
      unsigned short *o = reinterpret_cast<unsigned short *>(reinterpret_cast<char *>(g_smem) + g.L.mo_off);
      unsigned short *pp = reinterpret_cast<unsigned short *>(reinterpret_cast<char *>(g_smem) + g.L.mo_par);
      u32 *ev = reinterpret_cast<u32 *>(reinterpret_cast<char *>(g_smem) + g.L.mo_ev);
      for (u32 t = tid; t <= n; t += blockDim.x) o[t] = (unsigned short)loff[t];
      for (u32 j = tid; j < E; j += blockDim.x) pp[j] = (unsigned short)lpar[j];
      for (u32 w = tid; w <= (n + 31) / 32; w += blockDim.x) ev[w] = 0;
      __syncthreads();
    }
  }
  PROF_T(ti1);
  if (tid == 0) PROF_ADD(6, ti1 - ti0);
  u64 bytes = 0, evals = 0;
  // global-memory state: the dynamic shared memory holds the per-warp slow stacks (score_stream)
  const u32 nwarps = blockDim.x >> 5;
  const SlowStack wq = SM ? SlowStack{nullptr, 0, nullptr}
                          : SlowStack{reinterpret_cast<uint2 *>(g_smem) + warp * CTA_WQ_PAIRS, CTA_WQ_PAIRS,
                                      reinterpret_cast<u64 *>(g_smem + 2 * nwarps * CTA_WQ_PAIRS) + 32 * warp};
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
      if constexpr (CL) {   // closure caches: warp 0 walks the queued events (slot 0) before any scoring
        if (c.kind == CMD_ARGMIN && c.n_ev) closure_events(g, c, 0, sh.msps_tail);
      }
      if (c.kind == CMD_ARGMIN && c.pool_size <= WARP_TEAM_MAX && g.L.pool_key) {   // size / LRU: 64-bit keys
        PROF_T(t2);
        const u64 k = warp_min64(team_intkey_min(g, c, lane, 32, bytes, evals));
        PROF_T(t3);
        if (lane == 0) { res = intkey_cand(g, c, k); have = true; PROF_ADD(1, t3 - t2); PROF_ADD(3, 1); }
        continue;
      }
      // closure heuristics on global state: always the whole CTA (deep closure walks
      // dominate there, and eight warps drain their stacks concurrently)
      if (c.kind == CMD_ARGMIN && c.pool_size <= WARP_TEAM_MAX && (SM || !CL || !uses_closure(c.heur))) {
        PROF_T(t2);
        u32 bk;
        Cand best = team_score<SM, false, false, CL>(g, c, lane, 32, 0, 1, sh.msps_tail, bytes, evals, bk, wq);
        PROF_T(t3);
        best = warp_argmin_fast(best, bk, int_key_heur(c.heur));
        PROF_T(t4);
        if (lane == 0) { res = best; have = true; PROF_ADD(1, t3 - t2); PROF_ADD(2, t4 - t3); PROF_ADD(3, 1); }
        continue;
      }
      PROF_T(t5);
      if (lane == 0) { sh.cmd = c; sh.best = KEY_NONE; }
      __syncthreads();
      if (c.kind != CMD_ARGMIN) break;
      u32 bk;
      Cand best = team_score<SM, false, false, CL>(g, c, tid, blockDim.x, warp, blockDim.x >> 5, sh.msps_tail, bytes, evals, bk, wq,
                                                   &sh.best);
      best = block_argmin(best, bk, sh.red, int_key_heur(c.heur));
      PROF_T(t6);
      if (lane == 0) { res = best; have = true; PROF_ADD(4, t6 - t5); PROF_ADD(5, 1); }
    }
    if (lane == 0) write_row(*row, L.s, 0, 0, t_start);
  } else {
    for (;;) {
      __syncthreads();
      const Cmd c = sh.cmd;
      if (c.kind != CMD_ARGMIN) break;
      u32 bk;
      Cand best = team_score<SM, false, false, CL>(g, c, tid, blockDim.x, warp, blockDim.x >> 5, sh.msps_tail, bytes, evals, bk, wq,
                                                   &sh.best);
      block_argmin(best, bk, sh.red, int_key_heur(c.heur));
    }
  }
  block_sum2(bytes, evals, sh.red);
  if (tid == 0) { row->score_bytes = bytes; row->cand_evals = evals; }
}

// G = false: cells whose state is staged in shared memory (CTA_THREADS);
// G = true: cells whose state stays in the global workspace (CTA_G_THREADS:
// twice the warps to hide the L2 latency of the score pass; the leader then
// compiles under 128 registers, as in the whole-GPU engine)
template <bool CL, bool G>
__device__ __forceinline__ void cta_body(const u32 *words, const dtr_cell *cells, u32 c0, u32 n_run, char *ws,
                                         u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace, u32 smem_bytes,
                                         CtaShared &sh) {
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
  const u64 mine = cell_bytes(logw[2], logw[3], cell.heuristic, DTR_ENGINE_CTA);
  const bool fits = cta_smem_need(logw[2], logw[3], cell.heuristic) <= smem_bytes;
  if (mine == 0 || off + mine > ws_bytes || fits == G) {   // G launches take exactly the cells that do not fit
    if (tid == 0) {
      dtr_result r; memset(&r, 0, sizeof r);
      r.cell_id = cell.cell_id; r.status = ST_CAPACITY;
      rows[ci] = r;
    }
    return;
  }
  if constexpr (G) run_cta<false, CL>(logw, cell, (u32 *)(ws + off), &rows[ci], trace, sh, smem_bytes);
  else run_cta<true, CL>(logw, cell, nullptr, &rows[ci], trace, sh, smem_bytes);
}

template <bool CL>
__global__ void __launch_bounds__(CTA_THREADS, 1) cta_engine(const u32 *words, const dtr_cell *cells, u32 c0, u32 n_run,
                                                          char *ws, u64 ws_bytes, dtr_result *rows,
                                                          dtr_evict_rec *trace, u32 smem_bytes) {
  __shared__ CtaShared sh;
  cta_body<CL, false>(words, cells, c0, n_run, ws, ws_bytes, rows, trace, smem_bytes, sh);
}

template <bool CL>
__global__ void __launch_bounds__(CTA_G_THREADS, 1) cta_engine_g(const u32 *words, const dtr_cell *cells, u32 c0,
                                                              u32 n_run, char *ws, u64 ws_bytes, dtr_result *rows,
                                                              dtr_evict_rec *trace, u32 smem_bytes) {
  __shared__ CtaShared sh;
  cta_body<CL, true>(words, cells, c0, n_run, ws, ws_bytes, rows, trace, smem_bytes, sh);
}
