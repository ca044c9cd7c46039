// k_grid.cu -- K7, the whole GPU on one simulation, and K3+K4 alone (dtr_pool_argmin).
#include "kcommon.cuh"

namespace cg = cooperative_groups;
using namespace dtr;

// ---------------------------------------------------------------------------
// K7: the whole GPU on one simulation (cooperative launch).
// ---------------------------------------------------------------------------
struct __align__(16) GridShared {
  Cmd cmd;
  RedSmem red;
  ScanSmem scan;
  u32 msps_tail[GRID_THREADS / 32];
  uint2 wq[GRID_THREADS / 32][GRID_WQ_PAIRS];   // per-warp stacks of deferred candidates
  u64 msum[GRID_THREADS / 32][32];                // per-warp sums of the multi-candidate closure walk
  u32 best;                           // the block's best pass-1 key (score_stream pruning)
};

struct GridSync {
  __device__ void operator()() const { cg::this_grid().sync(); }
};

__global__ void __launch_bounds__(GRID_THREADS, 1) grid_engine(const u32 *words, const dtr_cell *cells, u32 ci,
                                                            char *ws, u64 ws_bytes, dtr_result *rows,
                                                            dtr_evict_rec *trace) {
  __shared__ GridShared sh;
  cg::grid_group grid = cg::this_grid();
  const u64 t_start = gtimer();
  const u32 tid = threadIdx.x;
  Cmd *gcmd = (Cmd *)ws;
  u64 *gstats = (u64 *)(ws + 64);   // [bytes, evals]
  Cand *partials = (Cand *)(ws + WS_PARTIALS);
  const dtr_cell cell = cells[ci];
  const u32 *logw = words + cell.log_offset;
  const u64 mine = cell_bytes(logw[2], logw[3], cell.heuristic, DTR_ENGINE_GRID);
  if (mine == 0 || WS_HEADER + mine > ws_bytes) {
    if (blockIdx.x == 0 && tid == 0) {
      dtr_result r; memset(&r, 0, sizeof r);
      r.cell_id = cell.cell_id; r.status = ST_CAPACITY;
      rows[ci] = r;
    }
    return;
  }
  Sim<false> g;
  g.m.gbase = (u32 *)(ws + WS_HEADER);
  cell_layout(g.L, logw[2], logw[3], cell.heuristic, DTR_ENGINE_GRID);
  g.m.lim = g.L.words;
  const u32 rank = blockIdx.x * blockDim.x + tid, size = gridDim.x * blockDim.x;
  const u32 wrank = rank >> 5, wsize = size >> 5;
  if (rank == 0) { gstats[0] = 0; gstats[1] = 0; *(u32 *)(ws + WS_PA_DONE) = 0; }
  init_sim(g, logw, rank, size, blockIdx.x == 0, sh.scan, GridSync());
  Leader<false, true> L;
  if (rank == 0) leader_init(L, g, logw, cell, trace);
  Cand res = cand_none();
  bool have = false;
  u64 bytes = 0, evals = 0;
  PROF_T(tg0);
  for (;;) {
    if (rank < 32) {                // the leader's warp
      Cmd c;
      u32 n_ev = 0, kind = 0;
      if (rank == 0) {
        PROF_T(a0);
        kind = L.resume(have, res);
        have = false;
        publish(c, kind, L.s);
        n_ev = c.n_ev;
        PROF_T(a1);
        PROF_ADD(0, a1 - a0);
      }
      // closure caches: the warp walks the queued events (slot 0; every other
      // warp is parked at the barrier below) before any scoring
      n_ev = __shfl_sync(0xffffffffu, n_ev, 0);
      kind = __shfl_sync(0xffffffffu, kind, 0);
      if (kind == CMD_ARGMIN && n_ev) {
        Cmd e;
        e.n_ev = n_ev; e.kind = kind; e.heur = cell.heuristic; e.n_ids = __shfl_sync(0xffffffffu, L.s.n_alloc, 0);
        closure_events(g, e, 0, sh.msps_tail);
      }
      if (rank == 0) *gcmd = c;
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
      c.n_ev = __ldcg(&gcmd->n_ev);
      sh.cmd = c;
      sh.best = KEY_NONE;
    }
    __syncthreads();
    if (sh.cmd.kind != CMD_ARGMIN) break;
    u32 bk;
    PROF_T(c0);
    Cand best = team_score<false, true, true>(g, sh.cmd, rank, size, wrank, wsize, sh.msps_tail, bytes, evals, bk,
                                              SlowStack{sh.wq[tid >> 5], GRID_WQ_PAIRS, sh.msum[tid >> 5]}, &sh.best);
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
    write_row(rows[ci], L.s, __ldcg(&gstats[0]), __ldcg(&gstats[1]), t_start);
    *(Scalars *)(ws + WS_SCALARS) = L.s;   // kept for dtr_pool_argmin
  }
}

// ---------------------------------------------------------------------------
// K3+K4 alone: score the current pool of the simulation left in a grid-engine
// workspace and reduce its argmin.  A plain (non-cooperative) persistent launch:
// every block writes its partial, and the LAST block to finish (a counter in
// the workspace header) reduces them -- no grid barrier anywhere.  Used to time
// the score pass in isolation (bench roofline_large_pool).
// ---------------------------------------------------------------------------
struct __align__(16) PaShared {
  RedSmem red;
  u32 msps_tail[PA_THREADS / 32];
  uint2 wq[PA_THREADS / 32][GRID_WQ_PAIRS];
  u64 msum[PA_THREADS / 32][32];
  u32 last, best;
};

// CL = false: the instantiation without the K5 closure pass (the hot h_DTR /
// h_DTR_eq pass then needs no spills under the 64-register bound)
template <bool CL>
__global__ void __launch_bounds__(PA_THREADS, 4) pool_argmin_kernel(const u32 *logw, u32 heur, char *ws,
                                                                    u64 *out /* num, den, id, bytes, evals */) {
  __shared__ PaShared sh;
  const u32 tid = threadIdx.x;
  Cand *partials = (Cand *)(ws + WS_PARTIALS);
  u32 *done = (u32 *)(ws + WS_PA_DONE);          // blocks finished (the last one resets it)
  Sim<false> g;
  g.m.gbase = (u32 *)(ws + WS_HEADER);
  cell_layout(g.L, logw[2], logw[3], heur, DTR_ENGINE_GRID);
  g.m.lim = g.L.words;
  const Scalars *sc = (const Scalars *)(ws + WS_SCALARS);
  Cmd cmd;
  cmd.kind = CMD_ARGMIN; cmd.pool_size = sc->pool_size; cmd.clock = sc->clock; cmd.decisions = sc->decisions;
  cmd.seed = sc->seed; cmd.heur = heur; cmd.n_ids = sc->n_alloc;
  cmd.n_ev = NONE;                 // the closure caches may lag the last decisions' events
  const u32 rank = blockIdx.x * blockDim.x + tid, size = gridDim.x * blockDim.x;
  u64 bytes = 0, evals = 0;
  u32 bk;
  if (tid == 0) sh.best = KEY_NONE;
  __syncthreads();
  Cand best = team_score<false, true, true, CL>(g, cmd, rank, size, rank >> 5, size >> 5, sh.msps_tail, bytes, evals,
                                                bk, SlowStack{sh.wq[tid >> 5], GRID_WQ_PAIRS, sh.msum[tid >> 5]},
                                                &sh.best);
  const bool ik = int_key_heur(heur);
  best = block_argmin(best, bk, sh.red, ik);
  block_sum2(bytes, evals, sh.red);
  u64 *bstats = (u64 *)(ws + WS_BSTATS);
  if (tid == 0) {
    partials[blockIdx.x] = best;
    bstats[2 * blockIdx.x] = bytes;
    bstats[2 * blockIdx.x + 1] = evals;
    __threadfence();
    sh.last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (sh.last) {                 // the last block reduces the partials (all loads in flight)
    __threadfence();
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
    if (tid == 0) { out[0] = w.num; out[1] = w.den; out[2] = w.id; out[3] = tb; out[4] = te; *done = 0; }
  }
}


// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
namespace dtr {

cudaError_t grid_occupancy(int *grid_per_sm, int *pa_per_sm) {
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(grid_per_sm, grid_engine, GRID_THREADS, 0);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(pa_per_sm, pool_argmin_kernel<false>, PA_THREADS, 0);
}

cudaError_t launch_grid(int blocks, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 ci, char *ws,
                        u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace) {
  void *args[] = {(void *)&words, (void *)&cells, (void *)&ci, (void *)&ws, (void *)&ws_bytes, (void *)&rows,
                  (void *)&trace};
  return cudaLaunchCooperativeKernel((void *)grid_engine, dim3(blocks), dim3(GRID_THREADS), args, 0, st);
}

cudaError_t launch_pool_argmin(int blocks, cudaStream_t st, const u32 *logw, u32 heur, char *ws, u64 *out) {
  if (uses_closure(heur)) pool_argmin_kernel<true><<<blocks, PA_THREADS, 0, st>>>(logw, heur, ws, out);
  else pool_argmin_kernel<false><<<blocks, PA_THREADS, 0, st>>>(logw, heur, ws, out);
  return cudaGetLastError();
}

#ifdef DTR_PROFILE
cudaError_t prof_read_grid(unsigned long long *out, int reset) {
  unsigned long long v[PROF_N];
  cudaError_t e = cudaMemcpyFromSymbol(v, g_prof, sizeof v);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < PROF_N; i++) out[i] += v[i];
  if (reset) { unsigned long long z[PROF_N] = {0}; e = cudaMemcpyToSymbol(g_prof, z, sizeof z); }
  return e;
}
#endif
}  // namespace dtr
