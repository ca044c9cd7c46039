// k_percall.cu -- the per-call runtime engine (simrd external API).
#include "kcommon.cuh"

namespace cg = cooperative_groups;
using namespace dtr;

// ---------------------------------------------------------------------------
// Per-call engine: apply ONE record to the persistent state of a runtime
// (global memory, linked children; the host writes srec[t] and the parent ids
// of each new tensor before the MAKE launch).
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(CTA_THREADS) percall_engine(PercallArgs a) {
  __shared__ CtaShared sh;
  const u32 tid = threadIdx.x;
  Sim<false> g;
  g.m.gbase = a.base;
  g.L = a.L;
  g.m.lim = g.L.words;
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
// Launchers
// ---------------------------------------------------------------------------
namespace dtr {

cudaError_t launch_percall(const PercallArgs &a, cudaStream_t st) {
  percall_engine<<<1, CTA_THREADS, 0, st>>>(a);
  return cudaGetLastError();
}

#ifdef DTR_PROFILE
cudaError_t prof_read_percall(unsigned long long *out, int reset) {
  unsigned long long v[PROF_N];
  cudaError_t e = cudaMemcpyFromSymbol(v, g_prof, sizeof v);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < PROF_N; i++) out[i] += v[i];
  if (reset) { unsigned long long z[PROF_N] = {0}; e = cudaMemcpyToSymbol(g_prof, z, sizeof z); }
  return e;
}
#endif
}  // namespace dtr
