// k_adv.cu -- K8, the Theorem 2 online adversary.
#include "kcommon.cuh"

namespace cg = cooperative_groups;
using namespace dtr;

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
  const u64 t_start = gtimer();
  Sim<SM> g;
  g.m.gbase = gbase;
  AdvLay A;
  adv_layout(g.L, A, N, B, run.heuristic);
  g.m.lim = A.words;
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
  if (tid == 0) write_row(*row, L.s, bytes, evals, t_start);
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


// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
namespace dtr {

cudaError_t adv_set_attrs() {
  return cudaFuncSetAttribute(adversary_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX);
}

cudaError_t launch_adv(u32 n_runs, u32 smem, cudaStream_t st, const dtr_adversary *runs, char *ws, u64 ws_bytes,
                       dtr_result *rows, u32 *parents, dtr_evict_rec *trace) {
  adversary_engine<<<n_runs, CTA_THREADS, smem, st>>>(runs, n_runs, ws, ws_bytes, rows, parents, trace, smem);
  return cudaGetLastError();
}

#ifdef DTR_PROFILE
cudaError_t prof_read_adv(unsigned long long *out, int reset) {
  unsigned long long v[PROF_N];
  cudaError_t e = cudaMemcpyFromSymbol(v, g_prof, sizeof v);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < PROF_N; i++) out[i] += v[i];
  if (reset) { unsigned long long z[PROF_N] = {0}; e = cudaMemcpyToSymbol(g_prof, z, sizeof z); }
  return e;
}
#endif
}  // namespace dtr
