// engine.cuh -- device side of the DTR eviction-decision engine (sm_100a).
//
// One simulation = the simrd runtime with V2 banishing (PAPER.md Doc A,
// P:113-373).  Its control (make_tensor / get_internal recursion /
// release_internal / free / evict) is inherently sequential and runs
// on ONE leader thread as a resumable state machine with an explicit stack
// (leader.cuh); whenever free() needs a decision the leader hands the
// pool to its TEAM -- a whole CTA (one small simulation per CTA) or the whole
// grid (one large simulation per GPU) -- which scores every pool member and
// reduces the exact (score, id) argmin (team.cuh).
//
// Memory: every array of a simulation is addressed by a 32-bit WORD offset from
// one base -- the CTA's dynamic shared memory (SM = true: LDS/STS, 32-bit
// addresses) or the simulation's global workspace (SM = false).
//   srec[t] = {mem, cost, la, nev}                 the score record: mem and cost
//             static (from the log), la and nev dynamic -- everything a
//             candidate with no evicted neighbour needs, in one 16-B load
//   arec[t] = {par_off, npar, ch_off, nch}         adjacency record; the children
//             half (crec) is built on device | linked: {head, -}
//   state[t], rho[t], ell[t]                      (dynamic, compact u32 arrays: a
//             neighbour's state word shares its sector with nearby ids)
//   pool     R.pool (t.m = T and t.l = 0), one of two representations:
//            - compact list pool_ids[] + pool_pos[] (CTA engine, per-call): the
//              team scans exactly the P members;
//            - bitmap over tensor ids (whole-GPU engine): the team scans ids in
//              order, so a warp's candidates are consecutive ids whose (mostly
//              nearby) neighbours share sectors and L1 lines
//   state: bit31 material (t.m = T), bit30 computed once (reading C-19),
//          bit29 V1-banished, bits 0..28 label of t's evicted component (h_DTR;
//          a label is a slot of the component table, recycled through a free stack)
//   la:    last_access + 1, 0 = -inf (banish_V2)
//   nev:   number of t's neighbours (parents, children) that are evicted --
//          maintained by the leader on evict / rematerialize / V1 banish for the
//          heuristics that read neighbourhoods (Lay.track_nev); nev = 0 means
//          E(t) = e*(t) = e_R(t) = {} and the score needs no neighbour walk
//
// Independent of oracle/ (shares no code with it).
#pragma once
#include <stdint.h>

#ifdef DTR_PROFILE
// clock64 phase counters (probe builds only, scripts/probe_prof*.py):
// [0] leader resume cycles, [1] warp-team score cycles, [2] warp reduce cycles,
// [3] warp-team decisions, [4] cta-team cycles, [5] cta-team decisions, [6] init cycles,
// [8/9] record_and_evict cycles/calls, [10/11] complete_top, [12/13] push, [14] resume loop iterations
#define PROF_N 32
static __device__ unsigned long long g_prof[PROF_N];
#define PROF_T(x) unsigned long long x = clock64()
#define PROF_ADD(i, v) atomicAdd(&g_prof[i], (unsigned long long)(v))
#else
#define PROF_T(x)
#define PROF_ADD(i, v)
#endif

namespace dtr {

typedef uint32_t u32;
typedef unsigned long long u64;
typedef unsigned __int128 u128;

constexpr u32 NONE = 0xFFFFFFFFu;
constexpr u32 M_BIT = 1u << 31;
constexpr u32 O_BIT = 1u << 30;
constexpr u32 B_BIT = 1u << 29;              // V1-banished: removed from the graph
constexpr u32 COMP_MASK = (1u << 29) - 1;
constexpr u32 LIVE_BIT = 1u << 31;           // union-find compaction mark (in uf size)
constexpr u64 CLOCK_LIMIT = 0xFFFFFFFEull;   // reading C-14: la is stored as clock + 1 in u32

enum { H_DTR = 0, H_DTR_EQ = 1, H_LRU = 2, H_SIZE = 3, H_MSPS = 4, H_LOCAL = 5, H_RANDOM = 6,
       H_DTR_FULL = 7, H_ESTAR = 8, H_LAST = 8 };
// the D.1 ablation h'(s, m, c) (reading C-23): id = H_ABL + 4*c + 2*m + s,
// c in {e*, EqClass, local, no}
enum { H_ABL = 16, H_ABL_END = 32, ABL_ESTAR = 0, ABL_EQCLASS = 1, ABL_LOCAL = 2, ABL_NO = 3 };
__host__ __device__ __forceinline__ bool is_abl(u32 h) { return h >= H_ABL && h < H_ABL_END; }
__host__ __device__ __forceinline__ u32 abl_c(u32 h) { return (h - H_ABL) >> 2; }
__host__ __device__ __forceinline__ bool valid_heuristic(u32 h) { return h <= H_LAST || is_abl(h); }
// directed closures walked per candidate by one warp (MSPS, e*)
__host__ __device__ __forceinline__ bool uses_closure(u32 h) {
  return h == H_MSPS || h == H_DTR_FULL || h == H_ESTAR || (is_abl(h) && abl_c(h) == ABL_ESTAR);
}
// Integer keys (ik): h_size and h_LRU scores are 1/m and 1/s with integer m, s,
// so they order exactly by an integer: ~m, resp. la (encoded last access; 0 =
// -inf gives score 0, clock + 1 gives s = 0 = +inf); no division is needed.
__host__ __device__ __forceinline__ bool int_key_heur(u32 h) { return h == H_SIZE || h == H_LRU; }
// union-find evicted components
__host__ __device__ __forceinline__ bool uses_uf(u32 h) { return h == H_DTR_EQ || (is_abl(h) && abl_c(h) == ABL_EQCLASS); }
enum { OP_MAKE = 1, OP_GET = 2, OP_RELEASE = 3, OP_REMAT = 4, OP_ENSURE = 5, OP_DEBUG_EVICT = 6,
       OP_SCORES = 7 /* per-call only: score the whole pool */ };
// Cached closure sums (App. C "Caching metadata"): the
// leader queues every tensor whose evicted status flips (evict, finished
// rematerialization, V1 banish of an evicted tensor); before the next score
// pass the team walks from each queued tensor and marks stale the caches it may
// have changed.  More than EVQ_CAP events between two decisions = all stale.
constexpr u32 EVQ_CAP = 1024;
enum { DEALLOC_V2 = 0, DEALLOC_V1 = 1, DEALLOC_EAGER = 2, DEALLOC_IGNORE = 3 };
enum { ST_OK = 0, ST_INVAL = 1, ST_PRECOND = 2, ST_OOM = 3, ST_THRASH = 4, ST_CAPACITY = 5,
       ST_STATE = 6, ST_DECISION_CAP = 8 };

__host__ __device__ __forceinline__ bool is_evicted(u32 s) { return (s & (M_BIT | O_BIT | B_BIT)) == O_BIT; }
__host__ __device__ __forceinline__ bool is_banished(u32 s) { return (s & B_BIT) != 0; }
__host__ __device__ __forceinline__ bool is_material(u32 s) { return (s & M_BIT) != 0; }

// ---------------------------------------------------------------------------
// Layout: word offsets of every array of one simulation.
// ---------------------------------------------------------------------------
struct Lay {
  u32 n, E, heur, linked, track_nev;
  u32 srec, arec, par, ch, state, rho, ell, pool_bm, pool_words, pool_ids, pool_pos, fr, pb;
  u32 pool_key;                                        // compact list, size/LRU: u64 key per slot (0 = none)
  u32 mem_next, comp, comp_head, bfs_q, stamp;         // h_DTR (comp rec: {cost, nmax, maxla, size})
  u32 mem_prev, comp_free;                             // h_DTR: member lists are doubly linked; free label slots
  u32 node_of, uf, uf_size, uf_cap;                    // h_DTR_eq (uf rec: {cost lo, cost hi, maxla, parent})
  u32 msps_bm, msps_q, msps_words, msps_warps;         // closure BFS scratch: msps_warps slots
  u32 msps_lock;                                       // grid: slot locks (0 = CTA: slot = warp)
  u32 msps_d;                                          // per slot: candidate masks of the multi-candidate walk (0 = none)
  u32 e_next, e_child;                                 // linked children (per-call)
  u32 ccache, evq;                                     // closure cache {up+1, down+1} per tensor (0 = stale)
                                                       // + the leader's event queue (batch engines only)
  // walk mirror (global-state CTA cells of closure heuristics, when the launch's
  // dynamic shared memory has room): parent CSR as u16 + an evicted bitmap in
  // shared memory, so closure walks chase pointers at shared-memory latency.
  // Byte offsets into the dynamic shared memory; mirror = 0: none.
  u32 mirror, mo_off, mo_par, mo_ev;
  // h_DTR_eq (batch engines): per tensor the max union-find-root maxla of its
  // adjacent evicted components at its last exact score, + 1 (0 = none).  Root
  // maxla never decreases (reading C-9) and the adjacent roots only merge while
  // no neighbour flips, so it stays a LOWER bound of that max until the leader
  // clears it on a neighbour's flip: a tighter pruning bound (score_stream).
  u32 lcache;
  u32 words;                                           // total
};

// Sizes the workspace (host) and places it (device).  Returns false when the
// layout does not fit 32-bit word offsets (the caller reports DTR_E_CAPACITY).
// msps_warps: closure-BFS scratch slots (one per scoring warp on a CTA; on the
// whole-GPU engine a bounded number of slots that warps lock, grid_closure_slots).
// multi (global-state cells and the whole-GPU engine): closure heuristics get the
// per-slot mask arrays of the multi-candidate walk (closure_multi), h_DTR_eq the
// lcache pruning bound (score_stream).
__host__ __device__ inline bool make_layout(Lay &L, u32 n, u32 E, u32 heur, u32 linked, u32 msps_warps,
                                            u32 grid = 0, u32 multi = 0) {
  u64 o = 0;
  auto take = [&](u64 words) -> u32 { u64 p = o; o = (o + words + 3) & ~3ull; return (u32)p; };
  const u64 n1 = (u64)n + 1, e1 = (u64)E + 1;
  L.n = n; L.E = E; L.heur = heur; L.linked = linked;
  L.track_nev = heur == H_DTR || uses_uf(heur) || uses_closure(heur);
  L.srec = take(4 * n1);
  L.arec = take(4 * n1);
  L.par = take(e1);
  L.ch = linked ? 0 : take(e1);
  L.state = take(n1);
  L.rho = take(n1);
  L.ell = take(n1);
  L.pool_words = (u32)((n1 + 31) / 32);
  L.pool_bm = take(L.pool_words);
  L.pool_ids = take(n1);
  L.pool_pos = take(n1);
  L.pool_key = (int_key_heur(heur) && !grid) ? take(2 * n1) : 0;
  L.fr = take(4 * n1);
  L.pb = take(e1);
  L.mem_next = L.comp = L.comp_head = L.bfs_q = L.stamp = 0;
  L.mem_prev = L.comp_free = 0;
  L.node_of = L.uf = L.uf_size = L.uf_cap = 0;
  L.msps_bm = L.msps_q = L.msps_words = L.msps_warps = L.msps_lock = L.msps_d = 0;
  L.e_next = L.e_child = 0;
  L.ccache = L.evq = 0;
  L.mirror = L.mo_off = L.mo_par = L.mo_ev = 0;
  L.lcache = 0;
  if (heur == H_DTR) {
    L.mem_next = take(n1);
    L.mem_prev = take(n1);
    L.comp_free = take(n1);
    L.comp = take(4 * n1);
    L.comp_head = take(n1);
    L.bfs_q = take(n1);
    L.stamp = take(n1);
  } else if (uses_uf(heur)) {
    L.uf_cap = 2 * n + 64;                             // compaction at most once per n + 64 evictions
    L.node_of = take(n1);
    L.uf = take(4 * (u64)L.uf_cap);
    L.uf_size = take(L.uf_cap);
    if (heur == H_DTR_EQ && !linked && multi) L.lcache = take(n1);
  } else if (uses_closure(heur)) {
    L.msps_warps = msps_warps;
    L.msps_words = (u32)((n1 + 31) / 32);
    L.msps_bm = take((u64)L.msps_words * msps_warps);
    L.msps_q = take(n1 * msps_warps);
    if (grid) L.msps_lock = take(msps_warps);
    if (multi && !linked) L.msps_d = take(n1 * msps_warps);
    if (!linked) {                                     // cached closure sums
      L.ccache = take(2 * n1);
      L.evq = take(EVQ_CAP);
    }
  }
  if (linked) {
    L.e_next = take(e1);
    L.e_child = take(e1);
  }
  L.words = (u32)o;
  return o < 0xFFFFFFF0ull;
}

// Closure-BFS scratch slots of the whole-GPU engine: each slot is a visited
// bitmap + queue of n + 1 words, so the slots are bounded to ~64 Mi words
// (256 MiB) in total; the lane-parallel walk needs no scratch and the BFS is
// only the fallback for frontiers wider than the lane heap.
__host__ __device__ inline u32 grid_closure_slots(u32 n) {
  const u64 per = 2 * ((u64)n + 1) + ((u64)n + 32) / 32;
  u64 k = (64ull << 20) / per;
  return k < 1 ? 1u : (k > 1024 ? 1024u : (u32)k);
}

// ---------------------------------------------------------------------------
// Memory policy: SM -> dynamic shared memory, else a global base pointer.
// ---------------------------------------------------------------------------
extern __shared__ __align__(16) u32 g_smem[];

// DTR_BOUNDS (tools/bounds_check.sh; the compute-sanitizer is not available on
// the GPU pool): every access is checked against the simulation's layout size
// `lim` (words) and traps with the offending offset.
#ifdef DTR_BOUNDS
#define DTR_CHECK(o, k)                                                                                    \
  do {                                                                                                     \
    if ((u64)(o) + (k) > (u64)lim) {                                                                       \
      printf("dtr bounds: block %d thread %d offset %u + %u > %u\n", (int)blockIdx.x, (int)threadIdx.x,  \
             (unsigned)(o), (unsigned)(k), (unsigned)lim);                                                 \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define DTR_CHECK(o, k)
#endif

template <bool SM>
struct Mem {
  u32 *gbase;
  u32 lim = 0xFFFFFFFFu;   // the layout's words (DTR_BOUNDS builds check every access against it)
  // SM = false: gbase is a global-memory pointer; telling the compiler so lets
  // it emit LDG/STG (global) instead of generic LD/ST
  __device__ __forceinline__ u32 &w(u32 off) const {
    DTR_CHECK(off, 1);
    if constexpr (SM) return g_smem[off];
    else { __builtin_assume(__isGlobal(gbase)); return gbase[off]; }
  }
  __device__ __forceinline__ uint4 &q(u32 off) const {   // off multiple of 4
    DTR_CHECK(off, 4);
    if constexpr (SM) return reinterpret_cast<uint4 *>(g_smem)[off >> 2];
    else { __builtin_assume(__isGlobal(gbase)); return reinterpret_cast<uint4 *>(gbase)[off >> 2]; }
  }
  __device__ __forceinline__ uint2 &d(u32 off) const {   // off multiple of 2
    DTR_CHECK(off, 2);
    if constexpr (SM) return reinterpret_cast<uint2 *>(g_smem)[off >> 1];
    else { __builtin_assume(__isGlobal(gbase)); return reinterpret_cast<uint2 *>(gbase)[off >> 1]; }
  }
};

// ---------------------------------------------------------------------------
// Scalars of one simulation (leader state; persisted in device memory between
// per-call launches).
// ---------------------------------------------------------------------------
struct Scalars {
  u64 clock, M, B, peak_M, base_so_far, decisions, remats, computations, trace_hash, trace_n;
  u64 max_decisions, seed, trace_cap, trace_off;   // max_decisions: 0 = none (stored as ~0, norm_scalars)
  u32 n_alloc;        // tensors created (MAKE started)
  u32 pool_size;
  u32 status;         // sticky run status
  u32 heuristic;
  u32 thrash_kill;
  u32 records_done;
  u32 sp, pb_top;     // explicit get_internal stack
  u32 uf_n;           // union-find nodes in use
  u32 epoch;          // BFS stamps
  u32 edges_used;     // linked children (per-call mode)
  u32 cell_id;
  u32 last_rc;        // per-call: result code of the last op
  u32 pending_op;     // per-call: the op word being applied
  u32 n_scores;       // per-call OP_SCORES: pool size scored
  u32 dealloc;        // DEALLOC_*: what release does at rho = 0 (reading C-22)
  u32 comp_top;       // h_DTR: free label slots on the stack
  u32 comp_fresh;     // h_DTR: label slots never used yet
  u32 ev_n;           // closure cache: events queued since the last score pass (EVQ_CAP + 1 = overflow)
  u64 kill_limit;     // min(thrash_kill * base_so_far, CLOCK_LIMIT) (recomputed at every MAKE; kill 0 = off)
};

// leader-side encodings of the configuration: no decision cap = ~0, and the
// clock stop threshold before the first MAKE = CLOCK_LIMIT
__host__ __device__ __forceinline__ void norm_scalars(Scalars &s) {
  if (s.max_decisions == 0) s.max_decisions = ~0ull;
  s.kill_limit = CLOCK_LIMIT;
}

// ---------------------------------------------------------------------------
// Exact rational scores.  den == 0 encodes +infinity.
// ---------------------------------------------------------------------------
struct Cand {
  u64 num, den;
  u32 id;
};

// a.num * b.den < b.num * a.den, exactly.  Numerators are < 2^32 for every
// heuristic but h_random (whose den is 1): then each product is a 32 x 64-bit
// product compared as (high 64, low 32); else full 128-bit products.
__device__ __forceinline__ bool score_less(const Cand &a, const Cand &b) {
  if (((a.num | b.num) >> 32) == 0) {
    const u32 an = (u32)a.num, bn = (u32)b.num;
    const u64 l0 = (u64)an * (u32)b.den, l1 = (u64)an * (u32)(b.den >> 32);
    const u64 r0 = (u64)bn * (u32)a.den, r1 = (u64)bn * (u32)(a.den >> 32);
    const u64 lh = l1 + (l0 >> 32), rh = r1 + (r0 >> 32);
    if (lh != rh) return lh < rh;
    return (u32)l0 < (u32)r0;
  }
  return (u128)a.num * b.den < (u128)b.num * a.den;
}

__device__ __forceinline__ bool score_eq(const Cand &a, const Cand &b) {
  return !score_less(a, b) && !score_less(b, a);
}

// lexicographic (score, id): equal scores -> smaller id (reading C-5)
__device__ __forceinline__ bool cand_less(const Cand &a, const Cand &b) {
  if (a.num == b.num && a.den == b.den) return a.id < b.id;   // identical rationals (common: size, LRU)
  if (score_less(a, b)) return true;
  if (score_less(b, a)) return false;
  return a.id < b.id;
}

__device__ __forceinline__ Cand cand_none() { Cand c; c.num = 1; c.den = 0; c.id = NONE; return c; }

__device__ __forceinline__ u64 splitmix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// num / (mem * (clock - L)), la encoded as clock + 1 (0 = -inf).
//   L = -inf  -> 0           (V2 zero, reading C-4)
//   clock = L -> +inf        (reading C-3)
__device__ __forceinline__ void stale_score(u64 num, u32 mem, u32 L_enc, u64 clock, u64 &on, u64 &od) {
  if (L_enc == 0) { on = 0; od = 1; return; }
  u64 s = clock + 1 - (u64)L_enc;
  if (s == 0) { on = 1; od = 0; return; }
  on = num; od = (u64)mem * s;
}

__device__ __forceinline__ u64 mk64(u32 lo, u32 hi) { return (u64)lo | ((u64)hi << 32); }

// ---------------------------------------------------------------------------
// Graph access shared by the leader and the team.
// ---------------------------------------------------------------------------
template <bool SM>
struct Sim {
  Mem<SM> m;
  Lay L;

  __device__ __forceinline__ uint4 &srec(u32 t) const { return m.q(L.srec + 4 * t); }     // {mem, cost, la, nev}
  __device__ __forceinline__ u32 &la(u32 t) const { return m.w(L.srec + 4 * t + 2); }
  __device__ __forceinline__ u32 &nev(u32 t) const { return m.w(L.srec + 4 * t + 3); }
  __device__ __forceinline__ uint4 &arec(u32 t) const { return m.q(L.arec + 4 * t); }     // {par_off, npar, ch_off, nch}
  __device__ __forceinline__ uint2 &prec(u32 t) const { return m.d(L.arec + 4 * t); }     // {par_off, npar}
  __device__ __forceinline__ uint2 &crec(u32 t) const { return m.d(L.arec + 4 * t + 2); } // {ch_off, nch} | {head, -}
  __device__ __forceinline__ u32 &state(u32 t) const { return m.w(L.state + t); }
  __device__ __forceinline__ u32 &rho(u32 t) const { return m.w(L.rho + t); }
  __device__ __forceinline__ u32 &ell(u32 t) const { return m.w(L.ell + t); }
  __device__ __forceinline__ u32 &par(u32 j) const { return m.w(L.par + j); }
  __device__ __forceinline__ u32 &pool_word(u32 w) const { return m.w(L.pool_bm + w); }
  __device__ __forceinline__ bool in_pool(u32 t) const { return (pool_word(t >> 5) >> (t & 31)) & 1u; }
  __device__ __forceinline__ u32 &pool_ids(u32 i) const { return m.w(L.pool_ids + i); }
  __device__ __forceinline__ u32 &pool_pos(u32 t) const { return m.w(L.pool_pos + t); }
  __device__ __forceinline__ uint4 &comp(u32 c) const { return m.q(L.comp + 4 * c); }
  __device__ __forceinline__ uint4 &uf(u32 x) const { return m.q(L.uf + 4 * x); }
  __device__ __forceinline__ uint2 &ccache(u32 t) const { return m.d(L.ccache + 2 * t); }   // {up+1, down+1}

  // parents of t then children (ar = arec(t) already loaded; linked lists are
  // re-read from the live head)
  template <class F>
  __device__ __forceinline__ void for_each_nbr(u32 t, const uint4 &ar, F f) const {
    for (u32 j = 0; j < ar.y; j++) f(par(ar.x + j));
    if (!L.linked) {
      for (u32 j = 0; j < ar.w; j++) f(m.w(L.ch + ar.z + j));
    } else {
      for (u32 e = crec(t).x; e != NONE; e = m.w(L.e_next + e)) f(m.w(L.e_child + e));
    }
  }

  // closure-walk accessors: the shared-memory mirror when present, else the state
  __device__ __forceinline__ bool wev(u32 x) const {          // is_evicted(state(x))
    if (L.mirror) return (reinterpret_cast<const u32 *>(reinterpret_cast<const char *>(g_smem) + L.mo_ev)[x >> 5] >> (x & 31)) & 1u;
    return is_evicted(state(x));
  }
  __device__ __forceinline__ uint2 wprec(u32 x) const {       // {par_off, npar}
    if (L.mirror) {
      const unsigned short *o = reinterpret_cast<const unsigned short *>(reinterpret_cast<const char *>(g_smem) + L.mo_off);
      const u32 a = o[x], b = o[x + 1];
      return make_uint2(a, b - a);
    }
    return prec(x);
  }
  __device__ __forceinline__ u32 wpar(u32 j) const {
    if (L.mirror) return reinterpret_cast<const unsigned short *>(reinterpret_cast<const char *>(g_smem) + L.mo_par)[j];
    return par(j);
  }
  __device__ __forceinline__ void mirror_bit(u32 x, bool ev) const {   // leader: x's evicted status flipped
    if (!L.mirror) return;
    u32 *w = reinterpret_cast<u32 *>(reinterpret_cast<char *>(g_smem) + L.mo_ev) + (x >> 5);
    if (ev) *w |= 1u << (x & 31);
    else *w &= ~(1u << (x & 31));
  }

  // union-find find without compression (read-only: safe inside the parallel score pass)
  __device__ __forceinline__ u32 uf_root(u32 x, u32 &steps) const {
    u32 p = uf(x).w;
    while (p != x) { x = p; p = uf(x).w; steps++; }
    return x;
  }
};

}  // namespace dtr
