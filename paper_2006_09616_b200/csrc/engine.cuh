// engine.cuh -- device side of the DTR eviction-decision engine (sm_100a).
//
// One simulation = the simrd runtime with V2 banishing (PAPER.md Doc A,
// P:113-373).  Its control (make_tensor / get_internal recursion /
// release_internal / free / evict) is inherently sequential and runs
// on ONE leader thread as a resumable state machine with an explicit stack;
// whenever free() needs a decision the leader hands the pool to its
// TEAM -- a whole CTA (many small simulations per GPU, one per CTA) or the whole
// grid (one large simulation per GPU) -- which scores every pool member and
// reduces the exact (score, id) argmin.  All state lives in device memory.
//
// Independent of oracle/ (shares no code with it).
#pragma once
#include <stdint.h>
#include <cooperative_groups.h>

namespace dtr {

typedef uint32_t u32;
typedef unsigned long long u64;
typedef unsigned __int128 u128;

constexpr u32 NONE = 0xFFFFFFFFu;
// state word per tensor: bit31 material (t.m = T), bit30 computed at least
// once (reading C-19), bits 0..29: evicted-component id (h_DTR exact mode).
constexpr u32 M_BIT = 1u << 31;
constexpr u32 O_BIT = 1u << 30;
constexpr u32 COMP_MASK = (1u << 30) - 1;
constexpr u64 CLOCK_LIMIT = 0xFFFFFFFEull;   // reading C-14: la is stored as clock + 1 in u32

enum { H_DTR = 0, H_DTR_EQ = 1, H_LRU = 2, H_SIZE = 3, H_MSPS = 4, H_LOCAL = 5, H_RANDOM = 6 };
enum { OP_MAKE = 1, OP_GET = 2, OP_RELEASE = 3, OP_REMAT = 4, OP_ENSURE = 5, OP_DEBUG_EVICT = 6,
       OP_SCORES = 7 /* per-call only: score the whole pool */ };
enum { ST_OK = 0, ST_INVAL = 1, ST_PRECOND = 2, ST_OOM = 3, ST_THRASH = 4, ST_CAPACITY = 5,
       ST_STATE = 6, ST_DECISION_CAP = 8 };

__host__ __device__ inline bool is_evicted(u32 s) { return (s & (M_BIT | O_BIT)) == O_BIT; }
__host__ __device__ inline bool is_material(u32 s) { return (s & M_BIT) != 0; }
__host__ __device__ inline u64 align16(u64 x) { return (x + 15) & ~15ull; }

// ---------------------------------------------------------------------------
// Scalars of one simulation (leader state; persisted in device memory between
// per-call launches).
// ---------------------------------------------------------------------------
struct Scalars {
  u64 clock, M, B, peak_M, base_so_far, decisions, remats, computations, trace_hash, trace_n;
  u64 max_decisions, seed, trace_cap, trace_off;
  u32 n_alloc;        // tensors created (MAKE started)
  u32 pool_size;
  u32 status;         // sticky run status
  u32 heuristic;
  u32 thrash_kill;
  u32 records_done;
  u32 sp, pb_top;     // explicit get_internal stack
  u32 comp_free_top;  // exact components: free-id stack
  u32 uf_n, uf_cap;   // union-find nodes in use / capacity
  u32 epoch;
  u32 edges_used;     // linked children (per-call mode)
  u32 cell_id;
  u32 last_rc;        // per-call: result code of the last op
  u32 pending_op;     // per-call: the op word being applied
  u32 n_scores;       // per-call OP_SCORES: pool size scored
  u32 pad[3];
};

// ---------------------------------------------------------------------------
// Read-only graph of a log: tensor table + parents CSR (from the log) and the
// children lists built on the device.
// ---------------------------------------------------------------------------
struct Graph {
  u32 n, E, nops;
  const u32 *mem, *cost, *par_off, *par, *ops;
  u64 base;
  // children: CSR (batch) or linked lists (per-call)
  u32 linked;
  u32 *ch_off, *ch;                     // CSR: ch[ch_off[p] .. ch_off[p+1])
  u32 *ch_head, *e_next, *e_child;      // linked: e = ch_head[p]; e != NONE; e = e_next[e]
};

__host__ __device__ inline void graph_from_log(Graph &g, const u32 *w) {
  g.n = w[2]; g.E = w[3]; g.nops = w[4];
  g.base = (u64)w[6] | ((u64)w[7] << 32);
  g.mem = w + 16;
  g.cost = g.mem + g.n;
  g.par_off = g.cost + g.n;
  g.par = g.par_off + g.n + 1;
  g.ops = g.par + g.E;
  g.linked = 0;
}

// ---------------------------------------------------------------------------
// Per-simulation mutable state (structure of arrays in device memory).
// ---------------------------------------------------------------------------
struct Work {
  Scalars *sc;
  u32 *state, *la, *rho, *ell, *pool_ids, *pool_pos;
  u32 *fr_t, *fr_base, *fr_cnt, *fr_next, *pb;
  // exact evicted components (h_DTR)
  u64 *comp_cost;
  u32 *comp_maxla, *comp_head, *comp_size, *mem_next, *comp_free, *bfs_q, *stamp;
  // union-find (h_DTR_eq)
  u32 *node_of, *uf_parent, *uf_maxla, *uf_size, *uf_remap, *uf_roots, *uf_tmaxla, *uf_tsize;
  u64 *uf_cost, *uf_tcost;
  // children CSR scratch (batch) / linked lists (per-call)
  u32 *ch_off, *ch, *ch_fill;
  u32 *ch_head, *e_next, *e_child;
  // MSPS per-warp scratch
  u32 *msps_bm, *msps_q;
  u32 msps_words;
};

// Carve the workspace of one simulation.  Same function sizes it on the host
// (base = 0) and places it on the device.  Arrays unused by the heuristic get
// no space.
__host__ __device__ inline u64 carve(Work &w, uintptr_t base, u32 n, u32 E, u32 heur, u32 linked,
                                      u32 msps_warps) {
  u64 off = 0;
  auto take = [&](u64 bytes) -> uintptr_t { uintptr_t p = base + off; off = align16(off + bytes); return p; };
  u64 n1 = (u64)n + 1;
  w.sc = (Scalars *)take(sizeof(Scalars));
  w.state = (u32 *)take(4 * n1);
  w.la = (u32 *)take(4 * n1);
  w.rho = (u32 *)take(4 * n1);
  w.ell = (u32 *)take(4 * n1);
  w.pool_ids = (u32 *)take(4 * n1);
  w.pool_pos = (u32 *)take(4 * n1);
  w.fr_t = (u32 *)take(4 * n1);
  w.fr_base = (u32 *)take(4 * n1);
  w.fr_cnt = (u32 *)take(4 * n1);
  w.fr_next = (u32 *)take(4 * n1);
  w.pb = (u32 *)take(4 * ((u64)E + 1));
  w.comp_cost = nullptr; w.comp_maxla = w.comp_head = w.comp_size = w.mem_next = w.comp_free = nullptr;
  w.bfs_q = w.stamp = nullptr;
  if (heur == H_DTR) {
    w.comp_cost = (u64 *)take(8 * n1);
    w.comp_maxla = (u32 *)take(4 * n1);
    w.comp_head = (u32 *)take(4 * n1);
    w.comp_size = (u32 *)take(4 * n1);
    w.mem_next = (u32 *)take(4 * n1);
    w.comp_free = (u32 *)take(4 * n1);
    w.bfs_q = (u32 *)take(4 * n1);
    w.stamp = (u32 *)take(4 * n1);
  }
  w.node_of = w.uf_parent = w.uf_maxla = w.uf_size = w.uf_remap = w.uf_roots = w.uf_tmaxla = w.uf_tsize = nullptr;
  w.uf_cost = w.uf_tcost = nullptr;
  if (heur == H_DTR_EQ) {
    u64 cap = 2 * (u64)n + 64;
    w.node_of = (u32 *)take(4 * n1);
    w.uf_parent = (u32 *)take(4 * cap);
    w.uf_maxla = (u32 *)take(4 * cap);
    w.uf_size = (u32 *)take(4 * cap);
    w.uf_remap = (u32 *)take(4 * cap);
    w.uf_roots = (u32 *)take(4 * cap);
    w.uf_tmaxla = (u32 *)take(4 * cap);
    w.uf_tsize = (u32 *)take(4 * cap);
    w.uf_cost = (u64 *)take(8 * cap);
    w.uf_tcost = (u64 *)take(8 * cap);
  }
  w.msps_bm = w.msps_q = nullptr;
  w.msps_words = 0;
  if (heur == H_MSPS) {
    // MSPS closure scratch, one per scoring warp: visited bitmap + BFS queue
    w.msps_words = (u32)((n1 + 31) / 32);
    w.msps_bm = (u32 *)take(4 * (u64)w.msps_words * msps_warps);
    w.msps_q = (u32 *)take(4 * n1 * msps_warps);
  }
  w.ch_off = w.ch = w.ch_fill = w.ch_head = w.e_next = w.e_child = nullptr;
  if (!linked) {
    w.ch_off = (u32 *)take(4 * (n1 + 1));
    w.ch = (u32 *)take(4 * ((u64)E + 1));
    w.ch_fill = (u32 *)take(4 * n1);
  } else {
    w.ch_head = (u32 *)take(4 * n1);
    w.e_next = (u32 *)take(4 * ((u64)E + 1));
    w.e_child = (u32 *)take(4 * ((u64)E + 1));
  }
  return off;
}

// ---------------------------------------------------------------------------
// Exact rational scores.  den == 0 encodes +infinity.
// ---------------------------------------------------------------------------
struct Cand {
  u64 num, den;
  u32 id;
};

__device__ __forceinline__ bool cand_less(const Cand &a, const Cand &b) {
  u128 l = (u128)a.num * b.den, r = (u128)b.num * a.den;
  if (l != r) return l < r;
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

// ---------------------------------------------------------------------------
// Neighbour iteration: parents (log CSR) then visible children.
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void for_each_nbr(const Graph &g, u32 t, F f) {
  u32 b = __ldg(&g.par_off[t]), e = __ldg(&g.par_off[t + 1]);
  for (u32 j = b; j < e; j++) f(__ldg(&g.par[j]));
  if (!g.linked) {
    u32 cb = g.ch_off[t], ce = g.ch_off[t + 1];
    for (u32 j = cb; j < ce; j++) f(g.ch[j]);
  } else {
    for (u32 x = g.ch_head[t]; x != NONE; x = g.e_next[x]) f(g.e_child[x]);
  }
}

// union-find find without compression (read-only: used inside the parallel score pass)
__device__ __forceinline__ u32 uf_find_ro(const u32 *parent, u32 x) {
  u32 p = parent[x];
  while (p != x) { x = p; p = parent[x]; }
  return x;
}

// Sum of component costs over DISTINCT evicted components adjacent to t and the
// max of their la (h_DTR: exact labels; h_DTR_eq: UF roots).  Dedup: the last
// four distinct ids are kept in registers; beyond that an earlier-neighbour
// rescan decides.
// Algorithmic bytes: each neighbour costs its id + state
// word (8 B); each distinct component its cost + maxla (12 B); h_DTR_eq adds
// node_of (4 B) per evicted neighbour and 4 B per union-find parent step.
template <bool UF>
__device__ __forceinline__ void nbr_components(const Graph &g, const Work &w, u32 t, u64 &sum, u32 &L,
                                               u64 &bytes) {
  u32 c0 = NONE, c1 = NONE, c2 = NONE, c3 = NONE, nd = 0;
  u32 nb = 0, extra = 0;
  auto comp_of = [&](u32 q, u32 sq) -> u32 {
    if (UF) {
      u32 x = w.node_of[q], p = w.uf_parent[x];
      extra += 8;
      while (p != x) { x = p; p = w.uf_parent[x]; extra += 4; }
      return x;
    }
    return sq & COMP_MASK;
  };
  auto seen_earlier = [&](u32 upto_q_pos, u32 c) -> bool {
    // rescan neighbours at positions < upto_q_pos
    u32 pos = 0; bool found = false;
    for_each_nbr(g, t, [&](u32 y) {
      if (found || pos >= upto_q_pos) { pos++; return; }
      pos++;
      u32 sy = w.state[y];
      if (is_evicted(sy) && comp_of(y, sy) == c) found = true;
    });
    return found;
  };
  u32 pos = 0;
  for_each_nbr(g, t, [&](u32 q) {
    u32 my = pos++;
    nb++;
    u32 sq = w.state[q];
    if (!is_evicted(sq)) return;
    u32 c = comp_of(q, sq);
    if (c == c0 || c == c1 || c == c2 || c == c3) return;
    if (nd >= 4 && seen_earlier(my, c)) return;
    nd++;
    c3 = c2; c2 = c1; c1 = c0; c0 = c;
    if (UF) { sum += w.uf_cost[c]; u32 m = w.uf_maxla[c]; L = m > L ? m : L; }
    else { sum += w.comp_cost[c]; u32 m = w.comp_maxla[c]; L = m > L ? m : L; }
  });
  bytes += 8ull * nb + 12ull * nd + extra;
}

// score of one pool member (MSPS handled separately: it needs per-candidate scratch)
// bytes: algorithmic bytes this candidate's score reads, pool id included.
__device__ __forceinline__ void score_one(const Graph &g, const Work &w, u32 heur, u64 clock, u64 seed,
                                          u64 decisions, u32 t, u64 &num, u64 &den, u64 &bytes) {
  switch (heur) {
    case H_DTR: {
      u64 sum = 0; u32 L = w.la[t];
      nbr_components<false>(g, w, t, sum, L, bytes);
      stale_score((u64)__ldg(&g.cost[t]) + sum, __ldg(&g.mem[t]), L, clock, num, den);
      bytes += 4 + 12 + 16;   // pool id; mem, cost, la; parent + child CSR offsets
      return;
    }
    case H_DTR_EQ: {
      u64 sum = 0; u32 L = w.la[t];
      nbr_components<true>(g, w, t, sum, L, bytes);
      stale_score((u64)__ldg(&g.cost[t]) + sum, __ldg(&g.mem[t]), L, clock, num, den);
      bytes += 4 + 12 + 16;
      return;
    }
    case H_LRU:
      stale_score(1, 1, w.la[t], clock, num, den);
      bytes += 8;
      return;
    case H_SIZE:
      num = 1; den = __ldg(&g.mem[t]);
      bytes += 8;
      return;
    case H_LOCAL:
      stale_score((u64)__ldg(&g.cost[t]), __ldg(&g.mem[t]), w.la[t], clock, num, den);
      bytes += 16;
      return;
    case H_RANDOM:
      num = splitmix64(seed ^ (decisions << 32) ^ (u64)t); den = 1;
      bytes += 4;
      return;
  }
  num = 0; den = 1;
}

// ---------------------------------------------------------------------------
// Reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ Cand warp_argmin(Cand c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand d;
    d.num = __shfl_xor_sync(0xffffffffu, c.num, o);
    d.den = __shfl_xor_sync(0xffffffffu, c.den, o);
    d.id = __shfl_xor_sync(0xffffffffu, c.id, o);
    if (cand_less(d, c)) c = d;
  }
  return c;
}

struct RedSmem {
  Cand warp[32];
};

// block-wide argmin; the result is valid in warp 0 (all lanes) after return.
__device__ __forceinline__ Cand block_argmin(Cand c, RedSmem &sm) {
  c = warp_argmin(c);
  u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) sm.warp[wid] = c;
  __syncthreads();
  if (wid == 0) {
    c = lane < nw ? sm.warp[lane] : cand_none();
    c = warp_argmin(c);
  }
  return c;
}

}  // namespace dtr
