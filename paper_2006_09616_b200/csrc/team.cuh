// team.cuh -- K3 (score pass) + K4 (argmin) + K5 (MSPS closure) of one
// eviction decision, run by a whole team (CTA or grid) over the pool.
//
// score(t) per heuristic (exact rationals, den == 0 = +inf):
//   h_DTR     (c0(t) + sum over the DISTINCT evicted components adjacent to t of
//              their cost) / (m(t) * (clock - max(la(t), their max la)))
//   h_DTR_eq  same with union-find roots (no unions while querying)
//   h_LRU     1 / s(t)
//   h_size    1 / m(t)
//   h_MSPS    (c0(t) + sum_{e_R(t)} c0) / m(t)
//   h_local   c0(t) / (m(t) s(t))
//   h_random  splitmix64(seed ^ decision << 32 ^ t)                        P:1269 (C-15)
// A candidate whose evicted-neighbour count nev is 0 has E(t) = e*(t) = e_R(t)
// = {} and is scored from its 16-B score record {mem, cost, la, nev} alone;
// only candidates with nev > 0 walk their neighbour lists.
// Algorithmic bytes are counted as they are read: the
// pool bitmap (1 bit per tensor id), per candidate its own fields (h_DTR,
// h_DTR_eq, closures: score record 16; LRU la 4; size mem 4; local 12; random
// 4), and when nev > 0: the adjacency record 16, then 8 per neighbour (id +
// state word), 12 per distinct component (cost + max la), h_DTR_eq +4 per
// evicted neighbour (node id) and +4 per union-find step; MSPS +8 per parent
// examined, +16 per closure member.
#pragma once
#include "engine.cuh"
#include "leader.cuh"
#include <cooperative_groups.h>

namespace dtr {

namespace cg = cooperative_groups;

// Distinct adjacent evicted components: the last four labels are kept in
// registers; beyond four an earlier-neighbour rescan decides duplicates.
template <bool SM, bool UF>
__device__ __forceinline__ void nbr_components(const Sim<SM> &g, u32 t, const uint4 &ar, u64 &sum, u32 &L,
                                               u64 &bytes) {
  u32 c0 = NONE, c1 = NONE, c2 = NONE, c3 = NONE, nd = 0, nb = 0, extra = 0;
  auto comp_of = [&](u32 q, u32 sq, u32 &steps) -> u32 {
    if constexpr (UF) return g.uf_root(g.m.w(g.L.node_of + q), steps);
    else return sq & COMP_MASK;
  };
  u32 pos = 0;
  g.for_each_nbr(t, ar, [&](u32 q) {
    const u32 my = pos++;
    nb++;
    const u32 sq = g.state(q);
    if (!is_evicted(sq)) return;
    u32 steps = 0;
    const u32 c = comp_of(q, sq, steps);
    if constexpr (UF) extra += 4 + 4 * steps;
    if (c == c0 || c == c1 || c == c2 || c == c3) return;
    if (nd >= 4) {
      u32 p2 = 0;
      bool dup = false;
      g.for_each_nbr(t, ar, [&](u32 y) {
        if (dup || p2 >= my) { p2++; return; }
        p2++;
        u32 sy = g.state(y), st2 = 0;
        if (is_evicted(sy) && comp_of(y, sy, st2) == c) dup = true;
      });
      if (dup) return;
    }
    nd++;
    c3 = c2; c2 = c1; c1 = c0; c0 = c;
    uint4 cr = UF ? g.uf(c) : g.comp(c);
    sum += UF ? mk64(cr.x, cr.y) : (u64)cr.x;   // exact comp record {cost, nmax, maxla, size}
    L = cr.z > L ? cr.z : L;
  });
  bytes += 8ull * nb + 12ull * nd + extra;
}

// K5: warp-cooperative closures.  e_R(t) -- evicted ancestors reached through
// evicted parents (h_MSPS); with DOWN also the evicted descendants
// reached through evicted children, i.e. the directed e*(t) of P:2244-2258
// (h_DTR_full, h_e*).  Ancestors and descendants of t are disjoint in a DAG,
// so one per-warp visited bitmap + queue serves both passes; the sum of their
// c0 is returned in every lane.
template <bool SM>
__device__ u64 msps_closure(const Sim<SM> &g, const uint4 &ar, u32 wslot, volatile u32 *tail, u64 &bytes,
                            u32 t = NONE, bool down = false, u64 *up_out = nullptr) {
  const u32 lane = threadIdx.x & 31;
  const u32 bm = g.L.msps_bm + wslot * g.L.msps_words;
  const u32 q = g.L.msps_q + wslot * (g.L.n + 1);
  if (lane == 0) *tail = 0;
  __syncwarp();
  u64 sum = 0;
  auto visit = [&](u32 p) {
    bytes += 8;   // parent id + its state word
    if (!g.wev(p)) return;
    u32 bit = 1u << (p & 31);
    u32 old = atomicOr(&g.m.w(bm + (p >> 5)), bit);
    if (old & bit) return;
    bytes += 16;  // its score record
    sum += g.srec(p).y;
    u32 pos = atomicAdd((u32 *)tail, 1u);
    g.m.w(q + pos) = p;
  };
  for (u32 j = lane; j < ar.y; j += 32) visit(g.wpar(ar.x + j));
  __syncwarp();
  u32 head = 0, tl = *tail;
  __syncwarp();
  while (head < tl) {
    for (u32 i = head + lane; i < tl; i += 32) {
      u32 x = g.m.w(q + i);
      const uint2 px = g.wprec(x);
      for (u32 j = 0; j < px.y; j++) visit(g.wpar(px.x + j));
    }
    __syncwarp();
    head = tl;
    tl = *tail;
    __syncwarp();
  }
  u64 up = sum;
  if (down) {                                   // evicted descendants through evicted children
    auto children = [&](u32 x) {
      const uint2 cr = g.crec(x);
      bytes += 8;
      if (!g.L.linked) { for (u32 j = 0; j < cr.y; j++) visit(g.m.w(g.L.ch + cr.x + j)); }
      else { for (u32 e = cr.x; e != NONE; e = g.m.w(g.L.e_next + e)) visit(g.m.w(g.L.e_child + e)); }
    };
    if (lane == 0) children(t);
    __syncwarp();
    tl = *tail;
    __syncwarp();
    while (head < tl) {
      for (u32 i = head + lane; i < tl; i += 32) children(g.m.w(q + i));
      __syncwarp();
      head = tl;
      tl = *tail;
      __syncwarp();
    }
  }
  for (u32 i = lane; i < tl; i += 32) g.m.w(bm + (g.m.w(q + i) >> 5)) = 0;
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    up += __shfl_xor_sync(0xffffffffu, up, o);
  }
  if (up_out) *up_out = up;
  return sum;
}

// Closure-cache invalidation (App. C "Caching metadata"), run by
// ONE warp before a score pass over the events the leader queued since the
// last one (tensors whose evicted status flipped).  A flip of x can change
// e_R(t) only for the non-evicted t reached from x downwards through evicted
// tensors (the flipped tensor on the changed path closest to t sees only
// evicted tensors between itself and t, in the current state), and the
// descendant half of e*(t) only for the non-evicted t reached upwards; those
// caches (and x's own) are marked stale.  Walks use the current state, so the
// order of the events does not matter, and all events are walked as ONE
// multi-source search per direction (overlapping regions once).  Scratch:
// closure slot `slot`.
template <bool SM>
__device__ void closure_events(const Sim<SM> &g, const Cmd &cmd, u32 slot, volatile u32 *tail) {
  if (!g.L.ccache || cmd.n_ev == 0 || cmd.n_ev == NONE) return;
  const u32 lane = threadIdx.x & 31;
  const bool down = cmd.heur != H_MSPS;
  if (cmd.n_ev > EVQ_CAP) {                      // overflow: every cache is stale
    for (u32 t = lane; t < cmd.n_ids; t += 32) g.ccache(t) = make_uint2(0, 0);
    __syncwarp();
    return;
  }
  const u32 bm = g.L.msps_bm + slot * g.L.msps_words;
  const u32 q = g.L.msps_q + slot * (g.L.n + 1);
  PROF_T(ce0);
  // f = 0: ancestor caches (.x) of the tensors below; f = 1: descendant caches (.y) above
  auto visit = [&](u32 y, u32 f) {
    if (!g.wev(y)) { g.m.w(g.L.ccache + 2 * y + f) = 0; return; }
    const u32 bit = 1u << (y & 31);
    if (atomicOr(&g.m.w(bm + (y >> 5)), bit) & bit) return;
    g.m.w(q + atomicAdd((u32 *)tail, 1u)) = y;
  };
  auto step = [&](u32 y, u32 f) {                // the evicted-side neighbours of y in direction f
    if (f == 0) {
      const uint2 cr = g.crec(y);
      for (u32 j = 0; j < cr.y; j++) visit(g.m.w(g.L.ch + cr.x + j), 0);
    } else {
      const uint2 pr = g.wprec(y);
      for (u32 j = 0; j < pr.y; j++) visit(g.wpar(pr.x + j), 1);
    }
  };
  u32 nodes = 0;
  for (u32 f = 0; f < (down ? 2u : 1u); f++) {
    if (lane == 0) *tail = 0;
    __syncwarp();
    for (u32 e = lane; e < cmd.n_ev; e += 32) {  // every event is a source
      const u32 x = g.m.w(g.L.evq + e);
      if (f == 0) g.ccache(x) = make_uint2(0, 0);
      step(x, f);
    }
    __syncwarp();
    u32 head = 0, tl = *tail;
    __syncwarp();
    while (head < tl) {
      for (u32 i = head + lane; i < tl; i += 32) step(g.m.w(q + i), f);
      __syncwarp();
      head = tl;
      tl = *tail;
      __syncwarp();
    }
    for (u32 i = lane; i < tl; i += 32) g.m.w(bm + (g.m.w(q + i) >> 5)) = 0;   // fresh visited set per direction
    __syncwarp();
    nodes += tl;
  }
  PROF_T(ce1);
  if (lane == 0) { PROF_ADD(19, cmd.n_ev); PROF_ADD(20, nodes); PROF_ADD(21, ce1 - ce0); }
}

// K5, up to 32 candidates at once (one per lane; NONE = idle lane): ONE walk
// over the union of their closures, each node carrying the 32-bit mask of the
// candidates whose closure it is in (closure sets overlap heavily on these
// graphs: every candidate below an evicted trunk shares it).  visit(y, m): y
// joins the closures of the candidates in m it was not yet in (atomicOr on its
// mask word); each newly set bit adds c(y) to that candidate's sum, and y is
// queued to pass the new bits on -- a node is re-queued only when new bits
// reach it, so it is expanded at most once per arrival wave, never per
// candidate.  Up: through evicted parents (e_R); down (the e*
// family): through evicted children.  Scratch: the slot's mask
// array (zero on entry and exit) and queue; sums: st.msum.  Returns false
// (warp-uniform) when the queue overflows (the caller walks per lane instead).
template <bool SM>
__device__ bool closure_multi(const Sim<SM> &g, u32 t, u32 slot, volatile u32 *tail, u64 *msum, bool down, u64 &up,
                              u64 &dn, u64 &bytes) {
  const u32 lane = threadIdx.x & 31;
  const u32 n1 = g.L.n + 1;
  const u32 D = g.L.msps_d + slot * n1, q = g.L.msps_q + slot * n1;
  bool ovf = false;
  auto walk = [&](bool dn_dir) -> u64 {
    msum[lane] = 0;
    if (lane == 0) *tail = 0;
    __syncwarp();
    auto visit = [&](u32 y, u32 m) {
      bytes += 8;                                  // neighbour id + its state word
      if (!g.wev(y)) return;
      const u32 old = atomicOr(&g.m.w(D + y), m);
      const u32 nb = m & ~old;
      if (!nb) return;
      if (!old) bytes += 16;                       // its score record (first arrival)
      const u64 c = g.srec(y).y;
      for (u32 b = nb; b; b &= b - 1) atomicAdd(&msum[__ffs(b) - 1], c);
      const u32 pos = atomicAdd((u32 *)tail, 1u);
      if (pos < n1) g.m.w(q + pos) = y;
    };
    auto expand = [&](u32 x, u32 m) {
      if (!dn_dir) {
        const uint2 pr = g.wprec(x);
        for (u32 j = 0; j < pr.y; j++) visit(g.wpar(pr.x + j), m);
      } else {
        const uint2 cr = g.crec(x);
        bytes += 8;
        for (u32 j = 0; j < cr.y; j++) visit(g.m.w(g.L.ch + cr.x + j), m);
      }
    };
    if (t != NONE) expand(t, 1u << lane);
    __syncwarp();
    u32 head = 0, tl = *tail;
    __syncwarp();
    while (head < tl && tl <= n1) {
      for (u32 i = head + lane; i < tl; i += 32) {
        const u32 x = g.m.w(q + i);
        expand(x, atomicOr(&g.m.w(D + x), 0u));    // the mask as it stands (later bits re-queue x)
      }
      __syncwarp();
      head = tl;
      tl = *tail;
      __syncwarp();
    }
    if (tl > n1) {                                 // overflow: some marked nodes were not queued
      ovf = true;
      for (u32 y = lane; y < g.L.n; y += 32) g.m.w(D + y) = 0;
    } else {
      for (u32 i = lane; i < tl; i += 32) g.m.w(D + g.m.w(q + i)) = 0;
    }
    __syncwarp();
    const u64 r = msum[lane];
    __syncwarp();
    return r;
  };
  up = walk(false);
  dn = 0;
  if (down && !ovf) dn = walk(true);
  return !ovf;
}

// K5 closures of ONE candidate per lane (lane-parallel).  UP: e_R(t), the
// evicted ancestors reached through evicted parents (h_MSPS), walked in
// DECREASING id order through a small max-heap of ids; DOWN: the evicted
// descendants reached through evicted children (the other half of the
// directed e*(t)), in INCREASING id order through a min-heap.  Parents precede
// children in id order (the log is topologically ordered), so after x is
// popped every later pop lies beyond x and all copies of an id pop
// consecutively: duplicates are dropped by comparing with the last pop, and no
// visited set is needed.  Returns false when the frontier outgrows the heap
// (the caller then runs the warp BFS, msps_closure).  Bytes as in
// msps_closure: 8 per neighbour examined (+8 per children record), 16 per
// closure member.
constexpr u32 MSPS_HEAP = 24;

template <bool SM, bool DOWN>
__device__ __forceinline__ bool closure_lane(const Sim<SM> &g, u32 t, const uint4 &ar, u64 &sum, u64 &bytes) {
  u32 heap[MSPS_HEAP];
  u32 hn = 0;
  u64 b = 0, s = 0;
  auto before = [](u32 a, u32 c) { return DOWN ? a < c : a > c; };   // heap order: first out
  auto push = [&](u32 x) -> bool {
    if (hn == MSPS_HEAP) return false;
    u32 i = hn++;
    while (i > 0) {
      const u32 p = (i - 1) >> 1;
      if (!before(x, heap[p])) break;
      heap[i] = heap[p];
      i = p;
    }
    heap[i] = x;
    return true;
  };
  auto pop = [&]() -> u32 {
    const u32 top = heap[0], x = heap[--hn];
    u32 i = 0;
    for (;;) {
      const u32 l = 2 * i + 1;
      if (l >= hn) break;
      const u32 c = (l + 1 < hn && before(heap[l + 1], heap[l])) ? l + 1 : l;
      if (!before(heap[c], x)) break;
      heap[i] = heap[c];
      i = c;
    }
    heap[i] = x;
    return top;
  };
  // the evicted neighbours of x in the walk's direction
  auto expand = [&](u32 x, u32 off, u32 cnt) -> bool {
    if constexpr (!DOWN) {
      for (u32 j = 0; j < cnt; j++) {
        const u32 p = g.wpar(off + j);
        b += 8;
        if (g.wev(p) && !push(p)) return false;
      }
    } else {
      b += 8;                                            // children record
      if (!g.L.linked) {
        for (u32 j = 0; j < cnt; j++) {
          const u32 c = g.m.w(g.L.ch + off + j);
          b += 8;
          if (g.wev(c) && !push(c)) return false;
        }
      } else {
        for (u32 e = g.crec(x).x; e != NONE; e = g.m.w(g.L.e_next + e)) {
          const u32 c = g.m.w(g.L.e_child + e);
          b += 8;
          if (g.wev(c) && !push(c)) return false;
        }
      }
    }
    return true;
  };
  if (!(DOWN ? expand(t, ar.z, ar.w) : expand(t, ar.x, ar.y))) return false;
  // the members' costs are summed four at a time (their loads in flight together,
  // off the walk's dependent chain)
  u32 p0 = NONE, p1 = NONE, p2 = NONE, p3 = NONE, np = 0;
  auto flush = [&]() {
    const u32 c0 = p0 != NONE ? g.srec(p0).y : 0u, c1 = p1 != NONE ? g.srec(p1).y : 0u;
    const u32 c2 = p2 != NONE ? g.srec(p2).y : 0u, c3 = p3 != NONE ? g.srec(p3).y : 0u;
    s += (u64)c0 + c1 + c2 + c3;
    p0 = p1 = p2 = p3 = NONE;
    np = 0;
  };
  u32 last = NONE;
  while (hn) {
    const u32 x = pop();
    if (x == last) continue;
    last = x;
    p3 = p2; p2 = p1; p1 = p0; p0 = x;
    if (++np == 4) flush();
    b += 16;
    const uint4 ax = DOWN ? g.arec(x) : make_uint4(0, 0, 0, 0);
    const uint2 px = DOWN ? make_uint2(ax.z, ax.w) : g.wprec(x);
    if (!expand(x, px.x, px.y)) return false;
  }
  flush();
  sum = s;
  bytes += b;
  return true;
}

// ---------------------------------------------------------------------------
// Exact argmin with a fast path.  key(c) = float(num) / float(den) as monotone
// u32 bits (0 = score 0, 0x7F800000 = +inf, 0xFFFFFFFF = no candidate).  The
// computed key of a finite nonzero score has relative error < 6 * 2^-24, so
// keys more than KEY_MARGIN ulps apart order exactly like the rationals; only
// keys within the margin (near-ties) are compared exactly in 128 bits.  Scores
// 0 and +inf are exact classes (ties broken by the smaller id, reading C-5).
// ---------------------------------------------------------------------------
constexpr u32 KEY_NONE = 0xFFFFFFFFu, KEY_INF = 0x7F800000u, KEY_MARGIN = 256u;   // 256 ulps >= 2^-16 relative

// Integer keys (ik): h_size and h_LRU scores are 1/m and 1/s with integer m, s,
// so key = ~den orders them exactly (score 0 -> 0, +inf -> 0xFFFFFFFE); equal
// keys are still resolved exactly, so the margin is 0 and no division is done.

__device__ __forceinline__ u32 cand_key(const Cand &c, bool ik = false) {
  if (c.id == NONE) return KEY_NONE;
  if (c.num == 0) return 0u;
  if (ik) return c.den == 0 ? 0xFFFFFFFEu : ~(u32)c.den;
  if (c.den == 0) return KEY_INF;
  return __float_as_uint(__fdividef(__ull2float_rn(c.num), __ull2float_rn(c.den)));
}

// best := min(best, c) exactly; bk tracks key(best)
__device__ __forceinline__ void cand_take(Cand &best, u32 &bk, const Cand &c, bool ik = false) {
  const u32 k = cand_key(c, ik);
  if (k == KEY_NONE) return;
  const u32 mg = ik ? 0u : KEY_MARGIN;
  bool better;
  if (k + mg < bk) better = true;
  else if (bk != KEY_NONE && k > bk + mg) better = false;
  else better = cand_less(c, best);
  if (better) { best = c; bk = k; }
}

__device__ __forceinline__ Cand shfl_cand(const Cand &c, int src) {
  Cand r;
  r.num = __shfl_sync(0xffffffffu, c.num, src);
  r.den = __shfl_sync(0xffffffffu, c.den, src);
  r.id = __shfl_sync(0xffffffffu, c.id, src);
  return r;
}


// warp-wide exact argmin using the key fast path; every lane gets the result.
__device__ __forceinline__ Cand warp_argmin_fast(const Cand &c, u32 k, bool ik = false) {
  const u32 FULL = 0xffffffffu;
  const u32 kmin = __reduce_min_sync(FULL, k);
  if (kmin == KEY_NONE) return cand_none();
  if (kmin == 0u || (!ik && kmin == KEY_INF)) {    // exact class: smallest id wins
    const u32 idmin = __reduce_min_sync(FULL, k == kmin ? c.id : NONE);
    const u32 m = __ballot_sync(FULL, k == kmin && c.id == idmin);
    return shfl_cand(c, __ffs(m) - 1);
  }
  const bool in = k <= kmin + (ik ? 0u : KEY_MARGIN);
  const u32 cont = __ballot_sync(FULL, in);
  if (__popc(cont) == 1) return shfl_cand(c, __ffs(cont) - 1);
  // near-ties: take the contender with the smallest id as reference; if no
  // contender's score is strictly below it, it is the exact argmin (exact ties,
  // the common case for size / LRU); else reduce the strictly-smaller ones exactly
  const u32 idref = __reduce_min_sync(FULL, in ? c.id : NONE);
  const Cand ref = shfl_cand(c, __ffs(__ballot_sync(FULL, in && c.id == idref)) - 1);
  const bool below = in && score_less(c, ref);
  u32 bm = __ballot_sync(FULL, below);
  Cand b = ref;
  while (bm) {                                     // the strictly-smaller contenders, exactly
    const Cand x = shfl_cand(c, __ffs(bm) - 1);
    bm &= bm - 1;
    if (cand_less(x, b)) b = x;
  }
  return b;
}

// E(t) aggregation for one candidate with evicted neighbours, in fixed
// unrolled phases so every load of a phase is independent (in-order issue
// would otherwise pay one memory latency per neighbour): neighbour ids ->
// their states (-> union-find roots) -> distinct component records.  Only for
// deg(t) <= NB and CSR children (not the per-call linked lists); returns the
// sum of the distinct adjacent components' cost and the max of their max la
// with la(t).  Used per lane by the whole-GPU team's phase 2 and by score_h.
constexpr u32 NB = 8;


template <bool SM, bool UF, u32 NB = dtr::NB>
__device__ __forceinline__ void nbr_components_phased(const Sim<SM> &g, const uint4 &sr, const uint4 &ar,
                                                      u64 &sum, u32 &L, u64 &bytes, u32 *Lr = nullptr) {
  const u32 deg = ar.y + ar.w;
  u32 q[NB], lab[NB];
#pragma unroll
  for (u32 j = 0; j < NB; j++)
    q[j] = j < deg ? (j < ar.y ? g.par(ar.x + j) : g.m.w(g.L.ch + ar.z + (j - ar.y))) : NONE;
#pragma unroll
  for (u32 j = 0; j < NB; j++) lab[j] = q[j] != NONE ? g.state(q[j]) : 0;
#pragma unroll
  for (u32 j = 0; j < NB; j++) {
    const u32 sq = lab[j];
    if constexpr (UF) lab[j] = is_evicted(sq) ? g.m.w(g.L.node_of + q[j]) : NONE;
    else lab[j] = is_evicted(sq) ? (sq & COMP_MASK) : NONE;
  }
  if constexpr (UF) {                       // union-find roots: every chain advances one step per round
    u32 up[NB], steps = 0;
#pragma unroll
    for (u32 j = 0; j < NB; j++) { up[j] = lab[j] != NONE ? g.uf(lab[j]).w : NONE; bytes += lab[j] != NONE ? 4 : 0; }
    for (;;) {
      bool more = false;
#pragma unroll
      for (u32 j = 0; j < NB; j++) more = more || up[j] != lab[j];
      if (!more) break;
#pragma unroll
      for (u32 j = 0; j < NB; j++)
        if (up[j] != lab[j]) { lab[j] = up[j]; up[j] = g.uf(lab[j]).w; steps++; }
    }
    bytes += 4ull * steps;
  }
  u32 cc[NB], cl[NB], ch[NB], nd = 0;
#pragma unroll
  for (u32 j = 0; j < NB; j++) {
    bool first = lab[j] != NONE;
#pragma unroll
    for (u32 i = 0; i < j; i++) first = first && lab[i] != lab[j];
    ch[j] = first ? lab[j] : NONE;
  }
#pragma unroll
  for (u32 j = 0; j < NB; j++) {            // distinct component records, all in flight
    if (ch[j] != NONE) {
      const uint4 r = UF ? g.uf(ch[j]) : g.comp(ch[j]);
      cc[j] = r.x; cl[j] = r.z; ch[j] = UF ? r.y : 0u;   // ch reused: cost high word (exact comps: u32 cost)
      nd++;
    } else {
      cc[j] = 0; cl[j] = 0; ch[j] = 0;
    }
  }
  u64 s = 0;
  u32 mx = 0;                               // the components' max la (encoded)
#pragma unroll
  for (u32 j = 0; j < NB; j++) { s += mk64(cc[j], ch[j]); mx = cl[j] > mx ? cl[j] : mx; }
  sum = s;
  if (Lr) *Lr = mx;
  L = mx > sr.z ? mx : sr.z;
  bytes += 16 + 8ull * deg + 12ull * nd;     // adjacency record, ids + states, components
}

// h'(s, m, c) = c / (m * s) with ablated measures = 1 (reading C-23)
__device__ __forceinline__ void abl_finish(u64 c, u32 mem, u32 la, const Cmd &cmd, Cand &out) {
  const u32 code = cmd.heur - H_ABL;
  const u32 m = (code & 2) ? mem : 1u;
  if (code & 1) stale_score(c, m, la, cmd.clock, out.num, out.den);
  else { out.num = c; out.den = m; }
}

// per-heuristic score of pool member t
template <bool SM, int H>
__device__ __forceinline__ void score_h(const Sim<SM> &g, const Cmd &cmd, u32 t, Cand &c, u64 &bytes) {
  c.id = t;
  if constexpr (H == H_DTR || H == H_DTR_EQ) {
    const uint4 sr = g.srec(t);
    u64 sum = 0;
    u32 L = sr.z;
    bytes += 16;                  // score record
    if (sr.w) {                   // evicted neighbours: walk them
      const uint4 ar = g.arec(t);
      // h_DTR: phased gathers (measured -7 % on the bench's h_DTR cells); h_DTR_eq's
      // union-find finds are chains, where the sequential walk measured faster
      if (H == H_DTR && !g.L.linked && ar.y + ar.w <= NB) {
        nbr_components_phased<SM, false>(g, sr, ar, sum, L, bytes);   // counts the adjacency record
      } else {
        nbr_components<SM, H == H_DTR_EQ>(g, t, ar, sum, L, bytes);
        bytes += 16;              // adjacency record
      }
    }
    stale_score((u64)sr.y + sum, sr.x, L, cmd.clock, c.num, c.den);
  } else if constexpr (H == H_LRU) {
    stale_score(1, 1, g.la(t), cmd.clock, c.num, c.den);
    bytes += 4;
  } else if constexpr (H == H_SIZE) {
    c.num = 1; c.den = g.srec(t).x;
    bytes += 4;
  } else if constexpr (H == H_LOCAL) {
    const uint4 sr = g.srec(t);
    stale_score((u64)sr.y, sr.x, sr.z, cmd.clock, c.num, c.den);
    bytes += 12;
  } else if constexpr (H == H_ABL) {           // h'(s, m, c) with c in {EqClass, local, no}
    const uint4 sr = g.srec(t);
    const u32 cc = abl_c(cmd.heur);
    u64 num = 1;
    if (cc == ABL_EQCLASS) {                   // c(t) + the distinct adjacent sets' costs
      u64 sum = 0;
      u32 L = 0;
      if (sr.w) {
        nbr_components<SM, true>(g, t, g.arec(t), sum, L, bytes);
        bytes += 16;
      }
      num = (u64)sr.y + sum;
    } else if (cc == ABL_LOCAL) {
      num = sr.y;
    }
    abl_finish(num, sr.x, sr.z, cmd, c);
    bytes += 16;
  } else {
    c.num = splitmix64(cmd.seed ^ (cmd.decisions << 32) ^ (u64)t); c.den = 1;
    bytes += 4;
  }
}

// Warp-cooperative E(t) aggregation for ONE candidate t with evicted neighbours
// (whole-GPU team, phase 2): lane j takes neighbour j (chunks of 32), so the
// chain adjacency record -> neighbour ids -> states (-> union-find roots) ->
// distinct component records costs four round trips whatever the degree.
// Duplicate labels are dropped with __match_any_sync within a chunk and by a
// shuffle scan against earlier chunks (degree > 32 only).  All lanes return
// the sum of the distinct adjacent components' cost and the max of their max
// la with la(t) (sr.z); bytes are counted per lane.
template <bool SM, bool UF>
__device__ __forceinline__ void nbr_components_warp(const Sim<SM> &g, u32 t, const uint4 &sr, u64 &sum, u32 &L,
                                                    u64 &bytes, u32 *Lr = nullptr) {
  const u32 FULL = 0xffffffffu, lane = threadIdx.x & 31;
  const uint4 ar = g.arec(t);
  const u32 deg = ar.y + ar.w;
  auto label = [&](u32 j, u64 &b) -> u32 {
    if (j >= deg) return NONE;
    const u32 q = j < ar.y ? g.par(ar.x + j) : g.m.w(g.L.ch + ar.z + (j - ar.y));
    const u32 sq = g.state(q);
    b += 8;
    if (!is_evicted(sq)) return NONE;
    if constexpr (UF) {
      u32 steps = 0;
      const u32 r = g.uf_root(g.m.w(g.L.node_of + q), steps);
      b += 4 + 4ull * steps;
      return r;
    } else {
      return sq & COMP_MASK;
    }
  };
  u64 s = 0;
  u32 mx = 0;
  if (lane == 0) bytes += 16;                       // adjacency record
  for (u32 base = 0; base < deg; base += 32) {
    const u32 lab = label(base + lane, bytes);
    const u32 grp = __match_any_sync(FULL, lab);
    bool first = lab != NONE && (u32)(__ffs(grp) - 1) == lane;
    for (u32 b0 = 0; b0 < base; b0 += 32) {         // earlier chunks (degree > 32)
      u64 junk = 0;
      const u32 prev = label(b0 + lane, junk);
      for (u32 k = 0; k < 32; k++) {             // every lane shuffles (no short-circuit around a sync op)
        const u32 x = __shfl_sync(FULL, prev, k);
        first = first && x != lab;
      }
    }
    if (first) {
      const uint4 r = UF ? g.uf(lab) : g.comp(lab);
      s += UF ? mk64(r.x, r.y) : (u64)r.x;
      mx = r.z > mx ? r.z : mx;
      bytes += 12;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(FULL, s, o);
    const u32 m2 = __shfl_xor_sync(FULL, mx, o);
    mx = m2 > mx ? m2 : mx;
  }
  sum = s;
  if (Lr) *Lr = mx;
  L = mx > sr.z ? mx : sr.z;
}

// Score this thread's share of the compact pool list (CTA engine, per-call),
// K candidates at a time (independent chains in flight), into best: the
// members pool_ids[rank + j * size].
template <bool SM, int H, u32 K>
__device__ __forceinline__ void score_loop(const Sim<SM> &g, const Cmd &cmd, u32 rank, u32 size, Cand &best,
                                           u32 &bk, u64 &bytes, u64 &evals) {
  const u32 n = cmd.pool_size;
  for (u32 i = rank; i < n; i += K * size) {
    u32 cand[K];
#pragma unroll
    for (u32 r = 0; r < K; r++) cand[r] = i + r * size < n ? g.pool_ids(i + r * size) : NONE;
    Cand c[K];
#pragma unroll
    for (u32 r = 0; r < K; r++)
      if (cand[r] != NONE) { score_h<SM, H>(g, cmd, cand[r], c[r], bytes); bytes += 4; evals++; }
#pragma unroll
    for (u32 r = 0; r < K; r++)
      if (cand[r] != NONE) cand_take(best, bk, c[r], int_key_heur(H));
  }
}

// Key of c/(m (clock + 1 - L)) with no 64-bit arithmetic (nev = 0 candidates
// of h_DTR / h_DTR_eq): clock < 2^32 - 1 (reading C-14), so s fits u32.  Three
// u32 -> f32 roundings, one product and __fdividef (<= 2 ulp) give a relative
// error below 8 * 2^-24, far inside KEY_MARGIN (256 ulps): keys farther apart
// than the margin order exactly like the rationals.  0 = score 0, KEY_INF = +inf.
__device__ __forceinline__ u32 stale_key(u32 c, u32 m, u32 L, u32 clock1) {
  if (L == 0) return 0u;
  const u32 s = clock1 - L;
  if (s == 0) return KEY_INF;
  return __float_as_uint(__fdividef(__uint2float_rn(c), __uint2float_rn(m) * __uint2float_rn(s)));
}

// Per-warp stack of deferred candidates in shared memory: (id, key of a LOWER
// bound of its score) pairs.  e = null: no stack (the caller re-scans instead).
struct SlowStack {
  uint2 *e;
  u32 cap;     // pairs; >= 32 * U + 32 where it is used
  u64 *msum;   // 32 sums of the multi-candidate closure walk (closure_multi)
};

// Drain a warp's stack down to `keep` entries: first drop every entry whose
// bound key exceeds `cur` (an exact score some candidate already has) by more
// than KEY_MARGIN -- its exact score is higher, so it cannot be the argmin --
// then resolve the rest from the top, 32 per round, one per lane
// (resolve(NONE) = idle lane; resolve is warp-collective).
template <class R>
__device__ __forceinline__ void stack_drain(const SlowStack &st, u32 &nq, u32 keep, u32 cur, R resolve) {
  const u32 FULL = 0xffffffffu, lane = threadIdx.x & 31;
  u32 out = 0;
  for (u32 i0 = 0; i0 < nq; i0 += 32) {      // compact the survivors to the front (order is irrelevant)
    const u32 i = i0 + lane;
    uint2 x = make_uint2(NONE, 0);
    bool k = false;
    if (i < nq) { x = st.e[i]; k = cur == KEY_NONE || !(x.y > cur + KEY_MARGIN); }
    const u32 m = __ballot_sync(FULL, k);
    if (k) st.e[out + __popc(m & ((1u << lane) - 1))] = x;   // writes never pass this chunk's reads
    out += __popc(m);
    __syncwarp();
  }
  if (lane == 0) { PROF_ADD(22, nq); PROF_ADD(23, out); }
  nq = out;
  while (nq > keep) {
    u32 take = nq - keep;
    take = take > 32 ? 32 : take;
    const u32 t = lane < take ? st.e[nq - take + lane].x : NONE;
    nq -= take;
    __syncwarp();
    resolve(t);
  }
}

// The team's best key so far: the warp's, and (block team) the shared word
// every warp lowers with atomicMin.  Any value is an exact score some
// candidate has, so it is a safe pruning bound at any time.
__device__ __forceinline__ u32 team_bound(u32 bk, u32 *sbest) {
  u32 b = __reduce_min_sync(0xffffffffu, bk);
  if (sbest) {
    if ((threadIdx.x & 31) == 0) atomicMin(sbest, b);
    const u32 s2 = *(volatile u32 *)sbest;
    b = s2 < b ? s2 : b;
  }
  return b;
}

// Whole-GPU pass over the pool BITMAP (grid engine, dtr_pool_argmin).  Warp w
// takes bitmap words w, w + W, w + 2W, ... (W = warps in the team) and lane l
// the id 32 * word + l, so each step reads one broadcast bitmap word and 32
// consecutive score records (512 B, coalesced), U steps in flight per lane.
// BM = false: the same pass over the compact pool list (CTA engine with its
// state in global memory): lane l of warp w takes pool slots 32 w + l,
// 32 (w + W) + l, ...; the ids are a coalesced load, the records a gather.
//
// Exact branch and bound.  A candidate with nev = 0 is scored from its record
// alone (stale_key: no 64-bit arithmetic unless it is a new best or a
// near-tie).  For a candidate with evicted neighbours the same record gives a
// LOWER bound of its score: adjacent components only add cost to the numerator
// and can only raise the max last access, which shortens the staleness
// (h_DTR_eq and the EqClass ablation alike).  Such candidates are
// pushed with their bound key on the warp's shared-memory stack; after the
// stream (or when the stack runs full) the team's best key so far prunes them
// (stack_drain: a bound above an exact score already found, by more than the
// margin, cannot be the argmin -- a tie needs equality) and the survivors are
// resolved 32 at a time, one per lane (phased gathers, nbr_components_phased;
// degree > NB: the whole warp, nbr_components_warp).  sbest: a shared word of a
// block-wide team (every thread of the block takes part; the caller resets it
// to KEY_NONE before the barrier that starts the team: one barrier after the
// stream lets every warp prune with the block's best), or null for a one-warp
// team.
template <bool SM, bool BM, int H, u32 U>
__device__ __forceinline__ void score_stream(const Sim<SM> &g, const Cmd &cmd, u32 wrank, u32 wsize, Cand &best,
                                             u32 &bk, u64 &bytes, u64 &evals, const SlowStack &st, u32 *sbest) {
  const u32 FULL = 0xffffffffu, lane = threadIdx.x & 31;
  const u32 nwords = BM ? (cmd.n_ids + 31) / 32 : (cmd.pool_size + 31) / 32;
  const u32 clock1 = (u32)(cmd.clock + 1);
  constexpr bool NBR = H == H_DTR || H == H_DTR_EQ || H == H_ABL;
  constexpr bool UF = H != H_DTR;
  // neighbourhood-reading variant? (the ablation only for c = EqClass)
  const bool nbr = NBR && (H != H_ABL || abl_c(cmd.heur) == ABL_EQCLASS);
  // own-record score (exact for nev = 0; a lower bound otherwise): key, and the rational on demand
  auto own_cand = [&](u32 id, const uint4 &r) {
    Cand c;
    c.id = id;
    if constexpr (H == H_ABL) abl_finish(abl_c(cmd.heur) == ABL_NO ? 1ull : (u64)r.y, r.x, r.z, cmd, c);
    else stale_score((u64)r.y, r.x, r.z, cmd.clock, c.num, c.den);
    return c;
  };
  auto own_key = [&](const uint4 &r) -> u32 {
    if constexpr (H == H_ABL) return cand_key(own_cand(0, r));
    else return stale_key(r.y, r.x, r.z, clock1);
  };
  // one slow candidate per lane (NONE: idle lane)
  auto resolve = [&](u32 t) {
    uint4 sr = make_uint4(0, 0, 0, 0), ar = make_uint4(0, 0, 0, 0);
    if (t != NONE) { sr = g.srec(t); ar = g.arec(t); }
    const bool big = t != NONE && ar.y + ar.w > NB;
    auto finish = [&](u32 tt, const uint4 &s4, u64 sum, u32 L, u32 Lr) {
      Cand c;
      c.id = tt;
      if constexpr (H == H_ABL) abl_finish((u64)s4.y + sum, s4.x, s4.z, cmd, c);
      else stale_score((u64)s4.y + sum, s4.x, L, cmd.clock, c.num, c.den);
      if (H == H_DTR_EQ && g.L.lcache) g.m.w(g.L.lcache + tt) = Lr + 1u;
      cand_take(best, bk, c);
    };
    // all lanes' degrees <= 4 (the common case on the recurrent logs): half-width phases
    const bool narrow = __all_sync(FULL, t == NONE || ar.y + ar.w <= 4);
    if (t != NONE && !big) {
      u64 sum;
      u32 L, Lr;
      if (narrow) nbr_components_phased<SM, UF, 4>(g, sr, ar, sum, L, bytes, &Lr);
      else nbr_components_phased<SM, UF>(g, sr, ar, sum, L, bytes, &Lr);
      finish(t, sr, sum, L, Lr);
    }
    u32 bm = __ballot_sync(FULL, big);
    while (bm) {
      const u32 l = __ffs(bm) - 1;
      bm &= bm - 1;
      const u32 tt = __shfl_sync(FULL, t, l);
      uint4 s4;
      s4.x = __shfl_sync(FULL, sr.x, l); s4.y = __shfl_sync(FULL, sr.y, l);
      s4.z = __shfl_sync(FULL, sr.z, l); s4.w = __shfl_sync(FULL, sr.w, l);
      u64 sum;
      u32 L, Lr;
      nbr_components_warp<SM, UF>(g, tt, s4, sum, L, bytes, &Lr);
      if (lane == l) finish(tt, s4, sum, L, Lr);
    }
  };
  u32 nq = 0;                                  // warp-uniform stack depth
  for (u32 w0 = wrank; w0 < nwords; w0 += U * wsize) {
    u32 bits[U], tid[U];
    uint4 sr[U];
#pragma unroll
    for (u32 j = 0; j < U; j++) {              // pool ids (bitmap words) and score records, all in flight
      const u32 w = w0 + j * wsize;
      if constexpr (BM) {
        tid[j] = w * 32 + lane;
        bits[j] = w < nwords ? g.pool_word(w) : 0u;
      } else {
        const u32 i = w * 32 + lane;
        tid[j] = i < cmd.pool_size ? g.pool_ids(i) : NONE;
        bits[j] = __ballot_sync(FULL, tid[j] != NONE);
      }
    }
#pragma unroll
    for (u32 j = 0; j < U; j++) {
      const bool ok = BM ? tid[j] < cmd.n_ids : tid[j] != NONE;
      sr[j] = ok ? g.srec(tid[j]) : make_uint4(0, 0, 0, 0);
    }
    if constexpr (NBR) {
      if (nbr) {                               // evicted neighbours: deferred with their bound key
        u32 lc[U];                             // h_DTR_eq: cached lower bound of the roots' max la
#pragma unroll
        for (u32 j = 0; j < U; j++)
          lc[j] = (H == H_DTR_EQ && g.L.lcache && ((bits[j] >> lane) & 1u) && sr[j].w) ? g.m.w(g.L.lcache + tid[j]) : 0u;
#pragma unroll
        for (u32 j = 0; j < U; j++) {
          const bool slow = ((bits[j] >> lane) & 1u) && sr[j].w != 0;
          const u32 m = __ballot_sync(FULL, slow);
          if (slow) {
            uint4 r = sr[j];
            if (lc[j] && lc[j] - 1u > r.z) r.z = lc[j] - 1u;   // L >= max(la(t), cached roots' max la)
            st.e[nq + __popc(m & ((1u << lane) - 1))] = make_uint2(tid[j], own_key(r));
          }
          nq += __popc(m);
        }
      }
    }
#pragma unroll
    for (u32 j = 0; j < U; j++) {
      const bool in = (bits[j] >> lane) & 1u;
      const u32 id = tid[j];
      if (!in) continue;
      evals++;
      if constexpr (NBR) {
        bytes += BM ? 16 : 20;                 // score record (+ pool slot)
        if (nbr && sr[j].w != 0) continue;     // deferred
        const u32 k = own_key(sr[j]);
        const bool clear = k + KEY_MARGIN < bk;
        if (clear || (bk != KEY_NONE && k <= bk + KEY_MARGIN)) {   // new best, or a near-tie: exact
          const Cand c = own_cand(id, sr[j]);
          if (clear || cand_less(c, best)) { best = c; bk = k; }
        }
      } else {
        Cand c;
        c.id = id;
        if constexpr (!BM) bytes += 4;         // pool slot
        if constexpr (H == H_LRU) {
          stale_score(1, 1, sr[j].z, cmd.clock, c.num, c.den);
          bytes += 4;
        } else if constexpr (H == H_SIZE) {
          c.num = 1; c.den = sr[j].x;
          bytes += 4;
        } else if constexpr (H == H_LOCAL) {
          stale_score((u64)sr[j].y, sr[j].x, sr[j].z, cmd.clock, c.num, c.den);
          bytes += 12;
        } else {
          c.num = splitmix64(cmd.seed ^ (cmd.decisions << 32) ^ (u64)c.id); c.den = 1;
          bytes += 4;
        }
        cand_take(best, bk, c, int_key_heur(H));
      }
    }
    if constexpr (NBR) {
      __syncwarp();
      if (nq + 32 * U > st.cap) stack_drain(st, nq, st.cap / 2, team_bound(bk, sbest), resolve);   // make room
    }
  }
  if constexpr (NBR) {
    if (!nbr) return;
    u32 cur = team_bound(bk, sbest);
    if (sbest) {                               // every warp's stream is in: prune with the block's best
      __syncthreads();
      cur = team_bound(bk, sbest);
    }
    stack_drain(st, nq, 0, cur, resolve);
  }
}

// h_size / h_LRU over the compact list: every pool slot carries its exact
// 64-bit key (integer score key << 32 | id, leader.cuh pool_key_of), so the
// scan is a plain 64-bit min and the winner's (num, den) is rebuilt from its
// record.  ~0 = no candidate.
template <bool SM>
__device__ __forceinline__ u64 team_intkey_min(const Sim<SM> &g, const Cmd &cmd, u32 rank, u32 size, u64 &bytes,
                                               u64 &evals) {
  u64 kmin = ~0ull;
  u32 cnt = 0;
#pragma unroll 4
  for (u32 i = rank; i < cmd.pool_size; i += size) {
    const uint2 k = g.m.d(g.L.pool_key + 2 * i);
    const u64 kk = mk64(k.x, k.y);
    kmin = kk < kmin ? kk : kmin;
    cnt++;
  }
  bytes += 8ull * cnt;
  evals += cnt;
  return kmin;
}
__device__ __forceinline__ u64 warp_min64(u64 k) {
  const u32 hi = (u32)(k >> 32), lo = (u32)k;
  const u32 mh = __reduce_min_sync(0xffffffffu, hi);
  const u32 ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xFFFFFFFFu);
  return mk64(ml, mh);
}
template <bool SM>
__device__ __forceinline__ Cand intkey_cand(const Sim<SM> &g, const Cmd &cmd, u64 k) {
  Cand c;
  c.id = (u32)k;
  if (cmd.heur == H_SIZE) { c.num = 1; c.den = g.srec(c.id).x; }
  else stale_score(1, 1, g.la(c.id), cmd.clock, c.num, c.den);
  return c;
}

// K5 pass: h_MSPS and the e* family.  One candidate per lane; its closure sum
// comes from the cache (ccache, valid unless an event since marked it stale),
// else from a lane walk (closure_lane), else -- frontier wider than the lane
// heap -- from a warp BFS (msps_closure).  Exact branch and bound as in
// score_stream: every candidate whose closure is known (no evicted neighbour,
// or a cache hit) is scored in the stream; the score with an EMPTY closure is
// a lower bound of a stale one's (the closure only adds cost to the
// numerator), so only stale candidates whose bound is
// not excluded by the team's best key are walked.  With a stack (st.e: CTA
// cells with global state, the whole-GPU engine) the stale candidates are
// stacked during the stream; without one (state in shared memory) pass 2
// re-scans the pool.  sbest: as in score_stream (null: one-warp team).
template <bool SM, bool BM>
__device__ __forceinline__ void team_closure(const Sim<SM> &g, const Cmd &cmd, u32 wrank, u32 wsize,
                                             volatile u32 *msps_tail, u64 &bytes, u64 &evals, Cand &best, u32 &bk,
                                             const SlowStack &st, u32 *sbest) {
  // CTA: one BFS slot per scoring warp; whole GPU (msps_lock): every warp walks
  // lanes, and the rare BFS fallback locks one of the bounded slots
  const bool locked = g.L.msps_lock != 0;
  const u32 nw = locked || wsize < g.L.msps_warps ? wsize : g.L.msps_warps;
  const bool active = wrank < nw;
  const u32 lane = threadIdx.x & 31;
  const u32 FULL = 0xffffffffu, n = BM ? cmd.n_ids : cmd.pool_size;
  const bool down = cmd.heur != H_MSPS;
  const bool use_cc = g.L.ccache && cmd.n_ev != NONE;
  auto make = [&](u32 t, const uint4 &sr, u64 sum) {
    Cand c;
    c.id = t;
    if (cmd.heur == H_DTR_FULL) {            // (c(S) + sum_{e*(S)} c) / (size(S) * stale(S))
      stale_score((u64)sr.y + sum, sr.x, sr.z, cmd.clock, c.num, c.den);
    } else if (is_abl(cmd.heur)) {           // h'(s, m, e*)
      abl_finish((u64)sr.y + sum, sr.x, sr.z, cmd, c);
    } else {                                 // MSPS and h_e* (P:1835-1837): (c0 + sum) / m
      c.num = (u64)sr.y + sum;
      c.den = sr.x;
    }
    return c;
  };
  constexpr u32 U = SM ? 1 : 4;            // global-memory state: four chunks' loads in flight per lane
  // U chunks of candidates: ids, score records and (nev > 0) cached closure halves
  auto fetch = [&](u32 base, u32 *tj, uint4 *srj, uint2 *ccj) {
#pragma unroll
    for (u32 j = 0; j < U; j++) {
      const u32 i = base + j * nw * 32 + lane;
      tj[j] = NONE;
      if (i < n) {
        if constexpr (BM) { if (g.in_pool(i)) tj[j] = i; }
        else tj[j] = g.pool_ids(i);
      }
    }
#pragma unroll
    for (u32 j = 0; j < U; j++) srj[j] = tj[j] != NONE ? g.srec(tj[j]) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (u32 j = 0; j < U; j++) ccj[j] = use_cc && srj[j].w ? g.ccache(tj[j]) : make_uint2(0, 0);
  };
  auto known = [&](const uint4 &sr, const uint2 &cc) { return !sr.w || (cc.x && (!down || cc.y)); };
  // walk the stale closure of one candidate per lane (NONE: idle lane); warp-collective
  auto resolve = [&](u32 t) {
#ifdef DTR_PROFILE
    { const u32 m = __ballot_sync(FULL, t != NONE); if (lane == 0) PROF_ADD(17, __popc(m)); }
#endif
    if constexpr (!SM) {
      // two or more stale candidates: one walk over the union of their closures
      if (g.L.msps_d && !g.L.mirror && st.msum && __popc(__ballot_sync(FULL, t != NONE)) >= 2) {
        u32 slot = wrank;
        if (locked) {                          // acquire a free slot (its holder always finishes)
          if (lane == 0) {
            u32 k = wrank % g.L.msps_warps;
            while (atomicCAS(&g.m.w(g.L.msps_lock + k), 0u, 1u) != 0u) k = k + 1 == g.L.msps_warps ? 0 : k + 1;
            __threadfence();
            slot = k;
          }
          slot = __shfl_sync(FULL, slot, 0);
        }
        u64 up = 0, dn = 0;
        const bool okm = closure_multi(g, t, slot, msps_tail + (threadIdx.x >> 5), st.msum, down, up, dn, bytes);
        if (locked && lane == 0) { __threadfence(); atomicExch(&g.m.w(g.L.msps_lock + slot), 0u); }
        if (lane == 0) PROF_ADD(19 + 5, 1);
        if (okm) {
          if (t != NONE) {
            const uint4 sr = g.srec(t);
            if (use_cc) g.ccache(t) = make_uint2((u32)up + 1u, down ? (u32)dn + 1u : 0u);
            cand_take(best, bk, make(t, sr, up + dn));
            bytes += 16;
          }
          return;
        }
      }
    }
    uint4 sr = make_uint4(0, 0, 0, 0);
    uint2 cc = make_uint2(0, 0);
    if (t != NONE) { sr = g.srec(t); if (use_cc) cc = g.ccache(t); }
    bool ok = true;
    if (t != NONE) {
      u64 up = cc.x ? cc.x - 1u : 0, dn = cc.y ? cc.y - 1u : 0, b = 0;
      const bool wu = !cc.x, wd = down && !cc.y;
      const uint4 ar = g.arec(t);
      ok = (!wu || closure_lane<SM, false>(g, t, ar, up, b)) && (!wd || closure_lane<SM, true>(g, t, ar, dn, b));
      if (ok) {
        bytes += b;
        if (use_cc) g.ccache(t) = make_uint2((u32)up + 1u, down ? (u32)dn + 1u : 0u);
        cand_take(best, bk, make(t, sr, up + dn));
      }
      bytes += 16;                           // adjacency record
    }
    u32 ov = __ballot_sync(FULL, t != NONE && !ok);
    while (ov) {
      const u32 l = __ffs(ov) - 1;
      ov &= ov - 1;
      const u32 tt = __shfl_sync(FULL, t, l);
      u32 slot = wrank;
      if (locked) {                            // acquire a free slot (its holder always finishes)
        if (lane == 0) {
          u32 k = wrank % g.L.msps_warps;
          while (atomicCAS(&g.m.w(g.L.msps_lock + k), 0u, 1u) != 0u) k = k + 1 == g.L.msps_warps ? 0 : k + 1;
          __threadfence();
          slot = k;
        }
        slot = __shfl_sync(FULL, slot, 0);
      }
      u64 u2 = 0;
      if (lane == 0) PROF_ADD(18, 1);
      const u64 s2 = msps_closure(g, g.arec(tt), slot, msps_tail + (threadIdx.x >> 5), bytes, tt, down, &u2);
      if (locked && lane == 0) { __threadfence(); atomicExch(&g.m.w(g.L.msps_lock + slot), 0u); }
      if (lane == l) {
        if (use_cc) g.ccache(tt) = make_uint2((u32)u2 + 1u, down ? (u32)(s2 - u2) + 1u : 0u);
        cand_take(best, bk, make(tt, sr, s2));
      }
    }
  };
  u32 nq = 0;                                  // stack depth (warp-uniform)
  // ---- the stream: candidates whose closure is known; stale ones stacked (or left for the re-scan)
  if (active) {
    for (u32 base = wrank * 32; base < n; base += U * nw * 32) {
      u32 tj[U];
      uint4 srj[U];
      uint2 ccj[U];
      fetch(base, tj, srj, ccj);
      if (st.e) {
#pragma unroll
        for (u32 j = 0; j < U; j++) {
          const bool stale = tj[j] != NONE && !known(srj[j], ccj[j]);
          const u32 m = __ballot_sync(FULL, stale);
          if (stale) st.e[nq + __popc(m & ((1u << lane) - 1))] = make_uint2(tj[j], cand_key(make(tj[j], srj[j], 0)));
          nq += __popc(m);
        }
      }
#pragma unroll
      for (u32 j = 0; j < U; j++) {
        if (tj[j] == NONE) continue;
        evals++;
        bytes += 16;                           // score record
        if (srj[j].w) bytes += use_cc ? 8 : 0; // cached halves
        if (!known(srj[j], ccj[j])) continue;  // stale
        const u64 sum = srj[j].w ? (u64)(ccj[j].x - 1u) + (down ? (u64)(ccj[j].y - 1u) : 0ull) : 0ull;
        cand_take(best, bk, make(tj[j], srj[j], sum));
      }
#ifdef DTR_PROFILE
      for (u32 j = 0; j < U; j++) {
        const u32 m = __ballot_sync(FULL, tj[j] != NONE && srj[j].w && known(srj[j], ccj[j]));
        if (lane == 0) PROF_ADD(16, __popc(m));
      }
#endif
      if (st.e) {
        __syncwarp();
        if (nq + 32 * U > st.cap) stack_drain(st, nq, st.cap / 2, team_bound(bk, sbest), resolve);
      }
    }
  }
  // ---- the team's best key, then the stale closures it does not exclude
  u32 cur = team_bound(bk, sbest);
  if (sbest) {
    __syncthreads();
    cur = team_bound(bk, sbest);
  }
  if (!active) return;
  if (st.e) {
    stack_drain(st, nq, 0, cur, resolve);
    return;
  }
  for (u32 base = wrank * 32; base < n; base += U * nw * 32) {   // re-scan (state in shared memory)
    u32 tj[U];
    uint4 srj[U];
    uint2 ccj[U];
    fetch(base, tj, srj, ccj);
#pragma unroll
    for (u32 j = 0; j < U; j++) {
      u32 t = tj[j];
      if (t != NONE && known(srj[j], ccj[j])) t = NONE;
      if (t != NONE && cur != KEY_NONE) {
        const u32 lb = cand_key(make(t, srj[j], 0));
        const u32 c2 = bk < cur ? bk : cur;
        if (lb > c2 + KEY_MARGIN) t = NONE;    // excluded: lb > an exact score already found
      }
      resolve(t);
    }
  }
}

// Score every pool member of this thread's slice; return the slice argmin and
// its key.  rank/size: thread index in the team; wrank/wsize: warp index (MSPS).
// WIDE: global-memory team (four candidates in flight per thread, else two).
template <bool SM, bool BM, bool WIDE = false, bool CL = true>
__device__ Cand team_score(const Sim<SM> &g, const Cmd &cmd, u32 rank, u32 size, u32 wrank, u32 wsize,
                           volatile u32 *msps_tail, u64 &bytes, u64 &evals, u32 &bk,
                           const SlowStack &st = SlowStack{nullptr, 0, nullptr}, u32 *sbest = nullptr) {
  Cand best = cand_none();
  bk = KEY_NONE;
  if (BM && rank == 0) bytes += (cmd.n_ids + 7) / 8;     // the pool bitmap
  if constexpr (CL) {   // CL = false: a kernel built for batches without closure heuristics (dtr.cu)
    if (uses_closure(cmd.heur)) {
      team_closure<SM, BM>(g, cmd, wrank, wsize, msps_tail, bytes, evals, best, bk, st, sbest);
      return best;
    }
  }
  constexpr u32 K = WIDE ? 4 : 2;
  if constexpr (!SM && BM) {
    switch (cmd.heur) {
      case H_DTR: score_stream<false, true, H_DTR, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best;
      case H_DTR_EQ: score_stream<false, true, H_DTR_EQ, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best;
      case H_LRU: score_stream<false, true, H_LRU, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best;
      case H_SIZE: score_stream<false, true, H_SIZE, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best;
      case H_LOCAL: score_stream<false, true, H_LOCAL, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best;
      case H_RANDOM: score_stream<false, true, H_RANDOM, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best;
      default:
        if (is_abl(cmd.heur) && abl_c(cmd.heur) != ABL_ESTAR) {
          score_stream<false, true, H_ABL, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest);
          return best;
        }
        break;
    }
  } else {
  if (g.L.pool_key) {
    const u64 kmin = team_intkey_min(g, cmd, rank, size, bytes, evals);
    if (kmin != ~0ull) { best = intkey_cand(g, cmd, kmin); bk = cand_key(best, true); }
    return best;
  }
  if constexpr (!SM) {   // state in global memory (CTA engine): the stream pass with its slow stack
    if (st.e) {
      if (cmd.heur == H_DTR) { score_stream<false, false, H_DTR, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best; }
      if (cmd.heur == H_DTR_EQ) { score_stream<false, false, H_DTR_EQ, 4>(g, cmd, wrank, wsize, best, bk, bytes, evals, st, sbest); return best; }
    }
  }
  switch (cmd.heur) {
    case H_DTR: score_loop<SM, H_DTR, K>(g, cmd, rank, size, best, bk, bytes, evals); return best;
    case H_DTR_EQ: score_loop<SM, H_DTR_EQ, K>(g, cmd, rank, size, best, bk, bytes, evals); return best;
    case H_LRU: score_loop<SM, H_LRU, K>(g, cmd, rank, size, best, bk, bytes, evals); return best;
    case H_SIZE: score_loop<SM, H_SIZE, K>(g, cmd, rank, size, best, bk, bytes, evals); return best;
    case H_LOCAL: score_loop<SM, H_LOCAL, K>(g, cmd, rank, size, best, bk, bytes, evals); return best;
    case H_RANDOM: score_loop<SM, H_RANDOM, K>(g, cmd, rank, size, best, bk, bytes, evals); return best;
    default:
      if (is_abl(cmd.heur) && abl_c(cmd.heur) != ABL_ESTAR) {
        score_loop<SM, H_ABL, 2>(g, cmd, rank, size, best, bk, bytes, evals);
        return best;
      }
      break;
  }
  }
  return best;
}

// per-call OP_SCORES (compact pool): write every pool member's score (MSPS included)
template <bool SM>
__device__ void team_scores_out(const Sim<SM> &g, const Cmd &cmd, u32 rank, u32 size, volatile u32 *msps_tail,
                                u64 *onum, u64 *oden, u32 *oid) {
  const u32 P = cmd.pool_size;
  u64 junk = 0;
  if (uses_closure(cmd.heur)) {
    const u32 wr = rank >> 5, ws = (size + 31) >> 5, lane = threadIdx.x & 31;
    const u32 nw = ws < g.L.msps_warps ? ws : g.L.msps_warps;
    if (wr >= nw) return;
    for (u32 i = wr; i < P; i += nw) {
      const u32 t = g.pool_ids(i);
      const uint4 sr = g.srec(t);
      const u64 sum = sr.w ? msps_closure(g, g.arec(t), wr, msps_tail + (threadIdx.x >> 5), junk, t, cmd.heur != H_MSPS) : 0;
      if (lane == 0) {
        u64 num = (u64)sr.y + sum, den = sr.x;
        if (cmd.heur == H_DTR_FULL) stale_score((u64)sr.y + sum, sr.x, sr.z, cmd.clock, num, den);
        if (is_abl(cmd.heur)) {
          Cand c;
          abl_finish((u64)sr.y + sum, sr.x, sr.z, cmd, c);
          num = c.num; den = c.den;
        }
        onum[i] = num; oden[i] = den; oid[i] = t;
      }
    }
    return;
  }
  for (u32 i = rank; i < P; i += size) {
    const u32 t = g.pool_ids(i);
    Cand c;
    switch (cmd.heur) {
      case H_DTR: score_h<SM, H_DTR>(g, cmd, t, c, junk); break;
      case H_DTR_EQ: score_h<SM, H_DTR_EQ>(g, cmd, t, c, junk); break;
      case H_LRU: score_h<SM, H_LRU>(g, cmd, t, c, junk); break;
      case H_SIZE: score_h<SM, H_SIZE>(g, cmd, t, c, junk); break;
      case H_LOCAL: score_h<SM, H_LOCAL>(g, cmd, t, c, junk); break;
      case H_RANDOM: score_h<SM, H_RANDOM>(g, cmd, t, c, junk); break;
      default: score_h<SM, H_ABL>(g, cmd, t, c, junk); break;
    }
    onum[i] = c.num; oden[i] = c.den; oid[i] = t;
  }
}

// ---------------------------------------------------------------------------
// Reductions
// ---------------------------------------------------------------------------
struct RedSmem {
  Cand warp[32];
};

// block-wide argmin; the result is valid in warp 0 (all lanes) after return.
__device__ __forceinline__ Cand block_argmin(const Cand &c, u32 k, RedSmem &sm, bool ik = false) {
  Cand w = warp_argmin_fast(c, k, ik);
  const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) sm.warp[wid] = w;
  __syncthreads();
  if (wid == 0) {
    w = lane < nw ? sm.warp[lane] : cand_none();
    w = warp_argmin_fast(w, cand_key(w, ik), ik);
  }
  return w;
}

// block-wide sum of two counters; result valid in thread 0
__device__ __forceinline__ void block_sum2(u64 &a, u64 &b, RedSmem &sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) { sm.warp[wid].num = a; sm.warp[wid].den = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0; b = 0;
    for (u32 i = 0; i < nw; i++) { a += sm.warp[i].num; b += sm.warp[i].den; }
  }
  __syncthreads();
}

}  // namespace dtr
