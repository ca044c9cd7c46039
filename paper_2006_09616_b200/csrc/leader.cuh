// leader.cuh -- the sequential control of one simrd simulation, run by ONE
// leader thread as a resumable state machine (explicit get_internal stack).
//
//   make_tensor      P:327-343       get_internal   P:213-245 (depth-first)
//   release_internal P:247-259       evict
//   free             P:273-284       banish_V2
//   get / release / rematerialize
//   union-find evicted components with approximate split (h_DTR_eq)
//                                    P:1236-1250
//   exact evicted components (h_DTR: E(t) of P:63-68 is the union of the
//   components adjacent to t; maintained incrementally -- merge the smaller
//   into the larger on evict; on rematerialization, interleaved searches from
//   t's evicted neighbours split off only the smaller pieces).  Labels are
//   slots of the component table, recycled through a free stack.
//
// resume() runs until free() needs an eviction decision (returns CMD_ARGMIN;
// the team computes it and the next resume() applies it) or the op range is
// exhausted / the run stops (CMD_DONE).
#pragma once
#include "engine.cuh"
#include "../../include/dtr.h"

namespace dtr {

enum { PH_OP = 0, PH_GI = 1, PH_FREE = 2, PH_SCORED = 3, PH_DONE = 4 };
enum { CMD_DONE = 0, CMD_ARGMIN = 1, CMD_SCORES = 2 };

struct Cmd {
  u64 clock, decisions, seed;
  u32 kind, pool_size, heur, n_ids;   // n_ids: tensor ids [0, n_ids) to scan for pool members
  u32 n_ev;                           // closure cache: events queued (NONE: do not use the cache)
};

template <bool SM, bool BM>
struct Leader {
  Sim<SM> g;
  Scalars s;
  const u32 *ops;         // op stream (batch) -- null in per-call mode
  dtr_evict_rec *trace;   // cell's trace region (may be null)
  u32 op_idx, op_end;
  u32 phase, post, root;
  u32 percall;
  u64 free_size;

  // ------------------------------------------------------------- pool
  // R.pool: bitmap over tensor ids (BM) or compact list with positions
  // size / LRU over a compact list: the slot's exact integer key (engine.cuh)
  __device__ __forceinline__ uint2 pool_key_of(u32 t) {
    const uint4 sr = g.srec(t);
    return make_uint2(t, s.heuristic == H_SIZE ? ~sr.x : sr.z);
  }
  __device__ __forceinline__ void pool_add(u32 t) {
    if constexpr (BM) {
      g.pool_word(t >> 5) |= 1u << (t & 31);
      s.pool_size++;
    } else {
      const u32 k = s.pool_size++;
      g.pool_pos(t) = k;
      g.pool_ids(k) = t;
      if (g.L.pool_key) g.m.d(g.L.pool_key + 2 * k) = pool_key_of(t);
    }
  }
  // la(t) changed: refresh t's key if it is a pool member (LRU)
  __device__ __forceinline__ void pool_rekey(u32 t) {
    if constexpr (!BM) {
      if (g.L.pool_key && s.heuristic == H_LRU) {
        const u32 p = g.pool_pos(t);
        if (p != NONE) g.m.d(g.L.pool_key + 2 * p) = pool_key_of(t);
      }
    }
  }
  __device__ __forceinline__ void pool_remove(u32 t) {
    if constexpr (BM) {
      const u32 w = g.pool_word(t >> 5), b = 1u << (t & 31);
      if (!(w & b)) return;
      g.pool_word(t >> 5) = w & ~b;
      s.pool_size--;
    } else {
      const u32 p = g.pool_pos(t);
      if (p == NONE) return;
      const u32 last = g.pool_ids(--s.pool_size);
      g.pool_ids(p) = last;
      g.pool_pos(last) = p;
      g.pool_pos(t) = NONE;
      if (g.L.pool_key) g.m.d(g.L.pool_key + 2 * p) = g.m.d(g.L.pool_key + 2 * s.pool_size);
    }
  }
  __device__ __forceinline__ bool pool_has(u32 t) {
    if constexpr (BM) return g.in_pool(t);
    else return g.pool_pos(t) != NONE;
  }
  // get_internal branch "t.m = T": l++, pool \ {t}
  __device__ __forceinline__ void lock(u32 t) {
    u32 l = g.ell(t);
    if (l == 0) pool_remove(t);
    g.ell(t) = l + 1;
  }
  // release_internal; V1 retries banishing here
  __device__ __forceinline__ void release_internal(u32 t) {
    u32 l = g.ell(t) - 1;
    g.ell(t) = l;
    if (l == 0 && !is_banished(g.state(t))) pool_add(t);
    if (s.dealloc == DEALLOC_V1) maybe_banish(t);
  }

  // ------------------------------------------------------------- V1 banishing (reading C-22)
  // children of t that exist (created), are not banished, and are not material?
  __device__ __forceinline__ bool child_not_material(u32 t) {
    const uint2 cr = g.crec(t);
    bool bad = false;
    if (!g.L.linked) {
      for (u32 j = 0; j < cr.y && !bad; j++) {
        const u32 c = g.m.w(g.L.ch + cr.x + j);
        if (c >= s.n_alloc) continue;                 // not created yet: not in t.C
        const u32 sc = g.state(c);
        if (!is_banished(sc) && !is_material(sc)) bad = true;
      }
    } else {
      for (u32 e = cr.x; e != NONE && !bad; e = g.m.w(g.L.e_next + e)) {
        const u32 sc = g.state(g.m.w(g.L.e_child + e));
        if (!is_banished(sc) && !is_material(sc)) bad = true;
      }
      // the tensor under creation is already in t.C but not yet linked
      if (!bad && s.n_alloc > 0 && !(g.state(s.n_alloc - 1) & O_BIT)) {
        const uint2 pn = g.prec(s.n_alloc - 1);
        for (u32 j = 0; j < pn.y; j++) if (g.par(pn.x + j) == t) bad = true;
      }
    }
    return bad;
  }
  __device__ __forceinline__ void maybe_banish(u32 t) {
    const u32 st = g.state(t);
    if (is_banished(st) || g.rho(t) != 0 || child_not_material(t)) return;
    // banish_V1
    const uint4 sr = g.srec(t);
    const uint4 ar = g.arec(t);
    g.state(t) = (st & O_BIT) | B_BIT;
    if (is_material(st)) {
      s.M -= sr.x;
      pool_remove(t);
    } else if (is_evicted(st)) {                     // leaves its evicted component
      ev_push(t);
      g.mirror_bit(t, false);
      nev_add(t, ar, NONE);
      if (s.heuristic == H_DTR) remat_exact(t, ar, st & COMP_MASK);
      else if (uses_uf(s.heuristic)) remat_uf(t, sr.y);
    }
    auto pin = [&](u32 c) {                           // c.l := c.l + 1 (pinned: out of the pool)
      if (is_banished(g.state(c))) return;
      const u32 l = g.ell(c);
      if (l == 0) pool_remove(c);
      g.ell(c) = l + 1;
    };
    const uint2 cr = g.crec(t);
    if (!g.L.linked) {
      for (u32 j = 0; j < cr.y; j++) { const u32 c = g.m.w(g.L.ch + cr.x + j); if (c < s.n_alloc) pin(c); }
    } else {
      for (u32 e = cr.x; e != NONE; e = g.m.w(g.L.e_next + e)) pin(g.m.w(g.L.e_child + e));
    }
  }

  // ------------------------------------------------------------- evicted-neighbour counts
  // t has just become evicted (d = 1) or stopped being evicted (d = -1): every
  // neighbour's nev changes by d.  Tensors not yet created may be counted too;
  // every such count is back to 0 by their first computation (all parents are
  // resident then), where it is reset anyway for the linked (per-call) lists.
  __device__ __forceinline__ void nev_add(u32 t, const uint4 &ar, u32 d) {
    if (!g.L.track_nev) return;
    if (g.L.lcache) g.for_each_nbr(t, ar, [&](u32 q) { g.nev(q) += d; g.m.w(g.L.lcache + q) = 0; });
    else g.for_each_nbr(t, ar, [&](u32 q) { g.nev(q) += d; });
  }

  // ------------------------------------------------------------- exact components
  // Component labels are slots of the component table, taken from a free stack
  // (or the never-used range) and returned when a component is absorbed or
  // dissolved; member lists are doubly linked.  Record {cost, nmax, maxla,
  // size}: cost = sum of the members' c0 (< 2^32, reading C-14), maxla = the
  // max encoded la over the members and nmax = how many members hold it, so
  // removing a holder forces a rescan only when it was the last one.
  __device__ __forceinline__ u32 comp_alloc() {
    if (s.comp_top) return g.m.w(g.L.comp_free + --s.comp_top);
    return s.comp_fresh++;
  }
  __device__ __forceinline__ void comp_release(u32 c) { g.m.w(g.L.comp_free + s.comp_top++) = c; }

  // merge component b into a (a, b labels; the larger keeps its label)
  __device__ __forceinline__ u32 comp_merge(u32 a, u32 b) {
    uint4 ca = g.comp(a), cb = g.comp(b);
    if (ca.w < cb.w) { u32 x = a; a = b; b = x; uint4 y = ca; ca = cb; cb = y; }
    u32 x = g.m.w(g.L.comp_head + b), last = NONE;
    while (x != NONE) { g.state(x) = O_BIT | a; last = x; x = g.m.w(g.L.mem_next + x); }
    const u32 ha = g.m.w(g.L.comp_head + a);
    g.m.w(g.L.mem_next + last) = ha;
    if (ha != NONE) g.m.w(g.L.mem_prev + ha) = last;
    g.m.w(g.L.comp_head + a) = g.m.w(g.L.comp_head + b);
    const u32 mx = ca.z > cb.z ? ca.z : cb.z;
    const u32 nm = (ca.z == mx ? ca.y : 0u) + (cb.z == mx ? cb.y : 0u);
    g.comp(a) = make_uint4(ca.x + cb.x, nm, mx, ca.w + cb.w);
    comp_release(b);
    return a;
  }

  // t has just become evicted: {t} joins the components of its evicted neighbours.
  // (fused: every neighbour's nev += 1)
  __device__ __forceinline__ void evict_exact(u32 t, const uint4 &sr, const uint4 &ar) {
    const u32 c0 = comp_alloc();
    g.comp(c0) = make_uint4(sr.y, 1, sr.z, 1);
    g.m.w(g.L.comp_head + c0) = t;
    g.m.w(g.L.mem_next + t) = NONE;
    g.m.w(g.L.mem_prev + t) = NONE;
    g.state(t) = O_BIT | c0;
    u32 cur = c0;
    g.for_each_nbr(t, ar, [&](u32 q) {
      g.nev(q) += 1;
      u32 sq = g.state(q);
      if (!is_evicted(sq)) return;
      u32 cq = sq & COMP_MASK;
      if (cq != cur) cur = comp_merge(cur, cq);
    });
  }

  // {max la, number of holders} over the members of c (la encoded, 0 = -inf)
  __device__ __forceinline__ uint2 comp_rescan_maxla(u32 c) {
    u32 mx = 0, nm = 0;
    for (u32 x = g.m.w(g.L.comp_head + c); x != NONE; x = g.m.w(g.L.mem_next + x)) {
      const u32 l = g.la(x);
      if (l > mx) { mx = l; nm = 1; } else if (l == mx) nm++;
    }
    return make_uint2(mx, nm);
  }

  __device__ __forceinline__ void list_unlink(u32 c, u32 x) {
    const u32 p = g.m.w(g.L.mem_prev + x), nx = g.m.w(g.L.mem_next + x);
    if (p != NONE) g.m.w(g.L.mem_next + p) = nx;
    else g.m.w(g.L.comp_head + c) = nx;
    if (nx != NONE) g.m.w(g.L.mem_prev + nx) = p;
  }

  // BFS visit stamps: (epoch << 5) | search id; the epoch wraps after 2^27 splits
  __device__ __forceinline__ u32 next_epoch() {
    if (s.epoch == (1u << 27) - 1) {
      for (u32 q = 0; q < s.n_alloc; q++) g.m.w(g.L.stamp + q) = 0;
      s.epoch = 0;
    }
    return (++s.epoch) << 5;
  }

  // Removing t from its component c may split c \ {t} into up to k = nev(t)
  // pieces, one per evicted neighbour of t at most.  k = 0: c was {t}.  k = 1:
  // t was a leaf, c \ {t} stays connected.  k >= 2: one search per evicted
  // neighbour, expanded one node at a time in turn; searches that meet are
  // the same piece.  A search group whose queues run dry has found a whole
  // piece; the run stops as soon as at most one group is still growing --
  // that one is the rest of c and keeps its label and member list, so only
  // the smaller pieces are ever walked (all groups meeting = no split, the
  // common case when t's evicted neighbours are linked around it).
  static constexpr u32 KS = 32;
  __device__ void remat_exact(u32 t, const uint4 &ar, u32 c) {
    const uint4 cc = g.comp(c);
    if (cc.w == 1) { comp_release(c); return; }
    const uint4 st = g.srec(t);
    list_unlink(c, t);
    const u32 k = g.nev(t);
    if (k > KS) { split_all(t, ar, c); return; }
    u32 cost = cc.x - st.y, size = cc.w - 1, nmax = cc.y - (st.z == cc.z ? 1u : 0u);
    if (k >= 2) {
      u32 first[KS], cur[KS], last[KS], cst[KS], sz[KS], nmc[KS], up[KS];
      u32 nq = 0;
      const u32 ep = next_epoch();
      const u32 VN = g.L.bfs_q;                          // visit lists (vnext)
      auto seed = [&](u32 q) {
        const u32 i = nq++;
        const uint4 sq = g.srec(q);
        g.m.w(g.L.stamp + q) = ep | i;
        g.m.w(VN + q) = NONE;
        first[i] = cur[i] = last[i] = q;
        cst[i] = sq.y; sz[i] = 1; nmc[i] = sq.z == cc.z ? 1u : 0u; up[i] = i;
      };
      g.for_each_nbr(t, ar, [&](u32 q) { if (is_evicted(g.state(q))) seed(q); });
      auto root = [&](u32 i) { while (up[i] != i) i = up[i]; return i; };
      u32 nclass = nq, nopen = nq;
      while (nopen > 1 && nclass > 1) {
        for (u32 i = 0; i < nq; i++) {                   // one expansion per growing search
          const u32 x = cur[i];
          if (x == NONE) continue;
          cur[i] = x == last[i] ? NONE : g.m.w(VN + x);
          g.for_each_nbr(x, g.arec(x), [&](u32 y) {
            if (!is_evicted(g.state(y))) return;
            const u32 sy = g.m.w(g.L.stamp + y);
            if ((sy & ~31u) == ep) {                     // met another search: same piece
              const u32 a = root(i), b = root(sy & 31u);
              if (a != b) { up[b] = a; nclass--; }
              return;
            }
            const uint4 ry = g.srec(y);
            g.m.w(g.L.stamp + y) = ep | i;
            g.m.w(VN + y) = NONE;
            g.m.w(VN + last[i]) = y;
            last[i] = y;
            if (cur[i] == NONE) cur[i] = y;
            cst[i] += ry.y; sz[i]++; nmc[i] += ry.z == cc.z ? 1u : 0u;
          });
        }
        // growing groups: a group is growing while any of its searches has a queue
        u32 open = 0;
        for (u32 i = 0; i < nq; i++) if (up[i] == i) {
          bool g2 = false;
          for (u32 j = 0; j < nq && !g2; j++) if (cur[j] != NONE && root(j) == i) g2 = true;
          open += g2;
        }
        nopen = open;
      }
      if (nclass > 1) {
        // the group that keeps label c: the growing one, else the largest
        u32 keep = NONE, best = 0;
        for (u32 i = 0; i < nq; i++) if (cur[i] != NONE) keep = root(i);
        if (keep == NONE) {
          for (u32 i = 0; i < nq; i++) if (up[i] == i) {
            u32 tot = 0;
            for (u32 j = 0; j < nq; j++) if (root(j) == i) tot += sz[j];
            if (tot > best) { best = tot; keep = i; }
          }
        }
        for (u32 r = 0; r < nq; r++) {                   // every other group is a whole piece
          if (up[r] != r || r == keep) continue;
          const u32 nc = comp_alloc();
          u32 pc = 0, ps = 0, pm = 0, plst = NONE;
          for (u32 j = 0; j < nq; j++) {
            if (root(j) != r) continue;
            pc += cst[j]; ps += sz[j];
            for (u32 x = first[j];; x = g.m.w(VN + x)) {
              list_unlink(c, x);
              g.state(x) = O_BIT | nc;
              g.m.w(g.L.mem_next + x) = plst;
              g.m.w(g.L.mem_prev + x) = NONE;
              if (plst != NONE) g.m.w(g.L.mem_prev + plst) = x;
              plst = x;
              const u32 l = g.la(x);
              if (l > pm) pm = l;
              if (x == last[j]) break;
            }
          }
          u32 pn = 0;
          for (u32 x = plst; x != NONE; x = g.m.w(g.L.mem_next + x)) pn += g.la(x) == pm;
          g.m.w(g.L.comp_head + nc) = plst;
          g.comp(nc) = make_uint4(pc, pn, pm, ps);
          for (u32 j = 0; j < nq; j++) if (root(j) == r) nmax -= nmc[j];
          cost -= pc; size -= ps;
        }
      }
    }
    u32 mx = cc.z;
    if (nmax == 0) { const uint2 r = comp_rescan_maxla(c); mx = r.x; nmax = r.y; }
    g.comp(c) = make_uint4(cost, nmax, mx, size);
  }

  // fallback for k > KS searches: relabel every piece of c \ {t} by BFS from
  // t's evicted neighbours (c's label is released; t is already unlinked)
  __device__ void split_all(u32 t, const uint4 &ar, u32 c) {
    comp_release(c);
    const u32 ep = next_epoch();
    g.for_each_nbr(t, ar, [&](u32 q) {
      u32 sq = g.state(q);
      if (!is_evicted(sq) || (g.m.w(g.L.stamp + q) & ~31u) == ep) return;
      const u32 nc = comp_alloc();
      u32 head = 0, tail = 0;
      g.m.w(g.L.bfs_q + tail++) = q;
      g.m.w(g.L.stamp + q) = ep;
      u32 cost = 0, mx = 0, nm = 0, list = NONE, size = 0;
      while (head < tail) {
        u32 x = g.m.w(g.L.bfs_q + head++);
        const uint4 sx = g.srec(x);
        const uint4 ax = g.arec(x);
        g.state(x) = O_BIT | nc;
        g.m.w(g.L.mem_next + x) = list;
        g.m.w(g.L.mem_prev + x) = NONE;
        if (list != NONE) g.m.w(g.L.mem_prev + list) = x;
        list = x;
        size++;
        cost += sx.y;
        if (sx.z > mx) { mx = sx.z; nm = 1; } else if (sx.z == mx) nm++;
        g.for_each_nbr(x, ax, [&](u32 y) {
          if (is_evicted(g.state(y)) && (g.m.w(g.L.stamp + y) & ~31u) != ep) {
            g.m.w(g.L.stamp + y) = ep;
            g.m.w(g.L.bfs_q + tail++) = y;
          }
        });
      }
      g.m.w(g.L.comp_head + nc) = list;
      g.comp(nc) = make_uint4(cost, nm, mx, size);
    });
  }

  // V2 release of an evicted tensor: its la dropped from `old` to -inf (0)
  __device__ __forceinline__ void lower_maxla_exact(u32 t, u32 old) {
    const u32 c = g.state(t) & COMP_MASK;
    uint4 cc = g.comp(c);
    if (old != cc.z || old == 0) return;
    if (--cc.y == 0) { const uint2 r = comp_rescan_maxla(c); cc.z = r.x; cc.y = r.y; }
    g.comp(c) = cc;
  }

  // ------------------------------------------------------------- union-find
  __device__ __forceinline__ u32 uf_find(u32 x) {   // path halving
    u32 p = g.uf(x).w;
    while (p != x) {
      u32 gp = g.uf(p).w;
      g.uf(x).w = gp;
      x = gp;
      p = g.uf(x).w;
    }
    return x;
  }
  __device__ __forceinline__ void uf_union(u32 a, u32 b) {
    a = uf_find(a); b = uf_find(b);
    if (a == b) return;
    u32 sa = g.m.w(g.L.uf_size + a), sb = g.m.w(g.L.uf_size + b);
    if (sa < sb) { u32 x = a; a = b; b = x; }
    uint4 ra = g.uf(a), rb = g.uf(b);
    g.uf(b).w = a;
    g.m.w(g.L.uf_size + a) = sa + sb;
    u64 cost = mk64(ra.x, ra.y) + mk64(rb.x, rb.y);
    g.uf(a) = make_uint4((u32)cost, (u32)(cost >> 32), ra.z > rb.z ? ra.z : rb.z, a);
  }
  // Nodes are only referenced through node_of[] of evicted tensors.  When the
  // node array is full, renumber the live roots in place, in increasing old id
  // (new id <= old id, so no live record is overwritten before it moves): the
  // sets, their cost and maxla -- all the heuristic reads -- are unchanged.
  __device__ __forceinline__ void uf_compact() {
    const u32 SZ = g.L.uf_size;
    for (u32 q = 0; q < s.n_alloc; q++) {              // point every evicted tensor at its root
      if (!is_evicted(g.state(q))) continue;
      u32 x = g.m.w(g.L.node_of + q);
      if (x == NONE) continue;
      u32 r = uf_find(x);
      g.m.w(g.L.node_of + q) = r;
      g.m.w(SZ + r) = 1u | LIVE_BIT;                   // recount sizes below
    }
    u32 k = 0;
    for (u32 i = 0; i < s.uf_n; i++) {                 // new ids, stored in the parent field
      if (g.m.w(SZ + i) & LIVE_BIT) { g.uf(i).w = k++; }
    }
    for (u32 q = 0; q < s.n_alloc; q++) {
      if (!is_evicted(g.state(q))) continue;
      u32 r = g.m.w(g.L.node_of + q);
      if (r == NONE) continue;
      g.m.w(g.L.node_of + q) = g.uf(r).w;
    }
    u32 j = 0;
    for (u32 i = 0; i < s.uf_n; i++) {
      if (!(g.m.w(SZ + i) & LIVE_BIT)) continue;
      uint4 r = g.uf(i);
      g.uf(j) = make_uint4(r.x, r.y, r.z, j);
      g.m.w(SZ + j) = 1;
      j++;
    }
    s.uf_n = k;
  }
  __device__ __forceinline__ u32 uf_alloc() {
    if (s.uf_n == g.L.uf_cap) uf_compact();
    return s.uf_n++;
  }
  // "When a tensor t is evicted, its component is unioned with those of any
  // evicted neighbors and c0(t) is added to the component's running sum"
  // (fused: every neighbour's nev += 1)
  __device__ __forceinline__ void evict_uf(u32 t, const uint4 &sr, const uint4 &ar) {
    u32 n0 = uf_alloc();
    g.uf(n0) = make_uint4(sr.y, 0, sr.z, n0);
    g.m.w(g.L.uf_size + n0) = 1;
    g.m.w(g.L.node_of + t) = n0;
    g.for_each_nbr(t, ar, [&](u32 q) {
      g.nev(q) += 1;
      if (g.L.lcache) g.m.w(g.L.lcache + q) = 0;        // q's evicted neighbourhood changed
      if (is_evicted(g.state(q))) uf_union(n0, g.m.w(g.L.node_of + q));
    });
  }
  // "subtract c0(t) from its component's running sum and map t to a new
  // (empty) union-find component"
  __device__ __forceinline__ void remat_uf(u32 t, u32 cost_t) {
    u32 r = uf_find(g.m.w(g.L.node_of + t));
    uint4 rr = g.uf(r);
    u64 cost = mk64(rr.x, rr.y) - cost_t;
    g.uf(r).x = (u32)cost;
    g.uf(r).y = (u32)(cost >> 32);
    g.m.w(g.L.node_of + t) = NONE;
  }

  // la(p) of an evicted p rose from old to v (make_tensor of a child)
  __device__ __forceinline__ void raise_maxla(u32 p, u32 sp, u32 old, u32 v) {
    if (s.heuristic == H_DTR) {
      if (v == old) return;
      const u32 c = sp & COMP_MASK;
      uint4 cc = g.comp(c);
      if (v > cc.z) { cc.z = v; cc.y = 1; }
      else if (v == cc.z) cc.y++;
      else return;                        // v < max: old < v < max, the holders are unchanged
      g.comp(c) = cc;
    } else if (uses_uf(s.heuristic)) {
      u32 r = uf_find(g.m.w(g.L.node_of + p));
      if (v > g.uf(r).z) g.uf(r).z = v;
    }
  }

  // ------------------------------------------------------------- closure-cache events
  // t's evicted status flipped: queue it for the team's invalidation walk
  __device__ __forceinline__ void ev_push(u32 t) {
    if (!g.L.ccache) return;
    const u32 k = s.ev_n;
    if (k < EVQ_CAP) g.m.w(g.L.evq + k) = t;
    if (k <= EVQ_CAP) s.ev_n = k + 1;
  }

  // ------------------------------------------------------------- evict
  __device__ __forceinline__ void evict(u32 t) {
    const uint4 sr = g.srec(t);
    const uint4 ar = g.arec(t);
    ev_push(t);
    g.mirror_bit(t, true);
    g.state(t) = O_BIT;
    s.M -= sr.x;
    pool_remove(t);
    if (s.heuristic == H_DTR) evict_exact(t, sr, ar);
    else if (uses_uf(s.heuristic)) evict_uf(t, sr, ar);
    else nev_add(t, ar, 1u);
  }

  __device__ __forceinline__ void fnv(u64 v) { s.trace_hash = (s.trace_hash ^ v) * 1099511628211ull; }

  __device__ __forceinline__ void record_and_evict(const Cand &c) {
    if (trace && s.trace_n < s.trace_cap) {
      dtr_evict_rec r;
      r.clock = s.clock; r.id = c.id; r.pad = 0; r.num = c.num; r.den = c.den;
      trace[s.trace_n] = r;
      s.trace_n++;
    }
    fnv(s.clock); fnv(c.id); fnv(c.num); fnv(c.den);
    s.decisions++;
    evict(c.id);
  }

  // ------------------------------------------------------------- get_internal stack
  // frame k: fr[k] = {t, pb_base, pb_count, next}
  __device__ __forceinline__ void push(u32 t, const uint2 &pr) {
    u32 base = s.pb_top;
    for (u32 j = 0; j < pr.y; j++) {           // P_T locked now, P_B kept in order (reading C-6)
      u32 p = g.par(pr.x + j);
      if (is_material(g.state(p))) lock(p);
      else g.m.w(g.L.pb + s.pb_top++) = p;
    }
    g.m.q(g.L.fr + 4 * s.sp) = make_uint4(t, base, s.pb_top - base, 0);
    s.sp++;
  }
  __device__ __forceinline__ void start_gi(u32 t) {
    if (is_material(g.state(t))) lock(t);
    else push(t, g.prec(t));
  }

  __device__ __forceinline__ u32 stop(u32 st) {
    s.status = st;
    s.last_rc = st;
    phase = PH_DONE;
    return CMD_DONE;
  }

  // compute the top frame's tensor (its parents are all resident and locked,
  // and M + mem <= B): lines 234-240 of get_internal. Returns false on stop.
  __device__ __forceinline__ bool complete_top(u32 t, const uint4 &fr) {
    const uint4 sr = g.srec(t);
    const uint4 ar = g.arec(t);
    u32 st = g.state(t);
    g.state(t) = M_BIT | O_BIT;
    g.ell(t) = 1;
    s.M += sr.x;
    if (s.M > s.peak_M) s.peak_M = s.M;
    s.clock += sr.y;
    s.computations++;
    if (st & O_BIT) {
      s.remats++;
      ev_push(t);
      g.mirror_bit(t, false);
      nev_add(t, ar, NONE);
      if (s.heuristic == H_DTR) remat_exact(t, ar, st & COMP_MASK);
      else if (uses_uf(s.heuristic)) remat_uf(t, sr.y);
    } else {
      // first computation: every parent is resident and no child exists yet
      if (g.L.track_nev) g.nev(t) = 0;
      if (g.L.linked) {
        // t becomes a visible child of its parents (reading C-19)
        for (u32 j = 0; j < ar.y; j++) {
          u32 p = g.par(ar.x + j);
          u32 x = s.edges_used++;
          g.m.w(g.L.e_child + x) = t;
          g.m.w(g.L.e_next + x) = g.crec(p).x;
          g.crec(p).x = x;
        }
      }
    }
    if (s.clock > s.kill_limit) {                // one compare: kill_limit = min(kill x base, CLOCK_LIMIT)
      stop(s.clock > CLOCK_LIMIT ? ST_CAPACITY : ST_THRASH);
      return false;
    }
    for (u32 j = 0; j < ar.y; j++) release_internal(g.par(ar.x + j));
    s.pb_top = fr.y;
    s.sp--;
    return true;
  }

  __device__ __forceinline__ void finish_op() {
    if (post) release_internal(root);
    post = 0;
    s.records_done++;
    s.last_rc = ST_OK;
    op_idx++;
  }

  // precondition violation: per-call -> report, no state change; batch -> stop
  __device__ __forceinline__ bool precond() {
    if (percall) { s.last_rc = ST_PRECOND; op_idx++; return true; }
    stop(ST_PRECOND);
    return false;
  }

  // ------------------------------------------------------------- the state machine
  __device__ __forceinline__ u32 resume(bool have, const Cand &res) {
    if (phase == PH_FREE && have) {
      PROF_T(p0);
      record_and_evict(res);
      PROF_T(p1);
      PROF_ADD(8, p1 - p0); PROF_ADD(9, 1);
    }
    if (phase == PH_SCORED) { finish_op(); phase = PH_OP; }
    for (;;) {
      if (phase == PH_GI || phase == PH_FREE) {
        PROF_ADD(14, 1);
        if (s.sp == 0) { finish_op(); phase = PH_OP; continue; }
        const u32 k = s.sp - 1;
        uint4 fr = g.m.q(g.L.fr + 4 * k);
        if (phase == PH_GI && fr.w < fr.z) {
          g.m.w(g.L.fr + 4 * k + 3) = fr.w + 1;
          u32 p = g.m.w(g.L.pb + fr.y + fr.w);
          PROF_T(u0);
          if (is_material(g.state(p))) lock(p);
          else push(p, g.prec(p));
          PROF_T(u1);
          PROF_ADD(12, u1 - u0); PROF_ADD(13, 1);
          continue;
        }
        u32 t = fr.x;
        u64 need = phase == PH_FREE ? free_size : g.srec(t).x;
        if (s.M + need > s.B) {
          phase = PH_FREE; free_size = need;
          if (s.decisions >= s.max_decisions) return stop(ST_DECISION_CAP);   // 0 = none, normalised to ~0
          if (s.pool_size == 0) return stop(ST_OOM);
          return CMD_ARGMIN;
        }
        phase = PH_GI;
        PROF_T(c0);
        if (!complete_top(t, fr)) return CMD_DONE;
        PROF_T(c1);
        PROF_ADD(10, c1 - c0); PROF_ADD(11, 1);
        continue;
      }
      if (phase == PH_DONE) return CMD_DONE;
      // PH_OP
      if (op_idx >= op_end) return CMD_DONE;
      const u32 word = percall ? s.pending_op : ops[op_idx];
      const u32 op = word >> 29, id = word & ((1u << 29) - 1);
      if (op == OP_MAKE) {
        if (id != s.n_alloc || id >= g.L.n) { if (!precond()) return CMD_DONE; continue; }
        const u32 cost = g.srec(id).y;
        const uint2 pr = g.prec(id);
        bool ok = true;
        for (u32 j = 0; j < pr.y; j++) if (g.rho(g.par(pr.x + j)) == 0) ok = false;   // reading C-12
        if (!ok) { if (!precond()) return CMD_DONE; continue; }
        s.base_so_far += cost;
        s.kill_limit = s.thrash_kill && (u64)s.thrash_kill * s.base_so_far < CLOCK_LIMIT
                           ? (u64)s.thrash_kill * s.base_so_far : CLOCK_LIMIT;
        const u32 now = (u32)(s.clock + 1);
        g.state(id) = 0;
        g.la(id) = now;
        g.rho(id) = 1;
        g.ell(id) = 0;
        if constexpr (!BM) g.pool_pos(id) = NONE;
        if (uses_uf(s.heuristic)) g.m.w(g.L.node_of + id) = NONE;
        if (g.L.linked) g.crec(id) = make_uint2(NONE, 0);
        for (u32 j = 0; j < pr.y; j++) {          // p.C u= {t}; p.last_accessed := clock
          u32 p = g.par(pr.x + j);
          const u32 old = g.la(p);
          g.la(p) = now;
          pool_rekey(p);
          u32 sp = g.state(p);
          if (is_evicted(sp)) raise_maxla(p, sp, old, now);
        }
        s.n_alloc++;
        root = id; post = 1;
        push(id, pr);
        phase = PH_GI;
        continue;
      }
      if (op == OP_GET) {
        if (id >= s.n_alloc || g.rho(id) == 0) { if (!precond()) return CMD_DONE; continue; }
        g.rho(id)++;
        finish_op();
        continue;
      }
      if (op == OP_RELEASE) {
        if (id >= s.n_alloc || g.rho(id) == 0) { if (!precond()) return CMD_DONE; continue; }
        u32 r = g.rho(id) - 1;
        g.rho(id) = r;
        if (r == 0) {
          if (s.dealloc == DEALLOC_V2) {              // banish_V2
            u32 old = g.la(id);
            g.la(id) = 0;
            pool_rekey(id);
            if (s.heuristic == H_DTR && is_evicted(g.state(id))) lower_maxla_exact(id, old);
          } else if (s.dealloc == DEALLOC_V1) {
            maybe_banish(id);
          } else if (s.dealloc == DEALLOC_EAGER) {   // evict normally if possible
            if (pool_has(id)) evict(id);
          }
        }
        finish_op();
        continue;
      }
      if (op == OP_REMAT || op == OP_ENSURE) {
        u32 st = id < s.n_alloc ? g.state(id) : 0;
        bool bad = op == OP_REMAT ? !is_evicted(st) : (!(st & O_BIT) || is_banished(st));
        if (id >= s.n_alloc || bad) { if (!precond()) return CMD_DONE; continue; }
        root = id; post = op == OP_REMAT;
        start_gi(id);
        phase = PH_GI;
        continue;
      }
      if (op == OP_DEBUG_EVICT) {
        if (id >= s.n_alloc || !pool_has(id)) { if (!precond()) return CMD_DONE; continue; }
        evict(id);
        finish_op();
        continue;
      }
      if (op == OP_SCORES) { phase = PH_SCORED; return CMD_SCORES; }
      if (!precond()) return CMD_DONE;
    }
  }
};

}  // namespace dtr
