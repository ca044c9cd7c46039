// leader.cuh -- the sequential control of one simrd simulation, run by ONE
// leader thread as a resumable state machine (explicit get_internal stack).
//
//   make_tensor     P:327-343        get_internal   P:213-245 (depth-first)
//   release_internal P:247-259       evict
//   free            P:273-284        banish_V2
//   get / release / rematerialize
//   union-find evicted components with approximate split (h_DTR_eq)
//                                    P:1236-1250
//   exact evicted components (h_DTR: E(t) of P:63-68 as the union of the
//   components adjacent to t, maintained incrementally: merge on evict,
//   split by BFS on rematerialization)
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
  u32 kind, pool_size, heur, pad;
};

struct Leader {
  Graph *g;
  Work *w;
  Scalars *s;             // the leader's working copy (shared memory)
  dtr_evict_rec *trace;   // cell's trace region (may be null)
  u32 op_idx, op_end;
  u32 phase, post, root;
  u32 percall;
  u64 free_size;

  // ------------------------------------------------------------- pool
  __device__ void pool_add(u32 t) {
    u32 k = s->pool_size++;
    w->pool_pos[t] = k;
    w->pool_ids[k] = t;
  }
  __device__ void pool_remove(u32 t) {
    u32 p = w->pool_pos[t];
    if (p == NONE) return;
    u32 last = w->pool_ids[--s->pool_size];
    w->pool_ids[p] = last;
    w->pool_pos[last] = p;
    w->pool_pos[t] = NONE;
  }
  // get_internal branch "t.m = T": l++, pool \ {t}
  __device__ void lock(u32 t) {
    if (w->ell[t] == 0) pool_remove(t);
    w->ell[t]++;
  }
  // release_internal, V2
  __device__ void release_internal(u32 t) {
    if (--w->ell[t] == 0) pool_add(t);
  }

  // ------------------------------------------------------------- exact components
  __device__ u32 comp_alloc() { return w->comp_free[--s->comp_free_top]; }
  __device__ void comp_release(u32 c) { w->comp_free[s->comp_free_top++] = c; }

  __device__ u32 comp_merge(u32 a, u32 b) {
    if (w->comp_size[a] < w->comp_size[b]) { u32 x = a; a = b; b = x; }
    u32 x = w->comp_head[b], last = NONE;
    while (x != NONE) { w->state[x] = O_BIT | a; last = x; x = w->mem_next[x]; }
    w->mem_next[last] = w->comp_head[a];
    w->comp_head[a] = w->comp_head[b];
    w->comp_size[a] += w->comp_size[b];
    w->comp_cost[a] += w->comp_cost[b];
    if (w->comp_maxla[b] > w->comp_maxla[a]) w->comp_maxla[a] = w->comp_maxla[b];
    comp_release(b);
    return a;
  }

  // t has just become evicted: {t} joins the components of its evicted neighbours.
  __device__ void evict_exact(u32 t) {
    u32 c = comp_alloc();
    w->comp_cost[c] = g->cost[t];
    w->comp_maxla[c] = w->la[t];
    w->comp_head[c] = t;
    w->comp_size[c] = 1;
    w->mem_next[t] = NONE;
    w->state[t] = O_BIT | c;
    u32 cur = c;
    for_each_nbr(*g, t, [&](u32 q) {
      u32 sq = w->state[q];
      if (!is_evicted(sq)) return;
      u32 cq = sq & COMP_MASK;
      if (cq != cur) cur = comp_merge(cur, cq);
    });
  }

  // t (formerly in component c) has just become material: relabel c \ {t} by
  // BFS from t's evicted neighbours; each BFS tree is one new component.
  __device__ void remat_exact(u32 t, u32 c) {
    comp_release(c);
    if (w->comp_size[c] == 1) return;
    u32 ep = ++s->epoch;
    for_each_nbr(*g, t, [&](u32 q) {
      u32 sq = w->state[q];
      if (!is_evicted(sq) || w->stamp[q] == ep) return;
      u32 nc = comp_alloc();
      u32 head = 0, tail = 0;
      w->bfs_q[tail++] = q;
      w->stamp[q] = ep;
      u64 cost = 0;
      u32 mx = 0, list = NONE, size = 0;
      while (head < tail) {
        u32 x = w->bfs_q[head++];
        w->state[x] = O_BIT | nc;
        w->mem_next[x] = list;
        list = x;
        size++;
        cost += g->cost[x];
        u32 lx = w->la[x];
        mx = lx > mx ? lx : mx;
        for_each_nbr(*g, x, [&](u32 y) {
          if (is_evicted(w->state[y]) && w->stamp[y] != ep) { w->stamp[y] = ep; w->bfs_q[tail++] = y; }
        });
      }
      w->comp_head[nc] = list;
      w->comp_size[nc] = size;
      w->comp_cost[nc] = cost;
      w->comp_maxla[nc] = mx;
    });
  }

  // V2 release of an evicted tensor: its la dropped to -inf; rescan the max if it was the max.
  __device__ void lower_maxla_exact(u32 t, u32 old) {
    u32 c = w->state[t] & COMP_MASK;
    if (old != w->comp_maxla[c]) return;
    u32 mx = 0;
    for (u32 x = w->comp_head[c]; x != NONE; x = w->mem_next[x]) { u32 l = w->la[x]; mx = l > mx ? l : mx; }
    w->comp_maxla[c] = mx;
  }

  // ------------------------------------------------------------- union-find
  __device__ u32 uf_find(u32 x) {   // path halving
    while (w->uf_parent[x] != x) {
      u32 gp = w->uf_parent[w->uf_parent[x]];
      w->uf_parent[x] = gp;
      x = gp;
    }
    return x;
  }
  __device__ void uf_union(u32 a, u32 b) {
    a = uf_find(a); b = uf_find(b);
    if (a == b) return;
    if (w->uf_size[a] < w->uf_size[b]) { u32 x = a; a = b; b = x; }
    w->uf_parent[b] = a;
    w->uf_size[a] += w->uf_size[b];
    w->uf_cost[a] += w->uf_cost[b];
    if (w->uf_maxla[b] > w->uf_maxla[a]) w->uf_maxla[a] = w->uf_maxla[b];
  }
  // Nodes are only referenced through node_of[] of evicted tensors; when the
  // node array is full, renumber the live roots compactly (same sets, same
  // cost / maxla: the heuristic reads nothing else).
  __device__ void uf_compact() {
    u32 k = 0;
    for (u32 q = 0; q < s->n_alloc; q++) {
      if (!is_evicted(w->state[q]) || w->node_of[q] == NONE) continue;
      u32 r = uf_find(w->node_of[q]);
      u32 nk = w->uf_remap[r];
      if (nk == NONE) {
        nk = k++;
        w->uf_remap[r] = nk;
        w->uf_roots[nk] = r;
        w->uf_tcost[nk] = w->uf_cost[r];
        w->uf_tmaxla[nk] = w->uf_maxla[r];
        w->uf_tsize[nk] = 0;
      }
      w->uf_tsize[nk]++;
      w->node_of[q] = nk;
    }
    for (u32 i = 0; i < k; i++) {
      w->uf_remap[w->uf_roots[i]] = NONE;
    }
    for (u32 i = 0; i < k; i++) {
      w->uf_parent[i] = i;
      w->uf_cost[i] = w->uf_tcost[i];
      w->uf_maxla[i] = w->uf_tmaxla[i];
      w->uf_size[i] = w->uf_tsize[i];
    }
    s->uf_n = k;
  }
  __device__ u32 uf_alloc() {
    if (s->uf_n == s->uf_cap) uf_compact();
    return s->uf_n++;
  }
  // "When a tensor t is evicted, its component is unioned with those of any
  // evicted neighbors and c0(t) is added to the component's running sum"
  __device__ void evict_uf(u32 t) {
    u32 n0 = uf_alloc();
    w->uf_parent[n0] = n0;
    w->uf_cost[n0] = g->cost[t];
    w->uf_maxla[n0] = w->la[t];
    w->uf_size[n0] = 1;
    w->node_of[t] = n0;
    for_each_nbr(*g, t, [&](u32 q) {
      if (is_evicted(w->state[q])) uf_union(n0, w->node_of[q]);
    });
  }
  // "subtract c0(t) from its component's running sum and map t to a new
  // (empty) union-find component"
  __device__ void remat_uf(u32 t) {
    u32 r = uf_find(w->node_of[t]);
    w->uf_cost[r] -= g->cost[t];
    w->node_of[t] = NONE;
  }

  __device__ void raise_maxla(u32 p, u32 sp, u32 v) {
    if (s->heuristic == H_DTR) {
      u32 c = sp & COMP_MASK;
      if (v > w->comp_maxla[c]) w->comp_maxla[c] = v;
    } else if (s->heuristic == H_DTR_EQ) {
      u32 r = uf_find(w->node_of[p]);
      if (v > w->uf_maxla[r]) w->uf_maxla[r] = v;
    }
  }

  // ------------------------------------------------------------- evict
  __device__ void evict(u32 t) {
    w->state[t] = O_BIT;
    s->M -= g->mem[t];
    pool_remove(t);
    if (s->heuristic == H_DTR) evict_exact(t);
    else if (s->heuristic == H_DTR_EQ) evict_uf(t);
  }

  __device__ void fnv(u64 v) { s->trace_hash = (s->trace_hash ^ v) * 1099511628211ull; }

  __device__ void record_and_evict(const Cand &c) {
    if (trace && s->trace_n < s->trace_cap) {
      dtr_evict_rec *r = &trace[s->trace_n];
      r->clock = s->clock; r->id = c.id; r->pad = 0; r->num = c.num; r->den = c.den;
      s->trace_n++;
    }
    fnv(s->clock); fnv(c.id); fnv(c.num); fnv(c.den);
    s->decisions++;
    evict(c.id);
  }

  // ------------------------------------------------------------- get_internal stack
  __device__ void push(u32 t) {
    u32 base = s->pb_top;
    u32 b = g->par_off[t], e = g->par_off[t + 1];
    for (u32 j = b; j < e; j++) {           // P_T locked now, P_B kept in order (reading C-6)
      u32 p = g->par[j];
      if (is_material(w->state[p])) lock(p);
      else w->pb[s->pb_top++] = p;
    }
    u32 k = s->sp++;
    w->fr_t[k] = t;
    w->fr_base[k] = base;
    w->fr_cnt[k] = s->pb_top - base;
    w->fr_next[k] = 0;
  }
  __device__ void start_gi(u32 t) {
    if (is_material(w->state[t])) lock(t);
    else push(t);
  }

  __device__ u32 stop(u32 st) {
    s->status = st;
    s->last_rc = st;
    phase = PH_DONE;
    return CMD_DONE;
  }

  // compute the top frame's tensor (its parents are all resident and locked,
  // and M + mem <= B): lines 234-240 of get_internal. Returns false on stop.
  __device__ bool complete_top() {
    u32 k = s->sp - 1;
    u32 t = w->fr_t[k];
    u32 st = w->state[t];
    w->state[t] = M_BIT | O_BIT;
    w->ell[t] = 1;
    s->M += g->mem[t];
    if (s->M > s->peak_M) s->peak_M = s->M;
    s->clock += g->cost[t];
    s->computations++;
    if (st & O_BIT) {
      s->remats++;
      if (s->heuristic == H_DTR) remat_exact(t, st & COMP_MASK);
      else if (s->heuristic == H_DTR_EQ) remat_uf(t);
    } else if (g->linked) {
      // first computation: t becomes a visible child of its parents (reading C-19)
      u32 b = g->par_off[t], e = g->par_off[t + 1];
      for (u32 j = b; j < e; j++) {
        u32 p = g->par[j];
        u32 x = s->edges_used++;
        w->e_child[x] = t;
        w->e_next[x] = w->ch_head[p];
        w->ch_head[p] = x;
      }
    }
    if (s->clock > CLOCK_LIMIT) { stop(ST_CAPACITY); return false; }
    if (s->thrash_kill && s->clock > (u64)s->thrash_kill * s->base_so_far) { stop(ST_THRASH); return false; }
    u32 b = g->par_off[t], e = g->par_off[t + 1];
    for (u32 j = b; j < e; j++) release_internal(g->par[j]);
    s->pb_top = w->fr_base[k];
    s->sp = k;
    return true;
  }

  __device__ void finish_op() {
    if (post) release_internal(root);
    post = 0;
    s->records_done++;
    s->last_rc = ST_OK;
    op_idx++;
  }

  // precondition violation: per-call -> report, no state change; batch -> stop
  __device__ bool precond() {
    if (percall) { s->last_rc = ST_PRECOND; op_idx++; return true; }
    stop(ST_PRECOND);
    return false;
  }

  // ------------------------------------------------------------- the state machine
  __device__ u32 resume(bool have, const Cand &res) {
    if (phase == PH_FREE && have) record_and_evict(res);
    if (phase == PH_SCORED) { finish_op(); phase = PH_OP; }
    for (;;) {
      switch (phase) {
        case PH_DONE:
          return CMD_DONE;
        case PH_FREE:
          if (s->M + free_size > s->B) {
            if (s->max_decisions && s->decisions >= s->max_decisions) return stop(ST_DECISION_CAP);
            if (s->pool_size == 0) return stop(ST_OOM);
            return CMD_ARGMIN;
          }
          phase = PH_GI;
          if (!complete_top()) return CMD_DONE;
          break;
        case PH_GI: {
          if (s->sp == 0) { finish_op(); phase = PH_OP; break; }
          u32 k = s->sp - 1;
          u32 nx = w->fr_next[k];
          if (nx < w->fr_cnt[k]) {
            w->fr_next[k] = nx + 1;
            u32 p = w->pb[w->fr_base[k] + nx];
            if (is_material(w->state[p])) lock(p);
            else push(p);
            break;
          }
          u32 t = w->fr_t[k];
          if (s->M + g->mem[t] > s->B) { phase = PH_FREE; free_size = g->mem[t]; break; }
          if (!complete_top()) return CMD_DONE;
          break;
        }
        case PH_OP: {
          if (op_idx >= op_end) return CMD_DONE;
          u32 word = percall ? s->pending_op : g->ops[op_idx];
          u32 op = word >> 29, id = word & ((1u << 29) - 1);
          switch (op) {
            case OP_MAKE: {
              if (id != s->n_alloc || id >= g->n) { if (!precond()) return CMD_DONE; break; }
              u32 b = g->par_off[id], e = g->par_off[id + 1];
              bool ok = true;
              for (u32 j = b; j < e; j++) if (w->rho[g->par[j]] == 0) ok = false;   // reading C-12
              if (!ok) { if (!precond()) return CMD_DONE; break; }
              s->base_so_far += g->cost[id];
              u32 now = (u32)(s->clock + 1);
              w->la[id] = now;
              w->rho[id] = 1;
              w->ell[id] = 0;
              w->state[id] = 0;
              w->pool_pos[id] = NONE;
              if (s->heuristic == H_DTR_EQ) w->node_of[id] = NONE;
              if (g->linked) w->ch_head[id] = NONE;
              for (u32 j = b; j < e; j++) {          // p.C u= {t}; p.last_accessed := clock
                u32 p = g->par[j];
                w->la[p] = now;
                u32 sp = w->state[p];
                if (is_evicted(sp)) raise_maxla(p, sp, now);
              }
              s->n_alloc++;
              root = id; post = 1;
              start_gi(id);
              phase = PH_GI;
              break;
            }
            case OP_GET:
              if (id >= s->n_alloc || w->rho[id] == 0) { if (!precond()) return CMD_DONE; break; }
              w->rho[id]++;
              finish_op();
              break;
            case OP_RELEASE: {
              if (id >= s->n_alloc || w->rho[id] == 0) { if (!precond()) return CMD_DONE; break; }
              if (--w->rho[id] == 0) {               // banish_V2
                u32 old = w->la[id];
                w->la[id] = 0;
                if (s->heuristic == H_DTR && is_evicted(w->state[id])) lower_maxla_exact(id, old);
              }
              finish_op();
              break;
            }
            case OP_REMAT: {
              u32 st = id < s->n_alloc ? w->state[id] : 0;
              if (id >= s->n_alloc || !is_evicted(st)) { if (!precond()) return CMD_DONE; break; }
              root = id; post = 1;
              start_gi(id);
              phase = PH_GI;
              break;
            }
            case OP_ENSURE: {
              u32 st = id < s->n_alloc ? w->state[id] : 0;
              if (id >= s->n_alloc || !(st & O_BIT)) { if (!precond()) return CMD_DONE; break; }
              root = id; post = 0;
              start_gi(id);
              phase = PH_GI;
              break;
            }
            case OP_DEBUG_EVICT:
              if (id >= s->n_alloc || w->pool_pos[id] == NONE) { if (!precond()) return CMD_DONE; break; }
              evict(id);
              finish_op();
              break;
            case OP_SCORES:
              phase = PH_SCORED;
              return CMD_SCORES;
            default:
              if (!precond()) return CMD_DONE;
          }
          break;
        }
      }
    }
  }
};

}  // namespace dtr
