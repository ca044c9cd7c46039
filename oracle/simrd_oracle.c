/*
 * oracle/simrd_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  The CUDA path
 * (paper_2006_09616_b200/) never includes, links or calls anything here, and
 * this file includes nothing from it: the two share no code.
 *
 * A plain, slow, single-threaded CPU implementation of the simrd runtime with
 * V2 banishing, written line by line from PAPER.md (Doc A, the simrd spec):
 *
 *   tensor tuple t = (P, C, I, m, rho, l)
 *   heuristic metadata I = (mem, compute, last_access)
 *   evicted neighbourhood E(t) (undirected)
 *   staleness                                             P:83-94  (difference form, reading C-2)
 *   h_DTR
 *   runtime state clock / pool / M / B
 *   get_internal / release_internal / evict / free
 *   banish_V2
 *   rematerialize / make_tensor / get / release
 * plus the paper's heuristic variants (Doc C):
 *   h_DTR_eq with the union-find relaxation and split
 *   h_LRU, h_largest ("size"), h_MSPS
 *   h_DTR_local
 *   h_rand                                                P:1269-1270 (reading C-15)
 *   h_DTR_full over the DIRECTED e*(t) (ancestors and descendants reached
 *     through evicted tensors), own staleness
 *   h_e* "compute-memory" = (c(t) + c0) / m (Theorem 1)
 *   the ablation h'(s, m, c)(t) = c(t) / [m(t) s(t)]      P:2527-2536 (reading C-23)
 *
 * Readings of silent / ambiguous points are DESIGN.md's C-1 ... C-19; each is
 * cited where it is applied.  Scores are exact rationals (num, den) of
 * integers compared by 128-bit cross multiplication (reading C-5, C-14).
 *
 * Parity pins for every function here live in tests/test_oracle_*.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ---- status codes (the boundary's values, restated independently) ---- */
enum {
  OR_OK = 0, OR_PRECOND = 2, OR_OOM = 3, OR_THRASH = 4, OR_CAPACITY = 5,
  OR_STATE = 6, OR_DECISION_CAP = 8
};
/* ---- heuristic ids (the boundary's values) ---- */
enum { H_DTR = 0, H_DTR_EQ = 1, H_LRU = 2, H_SIZE = 3, H_MSPS = 4, H_LOCAL = 5, H_RANDOM = 6,
       H_DTR_FULL = 7, H_ESTAR = 8 };
/* the D.1 ablation h'(s, m, c): id = H_ABL + 4*c + 2*m + s with
 * c in {0: e*, 1: EqClass (e~*), 2: local, 3: no}, m, s in {0: no, 1: yes} (reading C-23) */
enum { H_ABL = 16, H_ABL_END = 32 };
enum { ABL_C_ESTAR = 0, ABL_C_EQCLASS = 1, ABL_C_LOCAL = 2, ABL_C_NO = 3 };
static int is_abl(int h) { return h >= H_ABL && h < H_ABL_END; }
/* heuristics that keep the union-find evicted components */
static int uses_uf(int h) { return h == H_DTR_EQ || (is_abl(h) && ((h - H_ABL) >> 2) == ABL_C_EQCLASS); }
/* ---- deallocation policies ---- */
enum { DEALLOC_V2 = 0, DEALLOC_V1 = 1, DEALLOC_EAGER = 2, DEALLOC_IGNORE = 3 };
/* ---- log opcodes (dtr_inputs/logfmt.py) ---- */
enum { OP_MAKE = 1, OP_GET = 2, OP_RELEASE = 3, OP_REMAT = 4, OP_ENSURE = 5, OP_DEBUG_EVICT = 6 };

#define NEG_INF INT64_MIN            /* last_access := -infinity (banish_V2) */
#define CLOCK_LIMIT 0xFFFFFFFEull    /* reading C-14: clock must stay < 2^32 - 1 */

typedef struct { uint64_t clock; uint32_t id; uint32_t pad; uint64_t num, den; } or_trace_rec;

typedef struct {
  uint32_t cell_id, status, records_done, n_trace;
  uint64_t clock, base, decisions, remats, computations, peak_M, trace_hash;
} or_result;

typedef struct { uint32_t *v; uint32_t n, cap; } vec32;

static void vpush(vec32 *a, uint32_t x) {
  if (a->n == a->cap) { a->cap = a->cap ? 2 * a->cap : 4; a->v = (uint32_t *)realloc(a->v, a->cap * sizeof(uint32_t)); }
  a->v[a->n++] = x;
}

static void vremove(vec32 *a, uint32_t x) {
  for (uint32_t i = 0; i < a->n; i++)
    if (a->v[i] == x) { memmove(&a->v[i], &a->v[i + 1], (a->n - i - 1) * sizeof(uint32_t)); a->n--; return; }
}

/* One union-find node: parent pointer, running cost sum, and the
 * max last_access of the set (reading C-9); size = nodes in the tree below it
 * (union by size keeps find O(log n); it shapes the tree, not the sets). */
typedef struct { uint64_t parent; uint64_t cost; int64_t maxla; uint64_t size; } uf_node;

typedef struct {
  /* configuration */
  int heuristic;
  uint64_t B;                 /* R.B */
  uint64_t seed;
  uint32_t thrash_kill;       /* reading C-13: abort when clock > kill * base_so_far */
  uint64_t max_decisions;     /* bounded samples: stop after this many decisions */
  int e_mode;                 /* 0: label evicted components once per decision; 1: literal BFS per candidate */
  int dealloc;                /* DEALLOC_*: what release() does at rho = 0 */

  /* tensors t = (P, C, I, m, rho, l) */
  uint32_t n, cap;
  vec32 *P, *C;
  uint64_t *mem, *compute;
  int64_t *last_access;
  uint8_t *m;                 /* materialized */
  uint8_t *computed_once;     /* reading C-19: evicted(x) := !m[x] && computed_once[x] */
  uint64_t *rho, *l;
  uint8_t *in_pool;           /* R.pool as a membership set over tensor ids */
  uint8_t *banished;          /* V1: permanently evicted and removed from the graph */

  /* union-find for h_DTR_eq */
  uint64_t *set_of;           /* T.set: the UF node of each tensor */
  uf_node *uf; uint64_t uf_n, uf_cap;

  /* runtime state R */
  uint64_t clock, M, peak_M;
  uint64_t base_so_far;
  uint64_t decisions, remats, computations;
  uint64_t trace_hash;
  int status;                 /* sticky OOM / THRASH / CAPACITY / DECISION_CAP */

  /* trace */
  or_trace_rec *trace; uint64_t trace_cap, trace_n;

  /* scratch for E(t) */
  uint32_t *label, *queue; uint64_t *lab_cost; int64_t *lab_maxla; uint32_t scratch_cap;
  uint32_t *stamp; uint32_t epoch;
} Sim;

/* ------------------------------------------------------------------ */
/* allocation                                                          */
/* ------------------------------------------------------------------ */

static void grow(Sim *s, uint32_t need) {
  if (need <= s->cap) return;
  uint32_t nc = s->cap ? s->cap : 16;
  while (nc < need) nc *= 2;
#define RE(f, T) s->f = (T *)realloc(s->f, (size_t)nc * sizeof(T))
  RE(P, vec32); RE(C, vec32); RE(mem, uint64_t); RE(compute, uint64_t); RE(last_access, int64_t);
  RE(m, uint8_t); RE(computed_once, uint8_t); RE(rho, uint64_t); RE(l, uint64_t); RE(in_pool, uint8_t);
  RE(banished, uint8_t);
  RE(set_of, uint64_t); RE(label, uint32_t); RE(queue, uint32_t); RE(lab_cost, uint64_t);
  RE(lab_maxla, int64_t); RE(stamp, uint32_t);
#undef RE
  for (uint32_t i = s->cap; i < nc; i++) {
    memset(&s->P[i], 0, sizeof(vec32)); memset(&s->C[i], 0, sizeof(vec32)); s->stamp[i] = 0;
  }
  s->cap = nc;
}

Sim *oracle_create(int heuristic, uint64_t budget, uint64_t seed, uint32_t thrash_kill,
                   uint64_t max_decisions, uint64_t trace_cap, int e_mode) {
  Sim *s = (Sim *)calloc(1, sizeof(Sim));
  s->heuristic = heuristic; s->B = budget; s->seed = seed; s->thrash_kill = thrash_kill;
  s->max_decisions = max_decisions; s->e_mode = e_mode;
  s->trace_cap = trace_cap;
  s->trace = trace_cap ? (or_trace_rec *)calloc(trace_cap, sizeof(or_trace_rec)) : NULL;
  s->trace_hash = 14695981039346656037ull;   /* FNV-1a 64 offset basis */
  return s;
}

void oracle_destroy(Sim *s) {
  if (!s) return;
  for (uint32_t i = 0; i < s->cap; i++) { free(s->P[i].v); free(s->C[i].v); }
  free(s->P); free(s->C); free(s->mem); free(s->compute); free(s->last_access); free(s->m);
  free(s->computed_once); free(s->rho); free(s->l); free(s->in_pool); free(s->banished); free(s->set_of);
  free(s->label); free(s->queue); free(s->lab_cost); free(s->lab_maxla); free(s->stamp);
  free(s->uf); free(s->trace); free(s);
}

/* ------------------------------------------------------------------ */
/* union-find                                            */
/* ------------------------------------------------------------------ */

/* "when a storage is first computed, its evicted component is also initialized
 * to be empty"; "assign S to a new empty UF set". */
static uint64_t uf_new_empty(Sim *s) {
  if (s->uf_n == s->uf_cap) {
    s->uf_cap = s->uf_cap ? 2 * s->uf_cap : 64;
    s->uf = (uf_node *)realloc(s->uf, s->uf_cap * sizeof(uf_node));
  }
  uint64_t x = s->uf_n++;
  s->uf[x].parent = x; s->uf[x].cost = 0; s->uf[x].maxla = NEG_INF; s->uf[x].size = 1;
  return x;
}

static uint64_t uf_find(Sim *s, uint64_t x) {
  while (s->uf[x].parent != x) x = s->uf[x].parent;   /* no path compression: plain */
  return x;
}

/* "the union of two components having the sum of each constituent cost" */
static void uf_union(Sim *s, uint64_t a, uint64_t b) {
  a = uf_find(s, a); b = uf_find(s, b);
  if (a == b) return;
  if (s->uf[a].size < s->uf[b].size) { uint64_t x = a; a = b; b = x; }   /* union by size */
  s->uf[b].parent = a;
  s->uf[a].size += s->uf[b].size;
  s->uf[a].cost += s->uf[b].cost;
  if (s->uf[b].maxla > s->uf[a].maxla) s->uf[a].maxla = s->uf[b].maxla;   /* reading C-9 */
}

/* ------------------------------------------------------------------ */
/* pool: t in pool  <=>  t.m = T and t.l = 0                */
/* ------------------------------------------------------------------ */

/* C-19; a V1-banished tensor is no longer part of the graph */
static int evicted(const Sim *s, uint32_t x) { return !s->m[x] && s->computed_once[x] && !s->banished[x]; }

/* ------------------------------------------------------------------ */
/* Evicted neighbourhood E(t): evicted tensors weakly reachable from
 * t when all other material tensors are deleted from the graph.            */
/* ------------------------------------------------------------------ */

/* Mode 0: label the connected components of the undirected graph induced on
 * evicted tensors (once per decision); E(t) is the union of the components of
 * t's evicted neighbours (P:2270-2276 describes exactly this decomposition). */
static void label_components(Sim *s) {
  const uint32_t NONE = 0xFFFFFFFFu;
  for (uint32_t i = 0; i < s->n; i++) s->label[i] = NONE;
  uint32_t nlab = 0;
  for (uint32_t r = 0; r < s->n; r++) {
    if (!evicted(s, r) || s->label[r] != NONE) continue;
    uint32_t qh = 0, qt = 0;
    s->queue[qt++] = r; s->label[r] = nlab;
    uint64_t cost = 0; int64_t mx = NEG_INF;
    while (qh < qt) {
      uint32_t x = s->queue[qh++];
      cost += s->compute[x];
      if (s->last_access[x] > mx) mx = s->last_access[x];
      for (int side = 0; side < 2; side++) {
        vec32 *adj = side ? &s->C[x] : &s->P[x];
        for (uint32_t j = 0; j < adj->n; j++) {
          uint32_t y = adj->v[j];
          if (evicted(s, y) && s->label[y] == NONE) { s->label[y] = nlab; s->queue[qt++] = y; }
        }
      }
    }
    s->lab_cost[nlab] = cost; s->lab_maxla[nlab] = mx;
    nlab++;
  }
}

/* sum of compute over E(t), and max last_access over E(t) (NEG_INF if E empty) */
static void neighbourhood(Sim *s, uint32_t t, uint64_t *sum, int64_t *mx) {
  *sum = 0; *mx = NEG_INF;
  if (s->e_mode == 0) {
    /* distinct components adjacent to t */
    s->epoch++;
    for (int side = 0; side < 2; side++) {
      vec32 *adj = side ? &s->C[t] : &s->P[t];
      for (uint32_t j = 0; j < adj->n; j++) {
        uint32_t y = adj->v[j];
        if (!evicted(s, y)) continue;
        uint32_t c = s->label[y];
        if (s->stamp[c] == s->epoch) continue;      /* stamp indexed by label id */
        s->stamp[c] = s->epoch;
        *sum += s->lab_cost[c];
        if (s->lab_maxla[c] > *mx) *mx = s->lab_maxla[c];
      }
    }
    return;
  }
  /* Mode 1: the definition literally -- BFS from t through evicted tensors only. */
  s->epoch++;
  uint32_t qh = 0, qt = 0;
  s->stamp[t] = s->epoch;
  s->queue[qt++] = t;
  while (qh < qt) {
    uint32_t x = s->queue[qh++];
    for (int side = 0; side < 2; side++) {
      vec32 *adj = side ? &s->C[x] : &s->P[x];
      for (uint32_t j = 0; j < adj->n; j++) {
        uint32_t y = adj->v[j];
        if (!evicted(s, y) || s->stamp[y] == s->epoch) continue;
        s->stamp[y] = s->epoch;
        s->queue[qt++] = y;
        *sum += s->compute[y];
        if (s->last_access[y] > *mx) *mx = s->last_access[y];
      }
    }
  }
}

/* e_R(t): "the set of evicted tensors that would have to be rematerialized in
 * order to rematerialize t" -- evicted ancestors reached through
 * evicted parents only.  Returns the sum of their compute. */
static uint64_t msps_closure(Sim *s, uint32_t t) {
  s->epoch++;
  uint32_t qh = 0, qt = 0;
  uint64_t sum = 0;
  s->queue[qt++] = t; s->stamp[t] = s->epoch;
  while (qh < qt) {
    uint32_t x = s->queue[qh++];
    for (uint32_t j = 0; j < s->P[x].n; j++) {
      uint32_t p = s->P[x].v[j];
      if (!evicted(s, p) || s->stamp[p] == s->epoch) continue;
      s->stamp[p] = s->epoch;
      s->queue[qt++] = p;
      sum += s->compute[p];
    }
  }
  return sum;
}

/* e*(S): the evicted storages that must be resident to compute
 * S (transitive closure through evicted deps) together with the evicted
 * storages that need S to be resident (closure through evicted dependents).
 * Returns the sum of their compute. */
static uint64_t estar_closure(Sim *s, uint32_t t) {
  uint64_t sum = msps_closure(s, t);               /* ancestors through evicted parents */
  s->epoch++;
  uint32_t qh = 0, qt = 0;
  s->queue[qt++] = t; s->stamp[t] = s->epoch;
  while (qh < qt) {                                /* descendants through evicted children */
    uint32_t x = s->queue[qh++];
    for (uint32_t j = 0; j < s->C[x].n; j++) {
      uint32_t c = s->C[x].v[j];
      if (!evicted(s, c) || s->stamp[c] == s->epoch) continue;
      s->stamp[c] = s->epoch;
      s->queue[qt++] = c;
      sum += s->compute[c];
    }
  }
  return sum;
}

/* ------------------------------------------------------------------ */
/* scores: exact rationals (num, den); den = 0 encodes +infinity         */
/* ------------------------------------------------------------------ */

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* numerator / (mem * stale(L)), with stale = clock - L (reading C-2),
 * L = -inf -> score 0 (V2, P:110-111 / reading C-4), stale = 0 -> +inf (C-3). */
static void staleness_score(const Sim *s, uint64_t num, uint64_t mem, int64_t L,
                            uint64_t *on, uint64_t *od) {
  if (L == NEG_INF) { *on = 0; *od = 1; return; }
  uint64_t st = (uint64_t)((int64_t)s->clock - L);
  if (st == 0) { *on = 1; *od = 0; return; }
  *on = num; *od = mem * st;
}

/* e~*(t): the distinct union-find sets of t's evicted deps and
 * dependents; *sum = their total cost, *L = max(*L, their max last_access). */
static void eqclass_sum(Sim *s, uint32_t t, uint64_t *sum_out, int64_t *L_out) {
  uint64_t sum = 0; int64_t L = *L_out;
  uint64_t roots[2048]; uint32_t nr = 0;          /* distinct adjacent roots */
  uint64_t *rs = roots; uint64_t *heap = NULL;
  uint32_t deg = s->P[t].n + s->C[t].n;
  if (deg > 2048) { heap = (uint64_t *)malloc(deg * sizeof(uint64_t)); rs = heap; }
  for (int side = 0; side < 2; side++) {
    vec32 *adj = side ? &s->C[t] : &s->P[t];
    for (uint32_t j = 0; j < adj->n; j++) {
      uint32_t y = adj->v[j];
      if (!evicted(s, y)) continue;
      uint64_t r = uf_find(s, s->set_of[y]);     /* no unions when querying */
      int dup = 0;
      for (uint32_t k = 0; k < nr; k++) if (rs[k] == r) { dup = 1; break; }
      if (dup) continue;
      rs[nr++] = r;
      sum += s->uf[r].cost;
      if (s->uf[r].maxla > L) L = s->uf[r].maxla;
    }
  }
  free(heap);
  *sum_out = sum; *L_out = L;
}

static void score(Sim *s, uint32_t t, uint64_t *num, uint64_t *den) {
  switch (s->heuristic) {
    case H_DTR: {
      uint64_t sum; int64_t mx;
      neighbourhood(s, t, &sum, &mx);
      int64_t L = s->last_access[t] > mx ? s->last_access[t] : mx;
      staleness_score(s, s->compute[t] + sum, s->mem[t], L, num, den);
      return;
    }
    case H_DTR_EQ: {         /* P:2286-2293; staleness per reading C-9 */
      uint64_t sum; int64_t L = s->last_access[t];
      eqclass_sum(s, t, &sum, &L);
      staleness_score(s, s->compute[t] + sum, s->mem[t], L, num, den);
      return;
    }
    case H_LRU:              /* 1 / s(t) */
      staleness_score(s, 1, 1, s->last_access[t], num, den);
      return;
    case H_SIZE:             /* 1 / m(t) */
      *num = 1; *den = s->mem[t];
      return;
    case H_MSPS:             /* (c0(t) + sum_{e_R(t)} c0) / m(t) */
      *num = s->compute[t] + msps_closure(s, t); *den = s->mem[t];
      return;
    case H_LOCAL:            /* c0 / (m * s) */
      staleness_score(s, s->compute[t], s->mem[t], s->last_access[t], num, den);
      return;
    case H_DTR_FULL:         /* (c(S) + sum_{e*(S)} c) / (size(S) * stale(S)) */
      staleness_score(s, s->compute[t] + estar_closure(s, t), s->mem[t], s->last_access[t], num, den);
      return;
    case H_ESTAR:            /* h_e*(t) = (c(t) + c0(f_t)) / m(t) */
      *num = s->compute[t] + estar_closure(s, t); *den = s->mem[t];
      return;
    case H_RANDOM:           /* X ~ U(0,1) as a counter-based draw (reading C-15) */
      *num = splitmix64(s->seed ^ (s->decisions << 32) ^ (uint64_t)t); *den = 1;
      return;
  }
  if (is_abl(s->heuristic)) {  /* h'(s, m, c)(t) = c(t) / [m(t) s(t)]  (reading C-23) */
    const int code = s->heuristic - H_ABL, cc = code >> 2, use_m = (code >> 1) & 1, use_s = code & 1;
    uint64_t c = 1;                                            /* c = no: c(t) = 1 */
    if (cc == ABL_C_ESTAR) c = s->compute[t] + estar_closure(s, t);
    else if (cc == ABL_C_EQCLASS) {
      uint64_t sum; int64_t L = s->last_access[t];
      eqclass_sum(s, t, &sum, &L);                             /* the sets' costs; own staleness */
      c = s->compute[t] + sum;
    } else if (cc == ABL_C_LOCAL) c = s->compute[t];
    const uint64_t m = use_m ? s->mem[t] : 1;                  /* m = no: m(t) = 1 */
    if (use_s) staleness_score(s, c, m, s->last_access[t], num, den);   /* stale_T(t) */
    else { *num = c; *den = m; }                               /* s = no: s(t) = 1 */
    return;
  }
  *num = 0; *den = 1;
}

/* a < b  <=>  a.num * b.den < b.num * a.den (exact); equal scores -> smaller id (C-5) */
static int score_less(uint64_t an, uint64_t ad, uint32_t aid, uint64_t bn, uint64_t bd, uint32_t bid) {
  unsigned __int128 l = (unsigned __int128)an * bd, r = (unsigned __int128)bn * ad;
  if (l != r) return l < r;
  return aid < bid;
}

/* ------------------------------------------------------------------ */
/* internal API                                              */
/* ------------------------------------------------------------------ */

static void fnv(Sim *s, uint64_t v) { s->trace_hash ^= v; s->trace_hash *= 1099511628211ull; }

/* R.evict(t), plus the UF union on eviction. */
static void evict(Sim *s, uint32_t t) {
  s->m[t] = 0;
  s->M -= s->mem[t];
  s->in_pool[t] = 0;
  if (uses_uf(s->heuristic)) {
    uint64_t r = uf_find(s, s->set_of[t]);
    s->uf[r].cost += s->compute[t];                               /* "+c0(t)" */
    if (s->last_access[t] > s->uf[r].maxla) s->uf[r].maxla = s->last_access[t];
    for (int side = 0; side < 2; side++) {
      vec32 *adj = side ? &s->C[t] : &s->P[t];
      for (uint32_t j = 0; j < adj->n; j++) {
        uint32_t y = adj->v[j];
        if (evicted(s, y)) uf_union(s, s->set_of[t], s->set_of[y]);
      }
    }
  }
}

/* R.free(size): while M + size > B: evict argmin_{pool} h. */
static int free_mem(Sim *s, uint64_t size) {
  while (s->M + size > s->B) {
    if (s->max_decisions && s->decisions >= s->max_decisions) return OR_DECISION_CAP;
    int any = 0;
    for (uint32_t t = 0; t < s->n; t++) if (s->in_pool[t]) { any = 1; break; }
    if (!any) return OR_OOM;                                     /* P:175 "can fail (OOM)" */
    if (s->heuristic == H_DTR && s->e_mode == 0) label_components(s);
    uint64_t bn = 0, bd = 0; uint32_t best = 0xFFFFFFFFu;
    for (uint32_t t = 0; t < s->n; t++) {
      if (!s->in_pool[t]) continue;
      uint64_t num, den;
      score(s, t, &num, &den);
      if (best == 0xFFFFFFFFu || score_less(num, den, t, bn, bd, best)) { bn = num; bd = den; best = t; }
    }
    if (s->trace_n < s->trace_cap) {
      or_trace_rec *r = &s->trace[s->trace_n++];
      r->clock = s->clock; r->id = best; r->pad = 0; r->num = bn; r->den = bd;
    }
    fnv(s, s->clock); fnv(s, best); fnv(s, bn); fnv(s, bd);
    s->decisions++;
    evict(s, best);
  }
  return OR_OK;
}

/* R.banish_V1(t): evict t if material, pin its children (l + 1,
 * which takes them out of the pool: pool = {m and l = 0}, reading C-22), and
 * remove t from the graph; it never re-enters the pool.  A banished evicted
 * tensor leaves its union-find set like a rematerialized one (its cost is
 * subtracted, reading C-22). */
static void banish_v1(Sim *s, uint32_t t) {
  if (s->m[t]) {
    s->m[t] = 0;
    s->M -= s->mem[t];
    s->in_pool[t] = 0;
  } else if (uses_uf(s->heuristic) && evicted(s, t)) {
    uint64_t r = uf_find(s, s->set_of[t]);
    s->uf[r].cost -= s->compute[t];
  }
  s->banished[t] = 1;
  for (uint32_t j = 0; j < s->C[t].n; j++) {
    uint32_t c = s->C[t].v[j];
    s->l[c]++;
    s->in_pool[c] = 0;
    vremove(&s->P[c], t);
  }
  for (uint32_t j = 0; j < s->P[t].n; j++) vremove(&s->C[s->P[t].v[j]], t);
  s->C[t].n = 0;
  s->P[t].n = 0;
}

/* banish condition: rho = 0 and every child material (the lock
 * count is not consulted: a lock taken by a pending computation always comes
 * with a non-material child, and pinned tensors may be banished later,
 * P:2372-2375). */
static void maybe_banish_v1(Sim *s, uint32_t t) {
  if (s->dealloc != DEALLOC_V1 || s->banished[t] || s->rho[t] != 0) return;
  for (uint32_t j = 0; j < s->C[t].n; j++) if (!s->m[s->C[t].v[j]]) return;
  banish_v1(s, t);
}

/* R.release_internal(t). */
static void release_internal(Sim *s, uint32_t t) {
  s->l[t]--;
  if (s->l[t] == 0 && !s->banished[t]) s->in_pool[t] = 1;
  maybe_banish_v1(s, t);
}

/* R.get_internal(t). Recursive, depth-first. */
static int get_internal(Sim *s, uint32_t t) {
  if (s->m[t]) {
    s->l[t]++;
    s->in_pool[t] = 0;
    return OR_OK;
  }
  /* Let P_T := {p in t.P | p.m = T}; P_B := t.P \ P_T  (evaluated once, reading C-6) */
  uint32_t np = s->P[t].n;
  uint32_t *pt = (uint32_t *)malloc((np + 1) * sizeof(uint32_t));
  uint32_t *pb = (uint32_t *)malloc((np + 1) * sizeof(uint32_t));
  uint32_t nt = 0, nb = 0;
  for (uint32_t j = 0; j < np; j++) {
    uint32_t p = s->P[t].v[j];
    if (s->m[p]) pt[nt++] = p; else pb[nb++] = p;
  }
  int rc = OR_OK;
  for (uint32_t j = 0; j < nt && rc == OR_OK; j++) rc = get_internal(s, pt[j]);
  for (uint32_t j = 0; j < nb && rc == OR_OK; j++) rc = get_internal(s, pb[j]);
  free(pb);
  if (rc == OR_OK && s->M + s->mem[t] > s->B) rc = free_mem(s, s->mem[t]);
  if (rc != OR_OK) { free(pt); return rc; }
  /* the parents locked above, in t.P order: a V1 banish inside the release
   * loop removes that parent from t.P, so iterate a copy (reading C-22) */
  for (uint32_t j = 0; j < np; j++) pt[j] = s->P[t].v[j];
  s->m[t] = 1;
  s->l[t] = 1;
  s->M += s->mem[t];
  if (s->M > s->peak_M) s->peak_M = s->M;
  s->clock += s->compute[t];
  s->computations++;
  if (s->computed_once[t]) {
    s->remats++;
    if (uses_uf(s->heuristic)) {
      /* "S.set.cost := S.set.cost - cost(S); S.set := empty" */
      uint64_t r = uf_find(s, s->set_of[t]);
      s->uf[r].cost -= s->compute[t];
      s->set_of[t] = uf_new_empty(s);
    }
  } else {
    s->computed_once[t] = 1;
    if (uses_uf(s->heuristic)) s->set_of[t] = uf_new_empty(s);
  }
  if (s->clock > CLOCK_LIMIT) { free(pt); return OR_CAPACITY; }
  if (s->thrash_kill && s->clock > (uint64_t)s->thrash_kill * s->base_so_far) { free(pt); return OR_THRASH; }
  for (uint32_t j = 0; j < np; j++) release_internal(s, pt[j]);
  free(pt);
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* external API                                              */
/* ------------------------------------------------------------------ */

static int sticky(Sim *s) { return s->status != OR_OK; }

static int finish(Sim *s, int rc) {
  if (rc == OR_OOM || rc == OR_THRASH || rc == OR_CAPACITY || rc == OR_DECISION_CAP) s->status = rc;
  return rc;
}

/* R.make_tensor(f, P). Returns the new id in *out. */
int oracle_make(Sim *s, uint64_t mem, uint64_t compute, const uint32_t *parents, uint32_t np, uint32_t *out) {
  if (sticky(s)) return OR_STATE;
  for (uint32_t j = 0; j < np; j++)
    if (parents[j] >= s->n || s->rho[parents[j]] == 0) return OR_PRECOND;   /* reading C-12 */
  grow(s, s->n + 1);
  uint32_t t = s->n++;
  memset(&s->P[t], 0, sizeof(vec32)); memset(&s->C[t], 0, sizeof(vec32));
  for (uint32_t j = 0; j < np; j++) {          /* P is a set: first occurrence kept (C-7) */
    int dup = 0;
    for (uint32_t k = 0; k < s->P[t].n; k++) if (s->P[t].v[k] == parents[j]) dup = 1;
    if (!dup) vpush(&s->P[t], parents[j]);
  }
  /* Let I := (f.mem, f.compute, R.clock); t := (P, {}, I, bot, 1, 0) */
  s->mem[t] = mem; s->compute[t] = compute; s->last_access[t] = (int64_t)s->clock;
  s->m[t] = 0; s->computed_once[t] = 0; s->rho[t] = 1; s->l[t] = 0; s->in_pool[t] = 0; s->banished[t] = 0;
  s->set_of[t] = 0;
  s->base_so_far += compute;
  /* foreach p in P: p.C := p.C u {t}; p.I.last_accessed := R.clock */
  for (uint32_t j = 0; j < s->P[t].n; j++) {
    uint32_t p = s->P[t].v[j];
    vpush(&s->C[p], t);
    s->last_access[p] = (int64_t)s->clock;
    if (uses_uf(s->heuristic) && evicted(s, p)) {              /* reading C-9 */
      uint64_t r = uf_find(s, s->set_of[p]);
      if ((int64_t)s->clock > s->uf[r].maxla) s->uf[r].maxla = (int64_t)s->clock;
    }
  }
  if (out) *out = t;
  /* R.rematerialize(t) = get_internal(t); release_internal(t) */
  int rc = get_internal(s, t);
  if (rc != OR_OK) return finish(s, rc);
  release_internal(s, t);
  return OR_OK;
}

/* R.get(t) */
int oracle_get(Sim *s, uint32_t t) {
  if (sticky(s)) return OR_STATE;
  if (t >= s->n || s->rho[t] == 0) return OR_PRECOND;
  s->rho[t]++;
  return OR_OK;
}

/* R.release(t).  At rho = 0:
 *   V2     banish_V2: last_access := -inf
 *   V1     banish_V1 when every child is material
 *   eager  evict t normally if it is in the pool
 *   ignore nothing */
int oracle_release(Sim *s, uint32_t t) {
  if (sticky(s)) return OR_STATE;
  if (t >= s->n || s->rho[t] == 0) return OR_PRECOND;
  s->rho[t]--;
  if (s->rho[t] != 0) return OR_OK;
  if (s->dealloc == DEALLOC_V2) s->last_access[t] = NEG_INF;
  else if (s->dealloc == DEALLOC_V1) maybe_banish_v1(s, t);
  else if (s->dealloc == DEALLOC_EAGER && s->in_pool[t]) evict(s, t);
  return OR_OK;
}

/* R.rematerialize(t): precondition t.m = bot */
int oracle_rematerialize(Sim *s, uint32_t t) {
  if (sticky(s)) return OR_STATE;
  if (t >= s->n || s->m[t] || !s->computed_once[t] || s->banished[t]) return OR_PRECOND;  /* C-22 */
  int rc = get_internal(s, t);
  if (rc != OR_OK) return finish(s, rc);
  release_internal(s, t);
  return OR_OK;
}

/* Output condition (reading C-11): get_internal(t) with no matching release. */
int oracle_ensure(Sim *s, uint32_t t) {
  if (sticky(s)) return OR_STATE;
  if (t >= s->n || !s->computed_once[t] || s->banished[t]) return OR_PRECOND;  /* C-22 */
  int rc = get_internal(s, t);
  if (rc != OR_OK) return finish(s, rc);
  return OR_OK;
}

/* Test fixtures: R.evict(t) on a pool member, outside free(). */
int oracle_debug_evict(Sim *s, uint32_t t) {
  if (sticky(s)) return OR_STATE;
  if (t >= s->n || !s->in_pool[t]) return OR_PRECOND;
  evict(s, t);
  return OR_OK;
}

void oracle_set_budget(Sim *s, uint64_t B) { s->B = B; }
void oracle_set_dealloc(Sim *s, int policy) { s->dealloc = policy; }

/* Current (num, den) of every pool member, in id order. Returns the count. */
uint64_t oracle_scores(Sim *s, uint64_t *num, uint64_t *den, uint32_t *ids, uint64_t cap) {
  if (s->heuristic == H_DTR && s->e_mode == 0) label_components(s);
  uint64_t k = 0;
  for (uint32_t t = 0; t < s->n; t++) {
    if (!s->in_pool[t]) continue;
    if (k < cap) { score(s, t, &num[k], &den[k]); ids[k] = t; }
    k++;
  }
  return k;
}

/* E(t) as an explicit set (literal BFS), for the worked-example pins. */
uint32_t oracle_neighbourhood(Sim *s, uint32_t t, uint32_t *out, uint32_t cap) {
  s->epoch++;
  uint32_t qh = 0, qt = 0, k = 0;
  s->stamp[t] = s->epoch;
  s->queue[qt++] = t;
  while (qh < qt) {
    uint32_t x = s->queue[qh++];
    for (int side = 0; side < 2; side++) {
      vec32 *adj = side ? &s->C[x] : &s->P[x];
      for (uint32_t j = 0; j < adj->n; j++) {
        uint32_t y = adj->v[j];
        if (!evicted(s, y) || s->stamp[y] == s->epoch) continue;
        s->stamp[y] = s->epoch;
        s->queue[qt++] = y;
        if (k < cap) out[k] = y;
        k++;
      }
    }
  }
  return k;
}

/* e*(t) as an explicit set (directed), for the worked-example pins. */
uint32_t oracle_estar(Sim *s, uint32_t t, uint32_t *out, uint32_t cap) {
  uint32_t k = 0;
  for (int dir = 0; dir < 2; dir++) {
    s->epoch++;
    uint32_t qh = 0, qt = 0;
    s->queue[qt++] = t; s->stamp[t] = s->epoch;
    while (qh < qt) {
      uint32_t x = s->queue[qh++];
      vec32 *adj = dir ? &s->C[x] : &s->P[x];
      for (uint32_t j = 0; j < adj->n; j++) {
        uint32_t y = adj->v[j];
        if (!evicted(s, y) || s->stamp[y] == s->epoch) continue;
        s->stamp[y] = s->epoch;
        s->queue[qt++] = y;
        if (k < cap) out[k] = y;
        k++;
      }
    }
  }
  return k;
}

/* Introspection for invariant tests. */
void oracle_state(const Sim *s, uint64_t *scalars /* [8] */) {
  scalars[0] = s->clock; scalars[1] = s->M; scalars[2] = s->B; scalars[3] = s->n;
  scalars[4] = s->decisions; scalars[5] = s->remats; scalars[6] = s->computations;
  scalars[7] = (uint64_t)s->status;
}

/* per-tensor flags: bit0 m, bit1 computed_once, bit2 in_pool; plus rho, l, last_access */
void oracle_tensors(const Sim *s, uint8_t *flags, uint64_t *rho, uint64_t *l, int64_t *la) {
  for (uint32_t t = 0; t < s->n; t++) {
    flags[t] = (uint8_t)(s->m[t] | (s->computed_once[t] << 1) | (s->in_pool[t] << 2) | (s->banished[t] << 3));
    rho[t] = s->rho[t]; l[t] = s->l[t]; la[t] = s->last_access[t];
  }
}

/* UF invariants: sum of root costs, and per evicted tensor its root id. */
uint64_t oracle_uf_root_cost_sum(Sim *s) {
  uint64_t sum = 0;
  for (uint64_t x = 0; x < s->uf_n; x++) if (s->uf[x].parent == x) sum += s->uf[x].cost;
  return sum;
}

void oracle_uf_roots(Sim *s, uint64_t *root_of, uint64_t *root_cost, int64_t *root_maxla) {
  for (uint32_t t = 0; t < s->n; t++) {
    if (!evicted(s, t)) { root_of[t] = UINT64_MAX; root_cost[t] = 0; root_maxla[t] = NEG_INF; continue; }
    uint64_t r = uf_find(s, s->set_of[t]);
    root_of[t] = r; root_cost[t] = s->uf[r].cost; root_maxla[t] = s->uf[r].maxla;
  }
}

void oracle_result(const Sim *s, or_result *r) {
  r->status = (uint32_t)s->status;
  r->clock = s->clock; r->base = s->base_so_far; r->decisions = s->decisions;
  r->remats = s->remats; r->computations = s->computations; r->peak_M = s->peak_M;
  r->trace_hash = s->trace_hash;
  r->n_trace = (uint32_t)s->trace_n;
}

uint64_t oracle_trace(const Sim *s, or_trace_rec *buf, uint64_t cap) {
  uint64_t k = s->trace_n < cap ? s->trace_n : cap;
  memcpy(buf, s->trace, k * sizeof(or_trace_rec));
  return s->trace_n;
}

/* ------------------------------------------------------------------ */
/* log replay (format: dtr_inputs/logfmt.py)                              */
/* ------------------------------------------------------------------ */

typedef struct {
  Sim *s; const uint32_t *w; uint64_t nw; or_result *res; int rc;
} replay_args;

static void *replay_thread(void *arg) {
  replay_args *a = (replay_args *)arg;
  Sim *s = a->s; const uint32_t *w = a->w;
  uint32_t n = w[2], E = w[3], nops = w[4];
  const uint32_t *mem = w + 16, *cost = mem + n, *poff = cost + n, *par = poff + n + 1, *ops = par + E;
  (void)E;
  grow(s, n + 1);
  uint32_t done = 0;
  int rc = OR_OK;
  for (uint32_t k = 0; k < nops; k++) {
    uint32_t op = ops[k] >> 29, id = ops[k] & ((1u << 29) - 1);
    switch (op) {
      case OP_MAKE: {
        if (id != s->n) { rc = OR_PRECOND; break; }
        uint32_t out;
        rc = oracle_make(s, mem[id], cost[id], par + poff[id], poff[id + 1] - poff[id], &out);
        break;
      }
      case OP_GET: rc = oracle_get(s, id); break;
      case OP_RELEASE: rc = oracle_release(s, id); break;
      case OP_REMAT: rc = oracle_rematerialize(s, id); break;
      case OP_ENSURE: rc = oracle_ensure(s, id); break;
      case OP_DEBUG_EVICT: rc = oracle_debug_evict(s, id); break;
      default: rc = OR_PRECOND;
    }
    if (rc != OR_OK) break;
    done++;
  }
  if (rc == OR_PRECOND) s->status = OR_PRECOND;
  oracle_result(s, a->res);
  a->res->records_done = done;
  a->rc = rc;
  return NULL;
}

/* Replay a whole log on a fresh simulator. The recursion of get_internal can
 * be as deep as the longest evicted chain, so it runs on a thread with a large
 * stack. */
int oracle_replay(const uint32_t *words, uint64_t n_words, int heuristic, uint64_t budget,
                  uint64_t seed, uint32_t thrash_kill, uint64_t max_decisions, int e_mode, int dealloc,
                  or_result *res, or_trace_rec *trace, uint64_t trace_cap) {
  if (n_words < 16 || words[0] != 0x4C525444u) return OR_PRECOND;
  Sim *s = oracle_create(heuristic, budget, seed, thrash_kill, max_decisions, trace_cap, e_mode);
  s->dealloc = dealloc;
  memset(res, 0, sizeof(*res));
  replay_args a = { s, words, n_words, res, 0 };
  pthread_attr_t attr;
  pthread_attr_init(&attr);
  pthread_attr_setstacksize(&attr, (size_t)1 << 30);
  pthread_t th;
  if (pthread_create(&th, &attr, replay_thread, &a) != 0) { replay_thread(&a); }
  else pthread_join(th, NULL);
  pthread_attr_destroy(&attr);
  if (trace && trace_cap) memcpy(trace, s->trace, (s->trace_n < trace_cap ? s->trace_n : trace_cap) * sizeof(or_trace_rec));
  oracle_destroy(s);
  return OR_OK;
}
