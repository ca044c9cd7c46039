/*
 * dtr.h -- C ABI of the B200-native DTR eviction-decision engine (libdtr.so).
 *
 * Implements the simrd runtime with V2 banishing (PAPER.md Doc A)
 * and the eviction heuristics of the paper; every step of the replay runs in
 * CUDA kernels for sm_100a; the host side only marshals arguments, launches
 * and copies.  Plain C types only: no torch, no C++ in the signatures.
 *
 * Conventions (all calls):
 *   - Tensor ids are dense uint32 in creation order, starting at 0.  Ties in
 *     the eviction argmin go to the smallest id (reading C-5).
 *   - Scores are exact rationals (num, den) of uint64; den == 0 means +inf.
 *     Comparison is num_a*den_b vs num_b*den_a in 128 bits (reading C-14).
 *   - mem and compute are integers >= 1; the clock must stay below 2^32 - 1
 *     (reading C-14), else the run stops with DTR_E_CAPACITY.
 *   - "device" pointers are CUDA device memory (e.g. torch.empty(...,
 *     device='cuda').data_ptr()); "host" pointers are CPU memory.  Input
 *     buffers are read only during the call (or, for *_async device calls,
 *     until the work on `stream` completes); the caller owns every buffer.
 *   - Errors are returned as int codes (below); dtr_strerror() names them.
 *     A CUDA failure returns DTR_E_CUDA and the CUDA error string is kept in
 *     dtr_last_cuda_error().
 */
#ifndef DTR_H
#define DTR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status / error codes (also the `status` of a result row) ---------- */
#define DTR_OK 0
#define DTR_E_INVAL 1         /* bad argument: no state change                             */
#define DTR_E_PRECOND 2       /* simrd precondition violated (C-12)      */
#define DTR_E_OOM 3           /* free() found the pool empty while over budget */
#define DTR_E_THRASH 4        /* clock > thrash_kill * (compute of MAKEs so far) (C-13)    */
#define DTR_E_CAPACITY 5      /* preallocated capacity exceeded or clock >= 2^32 - 1       */
#define DTR_E_STATE 6         /* runtime is stopped by an earlier sticky OOM/THRASH/...   */
#define DTR_E_CUDA 7          /* CUDA runtime error                                        */
#define DTR_E_DECISION_CAP 8  /* stopped after max_decisions eviction decisions (sampling) */

/* ---- heuristics: score(t) evaluated over the pool; the argmin is evicted ---- */
typedef enum {
  DTR_H_DTR = 0,     /* h_DTR, undirected evicted neighbourhood E(t)        */
  DTR_H_DTR_EQ = 1,  /* h_DTR_eq, union-find evicted components + approximate split
                        (staleness: reading C-9)         */
  DTR_H_LRU = 2,     /* 1 / s(t)                                           */
  DTR_H_SIZE = 3,    /* 1 / m(t)              ("GreedyRemat")                            */
  DTR_H_MSPS = 4,    /* (c0(t) + sum_{e_R(t)} c0) / m(t), e_R = evicted ancestors */
  DTR_H_LOCAL = 5,   /* c0(t) / (m(t) s(t))                                      */
  DTR_H_RANDOM = 6,  /* splitmix64(seed ^ decision << 32 ^ id) (reading C-15)      */
  DTR_H_DTR_FULL = 7,/* (c0(t) + sum over the DIRECTED e*(t) of c0) / (m(t) s(t)): e* = evicted
                        ancestors and descendants reached through evicted tensors
                        (P:934-951); own staleness              */
  DTR_H_ESTAR = 8,   /* h_e* = (c0(t) + sum_{e*(t)} c0) / m(t), Theorem 1's compute-memory
                        heuristic                                             */
  DTR_H_ABL = 16     /* first of the 16 D.1 ablation variants, see DTR_H_ABLATION            */
} dtr_heuristic;

/* The D.1 ablation h'(s, m, c)(t) = c(t) / [m(t) * s(t)] (DESIGN.md
 * reading C-23).  c: 0 = e* (c0(t) + sum_{e*(t)} c0), 1 = EqClass (c0(t) + the costs
 * of the distinct union-find sets of t's evicted deps and dependents),
 * 2 = local (c0(t)), 3 = no (1); m, s: 1 = size / own staleness, 0 = the constant 1.
 * The heuristic id is DTR_H_ABLATION(c, m, s), i.e. 16 ... 31. */
#define DTR_H_ABLATION(c, m, s) (DTR_H_ABL + 4u * (uint32_t)(c) + 2u * (uint32_t)(m) + (uint32_t)(s))

/* ---- deallocation policies: what release(t) does when t.rho drops to 0 ----
 * (reading C-22) */
typedef enum {
  DTR_DEALLOC_V2 = 0,      /* banish_V2: last_access := -inf -- the default       */
  DTR_DEALLOC_V1 = 1,      /* banish_V1 once every child is material: evict, pin the children,
                              remove t from the graph       */
  DTR_DEALLOC_EAGER = 2,   /* evict t normally if it is in the pool */
  DTR_DEALLOC_IGNORE = 3   /* nothing                                            */
} dtr_dealloc;

/* ---- log encoding (little-endian uint32 words; see dtr_inputs/logfmt.py) ----
 * header[16]: magic 'DTRL', version 1, n_tensors, n_edges, n_ops, model_id,
 *             base(u64), peak_live(u64), peak_total(u64), seed(u64), max_parents, 0
 * then mem[n], cost[n], par_off[n+1], par[n_edges], ops[n_ops] (op << 29 | id).
 * Ops: MAKE=1 (make_tensor), GET=2, RELEASE=3 (P:357-373,
 * V2 banish), REMAT=4 (rematerialize), ENSURE=5 (output condition:
 * get_internal without release, reading C-11), DEBUG_EVICT=6 (evict a pool
 * member outside free(); fixtures only). */
#define DTR_LOG_MAGIC 0x4C525444u
#define DTR_LOG_HEADER_WORDS 16

/* One eviction decision: clock at the decision, evicted id, its score. 32 B. */
typedef struct {
  uint64_t clock;
  uint32_t id;
  uint32_t pad;
  uint64_t num;
  uint64_t den;
} dtr_evict_rec;

/* Per-run result row (96 B).  `status` is DTR_OK or the code that stopped the
 * run; counters are the state at the stop.  trace_hash = FNV-1a-64 folded over
 * (clock, id, num, den) of every decision, one 64-bit word at a time:
 * h = 14695981039346656037; for w in words: h = (h ^ w) * 1099511628211. */
typedef struct {
  uint32_t cell_id;
  uint32_t status;
  uint32_t records_done;   /* log records fully applied */
  uint32_t n_trace;        /* decisions written to the trace buffer */
  uint64_t clock;          /* R.clock */
  uint64_t base;           /* sum of compute of MAKE records started */
  uint64_t decisions;      /* evictions chosen by free() */
  uint64_t remats;         /* computations of already-computed tensors */
  uint64_t computations;   /* all computations */
  uint64_t peak_M;         /* max R.M */
  uint64_t trace_hash;
  uint64_t cand_evals;     /* pool members scored over all decisions (batch engines) */
  uint64_t score_bytes;    /* algorithmic bytes those score passes read (DESIGN.md Roofline) */
  uint64_t wall_ns;        /* device time of this run, first to last instruction (%globaltimer, ns;
                              batch engines and the adversary; 0 for the per-call runtime) */
} dtr_result;

/* One simulation of a sweep (64 B). */
typedef struct {
  uint64_t log_offset;     /* word offset of this cell's log in the packed words buffer */
  uint64_t budget;         /* R.B, same unit as mem */
  uint64_t seed;           /* DTR_H_RANDOM only */
  uint64_t max_decisions;  /* 0 = unlimited; else stop with DTR_E_DECISION_CAP */
  uint64_t trace_offset;   /* first record index of this cell in the trace buffer */
  uint64_t trace_cap;      /* records this cell may write (0 = none) */
  uint32_t heuristic;      /* dtr_heuristic */
  uint32_t thrash_kill;    /* 0 = off; else stop with DTR_E_THRASH when clock > kill*base */
  uint32_t cell_id;
  uint32_t dealloc;        /* dtr_dealloc: what release() does at rho = 0 */
} dtr_cell;

/* Engines: one CTA per simulation (many small runs, K6) or the whole GPU per
 * simulation (one large run, K7: cooperative persistent grid). */
#define DTR_ENGINE_CTA 1
#define DTR_ENGINE_GRID 2
/* Automatic engine choice (dtr_replay_batch_host with engine 0, and the
 * sweep's rank split): logs with at least this many tensors replay on the
 * whole-GPU engine. */
#define DTR_GRID_MIN_TENSORS 65536u

const char *dtr_strerror(int code);
const char *dtr_last_cuda_error(void);
int dtr_version(void);

/* ---------------------------------------------------------------------------
 * Batched replay (the throughput path, P:273-284 at every over-budget
 * allocation of every cell).
 * ------------------------------------------------------------------------- */

/* Device workspace needed by a batch.  dims: host array of n_cells triples
 * {n_tensors, n_edges, heuristic} (from each cell's log header).  `engine`:
 * DTR_ENGINE_CTA (cells run concurrently; sum of per-cell sizes) or
 * DTR_ENGINE_GRID (cells run one after another; max).  Returns DTR_OK or
 * DTR_E_INVAL. */
int dtr_batch_workspace_bytes(const uint32_t *dims, uint32_t n_cells, uint32_t engine,
                              uint64_t *bytes_out);

/* Shared-memory class of one CTA-engine cell (dims {n_tensors, n_edges,
 * heuristic} as above): 0 = small (several CTAs per SM), 1 = staged whole in
 * shared memory, 2 = state in the global workspace.  dtr_replay_batch makes
 * one launch per run of consecutive cells of one class, so a caller that
 * orders its cells (e.g. longest first, sweep.RankSweep) keeps each class
 * contiguous.  Host only, no device call.  Returns DTR_OK or DTR_E_INVAL. */
int dtr_cta_class(uint32_t n_tensors, uint32_t n_edges, uint32_t heuristic, uint32_t *class_out);

/* Replay every cell.  d_words: device, packed logs.  d_cells: device, n_cells
 * dtr_cell.  h_dims: HOST copy of the dims array above (sizes the workspace
 * and the shared-memory staging of each launch).  d_ws: device workspace of
 * ws_bytes (contents overwritten; cell regions are placed on the device).
 * d_rows: device, n_cells dtr_result (written).  d_trace: device
 * dtr_evict_rec buffer indexed by each cell's trace_offset (may be NULL when
 * every trace_cap is 0).  Asynchronous on `stream` (cudaStream_t, NULL =
 * legacy default); per-cell failures are reported in the rows.  Returns
 * DTR_E_INVAL / DTR_E_CAPACITY (workspace too small) / DTR_E_CUDA (launch).
 * CTA engine: one launch, one CTA per cell, each simulation's whole state in
 * shared memory when it fits (<= 200 KiB), else in its workspace region. */
int dtr_replay_batch(const uint32_t *d_words, const dtr_cell *d_cells, const uint32_t *h_dims,
                     uint32_t n_cells, uint32_t engine, void *d_ws, uint64_t ws_bytes,
                     dtr_result *d_rows, dtr_evict_rec *d_trace, void *stream);

/* K3+K4 alone (score pass + exact argmin) over the current pool of the
 * simulation left in a grid-engine workspace by the last dtr_replay_batch
 * (DTR_ENGINE_GRID) call -- e.g. one stopped with DTR_E_DECISION_CAP: "which
 * tensor would free() evict next".  d_log: device pointer to that cell's log
 * (words + log_offset).  heuristic: the cell's.  d_out: device, 5 uint64
 * {num, den, id, score_bytes, cand_evals}; id = 0xFFFFFFFF for an empty pool.
 * Asynchronous on `stream`; does not modify the simulation. */
int dtr_pool_argmin(const uint32_t *d_log, uint32_t heuristic, void *d_ws, uint64_t *d_out, void *stream);

/* End-to-end convenience: host inputs and outputs.  Copies h_words (n_words)
 * and h_cells to the device, replays (engine as above; 0 = choose per size),
 * copies rows (and trace_total trace records when h_trace != NULL) back, and
 * synchronizes `stream`.  Device memory is stream-ordered (cudaMallocAsync). */
int dtr_replay_batch_host(const uint32_t *h_words, uint64_t n_words, const dtr_cell *h_cells,
                          uint32_t n_cells, uint32_t engine, dtr_result *h_rows,
                          dtr_evict_rec *h_trace, uint64_t trace_total, void *stream);

/* ---------------------------------------------------------------------------
 * The Theorem 2 adversary (App. B; reading C-24): one
 * run per dtr_adversary, one CTA per run, all runs in one launch.  The graph is
 * generated online from the runtime's residency: t0 (unit size and cost,
 * locked resident by one ENSURE) gets B children t1..tB (the B paths); after
 * that every node is the child of the last node of the lowest-indexed path with
 * no resident node.  Unit sizes and costs; nothing is released.  The run stops
 * after N nodes (t0 included) or at the first error (OOM cannot happen for
 * B >= 3).  Static path-at-a-time cost is N.
 * ------------------------------------------------------------------------- */
typedef struct {
  uint32_t n;              /* N >= 1: nodes to reveal, t0 included (< 2^27)            */
  uint32_t budget;         /* B >= 3 memory units; t0 holds one          */
  uint32_t heuristic;      /* dtr_heuristic                                             */
  uint32_t cell_id;        /* copied to the result row                                  */
  uint64_t seed;           /* DTR_H_RANDOM draws                                        */
  uint64_t trace_offset;   /* first dtr_evict_rec of this run in d_trace                */
  uint32_t trace_cap;      /* eviction records kept for this run (0 = none)             */
  uint32_t reserved;       /* 0                                                         */
} dtr_adversary;           /* 40 bytes */

/* Device workspace for a batch of runs (h_runs on the HOST): 256 B plus one
 * 256-B aligned region per run (used when a run's state does not fit in
 * shared memory).  DTR_E_INVAL for n == 0, n >= 2^27, budget < 3 or an unknown
 * heuristic. */
int dtr_adversary_workspace_bytes(const dtr_adversary *h_runs, uint32_t n_runs, uint64_t *bytes);

/* Run the batch asynchronously on `stream`.  d_runs: the runs in device memory,
 * h_runs: the same array on the host (sizes the launch).  Outputs (device):
 * d_rows[n_runs] result rows (clock = computations for unit costs; status DTR_OK
 * when all N nodes were revealed); d_parents: for run i at offset sum_{k<i} n_k,
 * parents[t] = the parent of node t (0xFFFFFFFF for t0 and for unrevealed
 * nodes); d_trace: eviction records at each run's trace_offset (may be NULL when
 * every trace_cap is 0).  Returns DTR_E_INVAL / DTR_E_CAPACITY (ws too small) /
 * DTR_E_CUDA; per-run failures are reported in the rows. */
int dtr_adversary_batch(const dtr_adversary *d_runs, const dtr_adversary *h_runs, uint32_t n_runs, void *d_ws,
                        uint64_t ws_bytes, dtr_result *d_rows, uint32_t *d_parents, dtr_evict_rec *d_trace,
                        void *stream);

/* ---------------------------------------------------------------------------
 * Per-call runtime: the simrd external API, one call at a time.
 * The same device engine is fed one record per call; all state lives in
 * device memory owned by the runtime.  Calls are synchronous.
 * ------------------------------------------------------------------------- */
typedef struct dtr_runtime dtr_runtime;

typedef struct {
  uint64_t budget;         /* R.B */
  uint64_t seed;           /* DTR_H_RANDOM */
  uint64_t max_decisions;  /* 0 = unlimited */
  uint64_t trace_cap;      /* decisions kept for dtr_trace (0 = none) */
  uint32_t heuristic;      /* dtr_heuristic */
  uint32_t thrash_kill;    /* 0 = off */
  uint32_t cap_tensors;    /* preallocated tensor capacity (> 0) */
  uint32_t cap_edges;      /* preallocated parent-edge capacity */
  int device;              /* CUDA device ordinal */
  uint32_t dealloc;        /* dtr_dealloc */
  void *stream;            /* cudaStream_t for all work (NULL = legacy default) */
} dtr_config;

/* Create a runtime (allocates device memory).  DTR_E_INVAL on bad config. */
int dtr_create(const dtr_config *cfg, dtr_runtime **out);
int dtr_destroy(dtr_runtime *rt);

/* make_tensor(f, P): new tensor of `mem` and `compute` whose
 * parents are `parents[0..n_parents)` (host array; duplicates are dropped,
 * first occurrence kept -- P is a set).  Computes it (evicting as
 * needed).  *out_id receives the new id.  DTR_E_INVAL: mem/compute 0 or an
 * unknown parent (no state change).  DTR_E_PRECOND: a parent has rho = 0 (no
 * state change).  DTR_E_CAPACITY: cap_tensors/cap_edges exhausted.
 * DTR_E_OOM / DTR_E_THRASH / DTR_E_CAPACITY(clock): sticky; later calls
 * return DTR_E_STATE. */
int dtr_compute(dtr_runtime *rt, uint32_t mem, uint32_t compute, const uint32_t *parents,
                uint32_t n_parents, uint32_t *out_id);
/* get(t): rho++ ; DTR_E_PRECOND if rho == 0. */
int dtr_get(dtr_runtime *rt, uint32_t id);
/* release(t): rho-- ; at 0 the runtime's deallocation policy
 * (dtr_config.dealloc, reading C-22): banish_V2 by default (last_access := -inf,
 * P:303-311), V1 banishing, eager eviction or nothing. */
int dtr_release(dtr_runtime *rt, uint32_t id);
/* rematerialize(t): DTR_E_PRECOND unless t is evicted. */
int dtr_rematerialize(dtr_runtime *rt, uint32_t id);
/* Output condition (reading C-11): get_internal(t) without the release. */
int dtr_ensure(dtr_runtime *rt, uint32_t id);
/* Counters and status so far (cell_id = 0). */
int dtr_stats(dtr_runtime *rt, dtr_result *out);
/* Copy up to cap recorded decisions (host buffer); *n_out = decisions recorded. */
int dtr_trace(dtr_runtime *rt, dtr_evict_rec *buf, uint64_t cap, uint64_t *n_out);

/* Test fixtures (same semantics as the oracle's): evict a pool member outside
 * free() (no decision recorded); change R.B; score every pool member at the
 * current clock (host buffers, unordered; *n_out = pool size). */
int dtr_debug_evict(dtr_runtime *rt, uint32_t id);
int dtr_debug_set_budget(dtr_runtime *rt, uint64_t budget);
int dtr_debug_scores(dtr_runtime *rt, uint64_t *num, uint64_t *den, uint32_t *ids, uint64_t cap,
                     uint64_t *n_out);

/* Residency of every tensor created so far (the state of memory visualised in
 * PAPER.md App. A, Fig. "trace"): out[t] = DTR_T_UNCOMPUTED (0:
 * MAKE started, first computation not finished), DTR_T_RESIDENT (1: t.m = T),
 * DTR_T_EVICTED (2: t.m = F after a computation) or DTR_T_BANISHED (3: removed
 * from the graph by V1 banishing).  out: host, cap bytes; *n_out =
 * tensors created (only min(cap, n) are written).  Returns DTR_OK /
 * DTR_E_INVAL / DTR_E_CUDA; no state change. */
enum { DTR_T_UNCOMPUTED = 0, DTR_T_RESIDENT = 1, DTR_T_EVICTED = 2, DTR_T_BANISHED = 3 };
int dtr_debug_state(dtr_runtime *rt, uint8_t *out, uint64_t cap, uint64_t *n_out);

#ifdef __cplusplus
}
#endif
#endif /* DTR_H */
