// dtr.cu -- host side of libdtr.so: the C ABI of include/dtr.h.  No kernels
// here: they live in k_cta.cu (K6), k_grid.cu (K7, K3+K4 alone), k_percall.cu
// and k_adv.cu (K8), compiled as separate translation units and reached
// through the launchers declared in kcommon.cuh.
#include "kcommon.cuh"
#include <mutex>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges show up in nsys / ncu --nvtx, no-ops otherwise

namespace {
struct NvtxRange {   // one range per host entry point (RAII: every return path pops it)
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace dtr;

// ===========================================================================
// Host ABI
// ===========================================================================
static thread_local char g_cuda_err[256] = "";

static int cuda_fail(cudaError_t e) {
  snprintf(g_cuda_err, sizeof g_cuda_err, "%s", cudaGetErrorString(e));
  return DTR_E_CUDA;
}
#define CK(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return cuda_fail(_e); } while (0)

extern "C" {

const char *dtr_strerror(int code) {
  switch (code) {
    case DTR_OK: return "ok";
    case DTR_E_INVAL: return "invalid argument";
    case DTR_E_PRECOND: return "precondition violated";
    case DTR_E_OOM: return "out of memory (pool empty while over budget)";
    case DTR_E_THRASH: return "thrash kill-switch";
    case DTR_E_CAPACITY: return "capacity exceeded";
    case DTR_E_STATE: return "runtime stopped by an earlier error";
    case DTR_E_CUDA: return "CUDA error";
    case DTR_E_DECISION_CAP: return "decision cap reached";
  }
  return "unknown";
}

const char *dtr_last_cuda_error(void) { return g_cuda_err; }

int dtr_version(void) { return 1; }

#ifdef DTR_PROFILE
int dtr_debug_profile(unsigned long long *out, int reset) {
  for (int i = 0; i < 32; i++) out[i] = 0;
  CK(prof_read_cta_cl(out, reset));
  CK(prof_read_cta_nocl(out, reset));
  CK(prof_read_grid(out, reset));
  CK(prof_read_percall(out, reset));
  CK(prof_read_adv(out, reset));
  return DTR_OK;
}
#endif

int dtr_batch_workspace_bytes(const uint32_t *dims, uint32_t n_cells, uint32_t engine, uint64_t *bytes_out) {
  if (!bytes_out || (n_cells && !dims) || (engine != DTR_ENGINE_CTA && engine != DTR_ENGINE_GRID)) return DTR_E_INVAL;
  u64 cur = WS_HEADER, mx = 0;
  for (u32 i = 0; i < n_cells; i++) {
    if (!valid_heuristic(dims[3 * i + 2])) return DTR_E_INVAL;
    u64 b = cell_bytes(dims[3 * i], dims[3 * i + 1], dims[3 * i + 2], engine);
    if (b == 0) return DTR_E_CAPACITY;                 // does not fit 32-bit word offsets
    if (engine == DTR_ENGINE_GRID) mx = b > mx ? b : mx;
    else cur += b;
  }
  *bytes_out = engine == DTR_ENGINE_GRID ? cur + mx : cur;
  return DTR_OK;
}

static int cta_class_of(u32 n, u32 E, u32 heur) {
  const u64 s = cta_smem_need(n, E, heur);
  return s <= 48 * 1024 - 1024 ? 0 : (s <= CTA_SMEM_MAX ? 1 : 2);
}

int dtr_cta_class(uint32_t n_tensors, uint32_t n_edges, uint32_t heuristic, uint32_t *class_out) {
  if (!class_out || !valid_heuristic(heuristic)) return DTR_E_INVAL;
  *class_out = (uint32_t)cta_class_of(n_tensors, n_edges, heuristic);
  return DTR_OK;
}

// Per-device host state: forked class streams and events, SM count, kernel
// attributes, the occupancy of the cooperative kernels and the probe switches
// (read once).  Created on first use for the calling thread's current device
// under std::call_once, so concurrent first calls and several devices in one
// process are safe.  Every entry point works on the current device: the
// caller's buffers and stream must belong to it.
struct DevState {
  std::once_flag once;
  int err;                       // DTR_OK or the init failure
  int sm_count, grid_per_sm, pa_per_sm, grid_blocks_env;
  bool pack_ctas, debug;
  cudaStream_t cls_st[3];
  cudaEvent_t fork_ev, join_ev[3];
};
#define DTR_MAX_DEVICES 64
static DevState g_dev[DTR_MAX_DEVICES];

static int dev_init(DevState &d, int dev) {
  CK(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev));
  CK(cta_set_attrs_cl());
  CK(cta_set_attrs_nocl());
  CK(adv_set_attrs());
  CK(grid_occupancy(&d.grid_per_sm, &d.pa_per_sm));
  for (int k = 0; k < 3; k++) {
    CK(cudaStreamCreateWithFlags(&d.cls_st[k], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&d.join_ev[k], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&d.fork_ev, cudaEventDisableTiming));
  // the default pool keeps its memory between dtr_replay_batch_host calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  const char *e = getenv("DTR_GRID_BLOCKS");          // probes only
  d.grid_blocks_env = e ? atoi(e) : 0;
  d.pack_ctas = getenv("DTR_PACK_CTAS") != nullptr;   // probes only
  d.debug = getenv("DTR_DEBUG") != nullptr;
  return DTR_OK;
}

static int dev_state(DevState **out) {
  int dev;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= DTR_MAX_DEVICES) return DTR_E_INVAL;
  DevState &d = g_dev[dev];
  std::call_once(d.once, [&] {
    // the runtime binds the device to this thread already; keep it current
    d.err = dev_init(d, dev);
  });
  *out = &d;
  return d.err;
}

static int grid_blocks(int *blocks) {
  DevState *ds;
  int rc = dev_state(&ds);
  if (rc) return rc;
  if (ds->grid_per_sm < 1) return DTR_E_CUDA;
  *blocks = ds->sm_count * (ds->grid_per_sm > 2 ? 2 : ds->grid_per_sm);
  if (ds->grid_blocks_env > 0 && ds->grid_blocks_env < *blocks) *blocks = ds->grid_blocks_env;
  if (*blocks > 4096) *blocks = 4096;
  return DTR_OK;
}

int dtr_replay_batch(const uint32_t *d_words, const dtr_cell *d_cells, const uint32_t *h_dims, uint32_t n_cells,
                     uint32_t engine, void *d_ws, uint64_t ws_bytes, dtr_result *d_rows, dtr_evict_rec *d_trace,
                     void *stream) {
  NvtxRange nvtx_range("dtr_replay_batch");
  if (!n_cells) return DTR_OK;
  if (!d_words || !d_cells || !h_dims || !d_ws || !d_rows) return DTR_E_INVAL;
  if (engine != DTR_ENGINE_CTA && engine != DTR_ENGINE_GRID) return DTR_E_INVAL;
  uint64_t need = 0;
  int rc = dtr_batch_workspace_bytes(h_dims, n_cells, engine, &need);
  if (rc) return rc;
  if (ws_bytes < need) return DTR_E_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)d_ws;
  if (engine == DTR_ENGINE_CTA) {
    // Consecutive cells of the same shared-memory class form one launch: small
    // (<= 48 KiB: several CTAs per SM), large (<= 225 KiB staged), global (state
    // stays in the workspace).  Classes run concurrently on forked streams.
    DevState *ds;
    rc = dev_state(&ds);
    if (rc) return rc;
    const int sm_count = ds->sm_count;
    auto cls_of = [&](u32 i, u64 *need) -> int {
      *need = cta_smem_need(h_dims[3 * i], h_dims[3 * i + 1], h_dims[3 * i + 2]);
      return cta_class_of(h_dims[3 * i], h_dims[3 * i + 1], h_dims[3 * i + 2]);
    };
    bool used[3] = {false, false, false};
    u64 first_need;
    const int c_first = cls_of(0, &first_need);
    bool single = true;
    for (u32 i = 1; i < n_cells && single; i++) { u64 nd; single = cls_of(i, &nd) == c_first; }
    if (!single) CK(cudaEventRecord(ds->fork_ev, st));
    u32 i = 0;
    while (i < n_cells) {
      u64 need;
      const int c = cls_of(i, &need);
      // global state: the per-warp slow stacks (+ the walk mirror of closure cells, if it fits)
      auto g_smem_of = [&](u32 k) -> u64 {
        const u32 n = h_dims[3 * k], E = h_dims[3 * k + 1], h = h_dims[3 * k + 2];
        const u64 m = mirror_ok(n, E, h) ? (u64)CTA_WQ_BYTES + mirror_bytes(n, E) : (u64)CTA_WQ_BYTES;
        return m <= CTA_SMEM_MAX ? m : (u64)CTA_WQ_BYTES;
      };
      u64 smem = c == 2 ? g_smem_of(i) : need;
      u32 j = i + 1;
      bool cl = uses_closure(h_dims[3 * i + 2]);
      for (; j < n_cells; j++) {
        u64 nd;
        if (cls_of(j, &nd) != c) break;
        if (c != 2 && nd > smem) smem = nd;
        if (c == 2) smem = std::max<u64>(smem, g_smem_of(j));
        cl = cl || uses_closure(h_dims[3 * j + 2]);
      }
      smem = (smem + 15) & ~15ull;
      // at most one cell per SM: reserve more than half an SM's shared memory so
      // no two CTAs (each a latency-bound single-leader simulation) share an SM
      if (c != 2 && n_cells <= (u32)sm_count && !ds->pack_ctas) smem = std::max<u64>(smem, 116u * 1024u);
      cudaStream_t ls = st;
      if (!single) {
        ls = ds->cls_st[c];
        if (!used[c]) { CK(cudaStreamWaitEvent(ls, ds->fork_ev, 0)); used[c] = true; }
      }
      if (ds->debug) fprintf(stderr, "dtr: cta launch cells [%u,%u) class %d smem %llu\n", i, j, c, smem);
      // the K5 closure pass is compiled only into the _cl instantiation
      if (c == 2) {           // state in global memory: the wide instantiation
        if (cl) CK(launch_cta_g_cl(j - i, (u32)smem, ls, d_words, d_cells, i, ws, ws_bytes, d_rows, d_trace));
        else CK(launch_cta_g_nocl(j - i, (u32)smem, ls, d_words, d_cells, i, ws, ws_bytes, d_rows, d_trace));
      } else {
        if (cl) CK(launch_cta_cl(j - i, (u32)smem, ls, d_words, d_cells, i, ws, ws_bytes, d_rows, d_trace));
        else CK(launch_cta_nocl(j - i, (u32)smem, ls, d_words, d_cells, i, ws, ws_bytes, d_rows, d_trace));
      }
      i = j;
    }
    if (!single) {
      for (int k = 0; k < 3; k++) {
        if (!used[k]) continue;
        CK(cudaEventRecord(ds->join_ev[k], ds->cls_st[k]));
        CK(cudaStreamWaitEvent(st, ds->join_ev[k], 0));
      }
    }
  } else {
    int blocks;
    rc = grid_blocks(&blocks);
    if (rc) return rc;
    for (u32 i = 0; i < n_cells; i++) {
      CK(launch_grid(blocks, st, d_words, d_cells, i, ws, ws_bytes, d_rows, d_trace));
    }
  }
  return DTR_OK;
}

int dtr_pool_argmin(const uint32_t *d_log, uint32_t heuristic, void *d_ws, uint64_t *d_out, void *stream) {
  NvtxRange nvtx_range("dtr_pool_argmin");
  if (!d_log || !d_ws || !d_out || !valid_heuristic(heuristic)) return DTR_E_INVAL;
  DevState *ds;
  int rc = dev_state(&ds);
  if (rc) return rc;
  int blocks = ds->sm_count * (ds->pa_per_sm < 1 ? 1 : ds->pa_per_sm);
  if (blocks > 4096) blocks = 4096;
  CK(launch_pool_argmin(blocks, (cudaStream_t)stream, d_log, heuristic, (char *)d_ws, (u64 *)d_out));
  return DTR_OK;
}

int dtr_replay_batch_host(const uint32_t *h_words, uint64_t n_words, const dtr_cell *h_cells, uint32_t n_cells,
                          uint32_t engine, dtr_result *h_rows, dtr_evict_rec *h_trace, uint64_t trace_total,
                          void *stream) {
  NvtxRange nvtx_range("dtr_replay_batch_host");
  if (!n_cells) return DTR_OK;
  if (!h_words || !h_cells || !h_rows) return DTR_E_INVAL;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<u32> dims(3 * (size_t)n_cells);
  u32 max_n = 0;
  for (u32 i = 0; i < n_cells; i++) {
    u64 o = h_cells[i].log_offset;
    if (o + DTR_LOG_HEADER_WORDS > n_words || h_words[o] != DTR_LOG_MAGIC) return DTR_E_INVAL;
    dims[3 * i] = h_words[o + 2];
    dims[3 * i + 1] = h_words[o + 3];
    dims[3 * i + 2] = h_cells[i].heuristic;
    max_n = std::max(max_n, h_words[o + 2]);
  }
  if (engine == 0) engine = max_n >= DTR_GRID_MIN_TENSORS ? DTR_ENGINE_GRID : DTR_ENGINE_CTA;
  uint64_t ws_bytes = 0;
  int rc = dtr_batch_workspace_bytes(dims.data(), n_cells, engine, &ws_bytes);
  if (rc) return rc;
  DevState *ds;
  rc = dev_state(&ds);
  if (rc) return rc;
  u32 *d_words = nullptr;
  dtr_cell *d_cells = nullptr;
  dtr_result *d_rows = nullptr;
  dtr_evict_rec *d_trace = nullptr;
  void *d_ws = nullptr;
  cudaError_t e = cudaSuccess;
  // one cleanup path: whatever was allocated is freed (stream-ordered) and the
  // stream is synchronised before returning, on success and on failure
#define HCK(x) do { if (e == cudaSuccess) e = (x); } while (0)
  HCK(cudaMallocAsync((void **)&d_words, n_words * 4, st));
  HCK(cudaMallocAsync((void **)&d_cells, (size_t)n_cells * sizeof(dtr_cell), st));
  HCK(cudaMallocAsync((void **)&d_rows, (size_t)n_cells * sizeof(dtr_result), st));
  if (h_trace && trace_total) HCK(cudaMallocAsync((void **)&d_trace, trace_total * sizeof(dtr_evict_rec), st));
  HCK(cudaMallocAsync(&d_ws, ws_bytes, st));
  HCK(cudaMemcpyAsync(d_words, h_words, n_words * 4, cudaMemcpyHostToDevice, st));
  HCK(cudaMemcpyAsync(d_cells, h_cells, (size_t)n_cells * sizeof(dtr_cell), cudaMemcpyHostToDevice, st));
  if (e == cudaSuccess) {
    rc = dtr_replay_batch(d_words, d_cells, dims.data(), n_cells, engine, d_ws, ws_bytes, d_rows, d_trace, st);
    if (rc == DTR_OK) {
      HCK(cudaMemcpyAsync(h_rows, d_rows, (size_t)n_cells * sizeof(dtr_result), cudaMemcpyDeviceToHost, st));
      if (d_trace) HCK(cudaMemcpyAsync(h_trace, d_trace, trace_total * sizeof(dtr_evict_rec), cudaMemcpyDeviceToHost, st));
    }
  }
  if (d_words) cudaFreeAsync(d_words, st);
  if (d_cells) cudaFreeAsync(d_cells, st);
  if (d_rows) cudaFreeAsync(d_rows, st);
  if (d_trace) cudaFreeAsync(d_trace, st);
  if (d_ws) cudaFreeAsync(d_ws, st);
  const cudaError_t es = cudaStreamSynchronize(st);
#undef HCK
  if (e == cudaSuccess) e = es;
  if (e != cudaSuccess) return cuda_fail(e);
  return rc;
}

// ---------------------------------------------------------------------------
// Theorem 2 adversary batches
// ---------------------------------------------------------------------------
int dtr_adversary_workspace_bytes(const dtr_adversary *h_runs, uint32_t n_runs, uint64_t *bytes) {
  if (!bytes || (n_runs && !h_runs)) return DTR_E_INVAL;
  u64 total = 256;
  for (u32 i = 0; i < n_runs; i++) {
    const dtr_adversary &r = h_runs[i];
    if (r.n == 0 || r.n >= (1u << 27) || r.budget < 3 || !valid_heuristic(r.heuristic)) return DTR_E_INVAL;
    total += adv_bytes(r);
  }
  *bytes = total;
  return DTR_OK;
}

int dtr_adversary_batch(const dtr_adversary *d_runs, const dtr_adversary *h_runs, uint32_t n_runs, void *d_ws,
                        uint64_t ws_bytes, dtr_result *d_rows, uint32_t *d_parents, dtr_evict_rec *d_trace,
                        void *stream) {
  NvtxRange nvtx_range("dtr_adversary_batch");
  if (!d_runs || !h_runs || !d_rows || !d_parents || (n_runs && !d_ws)) return DTR_E_INVAL;
  if (n_runs == 0) return DTR_OK;
  uint64_t need = 0;
  int rc = dtr_adversary_workspace_bytes(h_runs, n_runs, &need);
  if (rc) return rc;
  if (ws_bytes < need) return DTR_E_CAPACITY;
  DevState *ds;
  rc = dev_state(&ds);
  if (rc) return rc;
  u64 smem = 0;
  for (u32 i = 0; i < n_runs; i++) {
    Lay L;
    AdvLay A;
    adv_layout(L, A, h_runs[i].n, h_runs[i].budget, h_runs[i].heuristic);
    const u64 b = (u64)A.words * 4;
    if (b <= CTA_SMEM_MAX && b > smem) smem = b;
  }
  smem = (smem + 15) & ~15ull;
  CK(launch_adv(n_runs, (u32)smem, (cudaStream_t)stream, d_runs, (char *)d_ws, ws_bytes, d_rows, d_parents, d_trace));
  return DTR_OK;
}

// ---------------------------------------------------------------------------
// per-call runtime
// ---------------------------------------------------------------------------
struct dtr_runtime {
  dtr_config cfg;
  cudaStream_t st;
  Lay L;
  u32 *d_ws;
  Scalars *d_sc;
  dtr_evict_rec *d_trace;
  u64 *d_num, *d_den;
  u32 *d_ids;
  u64 score_cap;
  u32 edges;      // parent edges written so far
  Scalars hs;     // mirror of the device scalars after the last call
};

static int rt_sync_scalars(dtr_runtime *rt) {
  CK(cudaMemcpyAsync(&rt->hs, rt->d_sc, sizeof(Scalars), cudaMemcpyDeviceToHost, rt->st));
  CK(cudaStreamSynchronize(rt->st));
  return DTR_OK;
}

static int rt_launch(dtr_runtime *rt, u32 init, u32 op_word) {
  PercallArgs a;
  a.L = rt->L; a.base = rt->d_ws; a.sc = rt->d_sc;
  a.trace = rt->d_trace; a.onum = rt->d_num; a.oden = rt->d_den; a.oid = rt->d_ids;
  a.init = init;
  if (!init) {
    CK(cudaMemcpyAsync((char *)rt->d_sc + offsetof(Scalars, pending_op), &op_word, 4, cudaMemcpyHostToDevice,
                       rt->st));
  }
  CK(launch_percall(a, rt->st));
  return rt_sync_scalars(rt);
}

int dtr_create(const dtr_config *cfg, dtr_runtime **out) {
  if (!cfg || !out || cfg->cap_tensors == 0 || !valid_heuristic(cfg->heuristic) || cfg->dealloc > DEALLOC_IGNORE)
    return DTR_E_INVAL;
  if (cfg->cap_tensors >= (1u << 29)) return DTR_E_INVAL;
  dtr_runtime *rt = new dtr_runtime();
  rt->cfg = *cfg;
  rt->st = (cudaStream_t)cfg->stream;
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) { delete rt; return cuda_fail(e); }
  const u32 n = cfg->cap_tensors, E = cfg->cap_edges;
  if (!make_layout(rt->L, n, E, cfg->heuristic, 1, CTA_THREADS / 32)) { delete rt; return DTR_E_INVAL; }
  rt->score_cap = (u64)n + 1;
#define AL(p, bytes) do { e = cudaMalloc((void **)&(p), (bytes)); if (e != cudaSuccess) { dtr_destroy(rt); return cuda_fail(e); } } while (0)
  AL(rt->d_ws, (u64)rt->L.words * 4);
  AL(rt->d_sc, sizeof(Scalars));
  AL(rt->d_num, 8 * rt->score_cap);
  AL(rt->d_den, 8 * rt->score_cap);
  AL(rt->d_ids, 4 * rt->score_cap);
  if (cfg->trace_cap) AL(rt->d_trace, cfg->trace_cap * sizeof(dtr_evict_rec));
#undef AL
  rt->edges = 0;
  Scalars s;
  memset(&s, 0, sizeof s);
  s.B = cfg->budget; s.seed = cfg->seed; s.max_decisions = cfg->max_decisions; s.trace_cap = cfg->trace_cap;
  s.heuristic = cfg->heuristic; s.thrash_kill = cfg->thrash_kill; s.dealloc = cfg->dealloc;
  s.trace_hash = 14695981039346656037ull;
  norm_scalars(s);
  e = cudaMemcpyAsync(rt->d_sc, &s, sizeof s, cudaMemcpyHostToDevice, rt->st);
  if (e != cudaSuccess) { dtr_destroy(rt); return cuda_fail(e); }
  int rc = rt_launch(rt, 1, 0);
  if (rc) { dtr_destroy(rt); return rc; }
  *out = rt;
  return DTR_OK;
}

int dtr_destroy(dtr_runtime *rt) {
  if (!rt) return DTR_OK;
  cudaFree(rt->d_ws); cudaFree(rt->d_sc); cudaFree(rt->d_num); cudaFree(rt->d_den); cudaFree(rt->d_ids);
  if (rt->d_trace) cudaFree(rt->d_trace);
  delete rt;
  return DTR_OK;
}

static bool sticky(const dtr_runtime *rt) { return rt->hs.status != ST_OK && rt->hs.status != ST_PRECOND; }

static int rt_op(dtr_runtime *rt, u32 op, u32 id) {
  if (!rt) return DTR_E_INVAL;
  if (sticky(rt)) return DTR_E_STATE;
  if (id >= (1u << 29)) return DTR_E_PRECOND;   // unknown tensor (device checks id < n_alloc)
  int rc = rt_launch(rt, 0, (op << 29) | id);
  if (rc) return rc;
  return (int)rt->hs.last_rc;
}

int dtr_compute(dtr_runtime *rt, uint32_t mem, uint32_t compute, const uint32_t *parents, uint32_t n_parents,
                uint32_t *out_id) {
  if (!rt || mem == 0 || compute == 0 || compute > 0x7FFFFFFFu || (n_parents && !parents)) return DTR_E_INVAL;
  if (sticky(rt)) return DTR_E_STATE;
  const u32 t = rt->hs.n_alloc;
  std::vector<u32> ps;
  ps.reserve(n_parents);
  for (u32 j = 0; j < n_parents; j++) {
    if (parents[j] >= t) return DTR_E_INVAL;
    if (std::find(ps.begin(), ps.end(), parents[j]) == ps.end()) ps.push_back(parents[j]);
  }
  if (t >= rt->cfg.cap_tensors) return DTR_E_CAPACITY;
  if ((u64)rt->edges + ps.size() > rt->cfg.cap_edges) return DTR_E_CAPACITY;
  const uint4 sr = make_uint4(mem, compute, 0, 0);            // {mem, cost, la, nev}
  const uint2 pr = make_uint2(rt->edges, (u32)ps.size());     // {par_off, npar}
  CK(cudaMemcpyAsync(rt->d_ws + rt->L.srec + 4 * (u64)t, &sr, 16, cudaMemcpyHostToDevice, rt->st));
  CK(cudaMemcpyAsync(rt->d_ws + rt->L.arec + 4 * (u64)t, &pr, 8, cudaMemcpyHostToDevice, rt->st));
  if (!ps.empty())
    CK(cudaMemcpyAsync(rt->d_ws + rt->L.par + rt->edges, ps.data(), 4 * ps.size(), cudaMemcpyHostToDevice, rt->st));
  int rc = rt_launch(rt, 0, (OP_MAKE << 29) | t);
  if (rc) return rc;
  if (rt->hs.n_alloc == t + 1) {
    rt->edges += (u32)ps.size();
    if (out_id) *out_id = t;
  }
  return (int)rt->hs.last_rc;
}

int dtr_get(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_GET, id); }
int dtr_release(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_RELEASE, id); }
int dtr_rematerialize(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_REMAT, id); }
int dtr_ensure(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_ENSURE, id); }
int dtr_debug_evict(dtr_runtime *rt, uint32_t id) { return rt_op(rt, OP_DEBUG_EVICT, id); }

int dtr_debug_set_budget(dtr_runtime *rt, uint64_t budget) {
  if (!rt) return DTR_E_INVAL;
  CK(cudaMemcpyAsync((char *)rt->d_sc + offsetof(Scalars, B), &budget, 8, cudaMemcpyHostToDevice, rt->st));
  return rt_sync_scalars(rt);
}

int dtr_debug_scores(dtr_runtime *rt, uint64_t *num, uint64_t *den, uint32_t *ids, uint64_t cap, uint64_t *n_out) {
  if (!rt || !n_out) return DTR_E_INVAL;
  int rc = rt_launch(rt, 0, (u32)OP_SCORES << 29);
  if (rc) return rc;
  u64 k = rt->hs.n_scores;
  *n_out = k;
  u64 m = std::min<u64>(k, (u64)cap);
  if (m) {
    CK(cudaMemcpyAsync(num, rt->d_num, 8 * m, cudaMemcpyDeviceToHost, rt->st));
    CK(cudaMemcpyAsync(den, rt->d_den, 8 * m, cudaMemcpyDeviceToHost, rt->st));
    CK(cudaMemcpyAsync(ids, rt->d_ids, 4 * m, cudaMemcpyDeviceToHost, rt->st));
    CK(cudaStreamSynchronize(rt->st));
  }
  return DTR_OK;
}

int dtr_debug_state(dtr_runtime *rt, uint8_t *out, uint64_t cap, uint64_t *n_out) {
  if (!rt || !n_out || (cap && !out)) return DTR_E_INVAL;
  int rc = rt_sync_scalars(rt);
  if (rc) return rc;
  const u64 n = rt->hs.n_alloc;
  *n_out = n;
  const u64 m = std::min<u64>(n, cap);
  if (!m) return DTR_OK;
  std::vector<u32> st(m);
  CK(cudaMemcpyAsync(st.data(), rt->d_ws + rt->L.state, 4 * m, cudaMemcpyDeviceToHost, rt->st));
  CK(cudaStreamSynchronize(rt->st));
  for (u64 t = 0; t < m; t++) {   // state word: bit31 material, bit30 computed once, bit29 banished
    const u32 w = st[t];
    out[t] = (w & B_BIT) ? DTR_T_BANISHED : (w & M_BIT) ? DTR_T_RESIDENT : (w & O_BIT) ? DTR_T_EVICTED : DTR_T_UNCOMPUTED;
  }
  return DTR_OK;
}

int dtr_stats(dtr_runtime *rt, dtr_result *out) {
  if (!rt || !out) return DTR_E_INVAL;
  int rc = rt_sync_scalars(rt);
  if (rc) return rc;
  const Scalars &s = rt->hs;
  memset(out, 0, sizeof *out);
  out->status = s.status; out->records_done = s.records_done; out->n_trace = (u32)s.trace_n;
  out->clock = s.clock; out->base = s.base_so_far; out->decisions = s.decisions; out->remats = s.remats;
  out->computations = s.computations; out->peak_M = s.peak_M; out->trace_hash = s.trace_hash;
  return DTR_OK;
}

int dtr_trace(dtr_runtime *rt, dtr_evict_rec *buf, uint64_t cap, uint64_t *n_out) {
  if (!rt || !n_out) return DTR_E_INVAL;
  u64 k = rt->hs.trace_n;
  *n_out = k;
  u64 m = std::min<u64>(k, (u64)cap);
  if (m && rt->d_trace) {
    CK(cudaMemcpyAsync(buf, rt->d_trace, m * sizeof(dtr_evict_rec), cudaMemcpyDeviceToHost, rt->st));
    CK(cudaStreamSynchronize(rt->st));
  }
  return DTR_OK;
}

}  // extern "C"

