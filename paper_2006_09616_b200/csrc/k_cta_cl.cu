// k_cta_cl.cu -- K6 with the K5 closure pass (see k_cta.cuh).
#include "k_cta.cuh"

namespace dtr {
cudaError_t cta_set_attrs_cl() {
  cudaError_t e = cudaFuncSetAttribute(cta_engine<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(cta_engine_g<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX);
}

cudaError_t launch_cta_cl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 c0,
                        char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace) {
  cta_engine<true><<<n_blocks, CTA_THREADS, smem, st>>>(words, cells, c0, n_blocks, ws, ws_bytes, rows, trace, smem);
  return cudaGetLastError();
}

cudaError_t launch_cta_g_cl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells,
                              u32 c0, char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace) {
  cta_engine_g<true><<<n_blocks, CTA_G_THREADS, smem, st>>>(words, cells, c0, n_blocks, ws, ws_bytes, rows, trace, smem);
  return cudaGetLastError();
}

#ifdef DTR_PROFILE
cudaError_t prof_read_cta_cl(unsigned long long *out, int reset) {
  unsigned long long v[PROF_N];
  cudaError_t e = cudaMemcpyFromSymbol(v, g_prof, sizeof v);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < PROF_N; i++) out[i] += v[i];
  if (reset) { unsigned long long z[PROF_N] = {0}; e = cudaMemcpyToSymbol(g_prof, z, sizeof z); }
  return e;
}
#endif
}  // namespace dtr
