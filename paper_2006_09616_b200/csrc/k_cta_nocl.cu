// k_cta_nocl.cu -- K6 without the K5 closure pass (see k_cta.cuh).
#include "k_cta.cuh"

namespace dtr {
cudaError_t cta_set_attrs_nocl() {
  cudaError_t e = cudaFuncSetAttribute(cta_engine<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(cta_engine_g<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTA_SMEM_MAX);
}

cudaError_t launch_cta_nocl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells, u32 c0,
                        char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace) {
  cta_engine<false><<<n_blocks, CTA_THREADS, smem, st>>>(words, cells, c0, n_blocks, ws, ws_bytes, rows, trace, smem);
  return cudaGetLastError();
}

cudaError_t launch_cta_g_nocl(u32 n_blocks, u32 smem, cudaStream_t st, const u32 *words, const dtr_cell *cells,
                              u32 c0, char *ws, u64 ws_bytes, dtr_result *rows, dtr_evict_rec *trace) {
  cta_engine_g<false><<<n_blocks, CTA_G_THREADS, smem, st>>>(words, cells, c0, n_blocks, ws, ws_bytes, rows, trace, smem);
  return cudaGetLastError();
}

#ifdef DTR_PROFILE
cudaError_t prof_read_cta_nocl(unsigned long long *out, int reset) {
  unsigned long long v[PROF_N];
  cudaError_t e = cudaMemcpyFromSymbol(v, g_prof, sizeof v);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < PROF_N; i++) out[i] += v[i];
  if (reset) { unsigned long long z[PROF_N] = {0}; e = cudaMemcpyToSymbol(g_prof, z, sizeof z); }
  return e;
}
#endif
}  // namespace dtr
