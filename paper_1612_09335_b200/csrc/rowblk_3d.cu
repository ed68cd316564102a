// Row-block kernel instantiations for d = 3 (see rowblk.cuh).
#include "rowblk.cuh"

namespace cwr {

PipeFn rowblk_fn_3d(int M, int V, bool full_tile) {
  if (M == 2) return rowblk_fn_v<3, 2>(V, full_tile);
  if (M == 3) return rowblk_fn_v<3, 3>(V, full_tile);
  return nullptr;
}

cudaError_t rowblk_upload_sigma_3d(const double* packed, size_t bytes, size_t offset) {
  return cudaMemcpyToSymbol(c_sig, packed, bytes, offset);
}

}  // namespace cwr

#ifdef CWR_TRACE
extern "C" int cwreco_debug_rb_trace(long long* out) {  // tuning builds only: [64][16] clock64 stamps of CTA 0
  return (int)cudaMemcpyFromSymbol(out, cwr::g_rb_trace, sizeof(cwr::g_rb_trace));
}
#endif
