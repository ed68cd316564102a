// Row-block kernel instantiations for d = 2 (see rowblk.cuh).
#include "rowblk.cuh"

namespace cwr {

PipeFn rowblk_fn_2d(int M, int V, bool full_tile) {
  if (M == 3) return rowblk_fn_v<2, 3>(V, full_tile);
  if (M == 4) return rowblk_fn_v<2, 4>(V, full_tile);
  return nullptr;
}

cudaError_t rowblk_upload_sigma_2d(const double* packed, size_t bytes, size_t offset) {
  return cudaMemcpyToSymbol(c_sig, packed, bytes, offset);
}

}  // namespace cwr
