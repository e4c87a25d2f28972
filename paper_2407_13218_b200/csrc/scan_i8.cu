// Explicit instantiation of the GEMV scan kernels for dtype LINR_I8 (split per dtype for parallel builds).
#include "scan_dispatch.cuh"

namespace linr {
cudaError_t launch_scan_gemv_i8(int dim, int nqv, const ScanParams& p, int grid, size_t smem, cudaStream_t st) {
  return ScanDispatch<LINR_I8>::launch(dim, nqv, p, grid, smem, st);
}
ScanCfg scan_cfg_i8(int dim, int nqv) { return ScanDispatch<LINR_I8>::cfg(dim, nqv); }
}  // namespace linr
