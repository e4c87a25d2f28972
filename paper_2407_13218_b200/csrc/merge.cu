// Standalone merge kernel (one CTA per user): used for cross-shard merges (linr_merge_keys) and
// for multi-group scans. The algorithm lives in merge.cuh (shared with the scan kernel's tail).
#include "merge.cuh"

namespace linr {

constexpr int kMergeNT = 512;

__global__ void __launch_bounds__(kMergeNT, 1) merge_kernel(const __grid_constant__ MergeParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  merge_user<kMergeNT>(p, blockIdx.x, smem_raw);
}

cudaError_t launch_merge(const MergeParams& p, int B, cudaStream_t st) {
  const size_t smem = merge_smem_bytes();
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(merge_kernel), smem);
  if (e != cudaSuccess) return e;
  merge_kernel<<<B, kMergeNT, smem, st>>>(p);
  return cudaGetLastError();
}

size_t merge_smem() { return merge_smem_bytes(); }

}  // namespace linr
