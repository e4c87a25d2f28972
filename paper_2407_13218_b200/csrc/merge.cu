// Standalone merge kernel (one CTA per user): used for cross-shard merges (linr_merge_keys) and
// for multi-group scans. The algorithm lives in merge.cuh (shared with the scan kernel's tail).
#include "merge.cuh"

namespace linr {

constexpr int kMergeNT = 512;

__global__ void __launch_bounds__(kMergeNT, 1) merge_kernel(const __grid_constant__ MergeParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // launched as a programmatic dependent of the scan: wait until the scan grid has completed and
  // its results are visible (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.gate != nullptr && *(volatile const int*)p.gate != p.gate_want) return;   // path not chosen
  merge_user<kMergeNT>(p, blockIdx.x, smem_raw);
}

cudaError_t launch_merge(const MergeParams& p0, int B, cudaStream_t st, bool pdl) {
  MergeParams p = p0;
  p.bucket_sort = env_int("LINR_MERGE_BUCKET", 0);
  const size_t smem = merge_smem_bytes();
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(merge_kernel), smem);
  if (e != cudaSuccess) return e;
  if (!pdl) {
    merge_kernel<<<B, kMergeNT, smem, st>>>(p);
    return cudaGetLastError();
  }
  // programmatic dependent launch right behind the scan: the merge CTA is resident (on the SM the
  // scan leaves free) when the scan completes, instead of paying a kernel launch after it
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)B);
  cfg.blockDim = dim3(kMergeNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, merge_kernel, p);
}

size_t merge_smem() { return merge_smem_bytes(); }

}  // namespace linr
