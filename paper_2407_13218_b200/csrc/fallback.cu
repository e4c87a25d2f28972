// Exact per-user recomputation for the batched tcgen05 path (reading R23), on the device.
//
// The batched path (scan_tc.cu) prunes with a sample-derived threshold T_u per user; its finalize
// kernel flags a user whose result is not provably exact (a candidate region overflowed, or fewer
// than K keys >= T_u were found). This kernel recomputes every flagged user exactly, on the same
// stream, with no host synchronisation: one cooperative launch of one CTA per SM that loops over
// the flagged users. Per user:
//   1. each CTA scans a contiguous item range: liveness + clauses (P:4266 semantics), dot product
//      against the user's V query vectors (max-merge, reading R12) for the passing rows only, and
//      keeps an exact CTA top-K (append keys >= the CTA threshold; when the buffer fills, radix-
//      select the K-th key and compact: keys below the K-th of K kept keys cannot enter the top-K);
//   2. grid barrier;
//   3. one CTA merges the per-CTA lists (union of exact partition top-Ks, reading R13), sorts and
//      writes the user's result over the uncertified one.
// When no user is flagged (the common case) every CTA reads the flags and exits. Scores are fp32
// dot products (R8 tolerance; int8 products and sums are exact integers in fp32 for d <= 1040).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"

namespace linr {

constexpr int kFbNT = 512;
constexpr int kFbBuf = 8192;   // soft capacity of the CTA key buffer (>= K); + kFbNT headroom per round

struct FbCtl {
  SelScratch sel;
  BucketScratch bs;
  int count;
  unsigned long long thr;
};

template <int DT>
LINR_DEV float fb_elem(const void* base, size_t i) {
  if constexpr (DT == LINR_F32) return reinterpret_cast<const float*>(base)[i];
  else if constexpr (DT == LINR_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  else if constexpr (DT == LINR_F16) return __half2float(reinterpret_cast<const __half*>(base)[i]);
  else return (float)reinterpret_cast<const int8_t*>(base)[i];
}

LINR_DEV void fb_grid_barrier(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (*(volatile unsigned int*)bar < target) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

// key getter for the CTA-wide select (a functor: lambdas here trip an nvcc 12.9 front-end assertion)
struct FbGet {
  const uint64_t* b;
  __device__ uint64_t operator()(int x) const { return b[x]; }
};

template <int DT>
__global__ void __launch_bounds__(kFbNT, 1) fallback_kernel(const __grid_constant__ FbParams p) {
  extern __shared__ __align__(16) unsigned char fsm[];
  FbCtl* ctl = reinterpret_cast<FbCtl*>(fsm);
  float* sq = reinterpret_cast<float*>(fsm + ((sizeof(FbCtl) + 15) & ~size_t(15)));
  uint64_t* buf = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sq) +
                                              (((size_t)p.V * p.dim * 4 + 15) & ~size_t(15)));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t lo = hwm * blockIdx.x / gridDim.x, hi = hwm * (blockIdx.x + 1) / gridDim.x;
  const int K = p.K, dim = p.dim, V = p.V;
  const size_t rowe = (size_t)dim;
  {   // common case: no user is flagged -- one coalesced read of the flags, then every CTA exits
    __shared__ int s_any;
    if (tid == 0) s_any = 0;
    __syncthreads();
    int any = 0;
    for (int u = tid; u < p.nu; u += kFbNT) any |= p.flags[u];
    if (any) atomicOr(&s_any, 1);
    __syncthreads();
    if (!s_any) return;   // uniform over the grid: no CTA reaches the grid barrier
  }
  unsigned int gen = 0;
  int ord = 0;   // ordinal of the flagged user (picks the merging CTA)
  for (int u = 0; u < p.nu; ++u) {
    if (!p.flags[u]) continue;   // uniform over the grid
    for (int i = tid; i < V * dim; i += kFbNT) sq[i] = fb_elem<DT>(p.q, (size_t)u * V * dim + i);
    const int ncl = p.ncl[u];
    const KClause* cl = p.cl + (size_t)u * 16;
    if (tid == 0) { ctl->count = 0; ctl->thr = 0ull; }
    __syncthreads();
    for (int64_t base = lo; base < hi; base += kFbNT) {   // uniform trip count within the CTA
      const int64_t i = base + tid;
      bool ok = i < hi && ((p.live[i >> 5] >> (i & 31)) & 1u);
      for (int c = 0; c < ncl && ok; ++c) {
        const KClause k = cl[c];
        const bool hit = (p.attr[(size_t)k.word * p.cap_pad + i] & k.mask) != 0ull;
        if (hit == (k.rev != 0u)) ok = false;
      }
      uint64_t mykey = 0ull;
      uint32_t bal = __ballot_sync(0xffffffffu, ok);
      while (bal) {   // the warp scores its passing rows one at a time (lanes split the dimension)
        const int r = __ffs(bal) - 1;
        bal &= bal - 1u;
        const int64_t row = base + warp * 32 + r;
        float best = -INFINITY;
        for (int v = 0; v < V; ++v) {
          float acc = 0.0f;
          for (int j = lane; j < dim; j += 32) acc = fmaf(fb_elem<DT>(p.emb, (size_t)row * rowe + j), sq[v * dim + j], acc);
#pragma unroll
          for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          best = fmaxf(best, acc);
        }
        if (lane == r) mykey = make_key(best, p.row0 + (uint32_t)row);
      }
      const bool cand = ok && mykey >= *(volatile unsigned long long*)&ctl->thr;
      const uint32_t cb = __ballot_sync(0xffffffffu, cand);
      if (cb) {
        const int leader = __ffs(cb) - 1;
        int pos0 = 0;
        if (lane == leader) pos0 = atomicAdd(&ctl->count, __popc(cb));
        pos0 = __shfl_sync(0xffffffffu, pos0, leader);
        if (cand) buf[pos0 + __popc(cb & lanemask_lt())] = mykey;   // a round appends <= kFbNT keys
      }
      __syncthreads();
      const int n = ctl->count;
      if (n > kFbBuf) {   // exact compaction to the K best keys
        const uint64_t T = block_select_ge<kFbNT>(FbGet{buf}, n, K, &ctl->sel);
        block_compact_ge<kFbNT>(buf, n, T, &ctl->sel);
        if (tid == 0) { ctl->count = K; ctl->thr = T; }
        __syncthreads();
      }
    }
    int n = ctl->count;
    if (n > K) {
      const uint64_t T = block_select_ge<kFbNT>(FbGet{buf}, n, K, &ctl->sel);
      n = block_compact_ge<kFbNT>(buf, n, T, &ctl->sel);
    }
    const int par = ord & 1;   // lists alternate so the merge of user j overlaps the scan of user j+1
    uint64_t* my = p.lists + ((size_t)par * gridDim.x + blockIdx.x) * K;
    for (int j = tid; j < K; j += kFbNT) my[j] = j < n ? buf[j] : 0ull;
    gen += gridDim.x;
    fb_grid_barrier(p.bar, gen);
    if ((int)blockIdx.x == ord % (int)gridDim.x) {
      // ---- merge: the K-th largest of the grid's lists, then sort the K survivors
      const uint64_t* all = p.lists + (size_t)par * gridDim.x * K;
      const int tot = (int)gridDim.x * K;
      int nz = 0;
      for (int j = tid; j < tot; j += kFbNT) nz += all[j] != 0ull;
      for (int o = 16; o; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
      if (tid == 0) ctl->count = 0;
      __syncthreads();
      if (lane == 0) atomicAdd(&ctl->count, nz);
      __syncthreads();
      const int nnz = ctl->count;
      __syncthreads();
      uint64_t T = 1ull;   // keep every nonzero key
      if (nnz > K) T = block_select_ge<kFbNT>(FbGet{all}, tot, K, &ctl->sel);
      if (tid == 0) ctl->count = 0;
      __syncthreads();
      for (int j0 = 0; j0 < tot; j0 += kFbNT) {
        const int j = j0 + tid;
        const uint64_t v = j < tot ? all[j] : 0ull;
        const bool keep = v != 0ull && v >= T;
        const uint32_t kb = __ballot_sync(0xffffffffu, keep);
        if (kb) {
          const int leader = __ffs(kb) - 1;
          int b0 = 0;
          if (lane == leader) b0 = atomicAdd(&ctl->count, __popc(kb));
          b0 = __shfl_sync(0xffffffffu, b0, leader);
          if (keep) buf[b0 + __popc(kb & lanemask_lt())] = v;
        }
      }
      __syncthreads();
      const int m = ctl->count;   // == min(K, nnz)
      uint64_t* sorted = buf + 2048;
      if (!block_bucket_sort_desc<kFbNT>(buf, m, sorted, &ctl->bs)) {
        const int P2 = next_pow2(m > 64 ? m : 64);
        for (int j = m + tid; j < P2; j += kFbNT) buf[j] = 0ull;
        __syncthreads();
        block_sort_desc<kFbNT>(buf, P2);
        sorted = buf;
      }
      for (int j = tid; j < K; j += kFbNT) {
        const int64_t at = (int64_t)u * K + j;
        if (p.out_keys) {
          p.out_keys[at] = j < m ? sorted[j] : 0ull;
        } else if (j < m) {
          p.out_ids[at] = key_id(sorted[j]);
          p.out_scores[at] = key_score(sorted[j]);
        } else {
          p.out_ids[at] = -1;
          p.out_scores[at] = -INFINITY;
        }
      }
      if (tid == 0) atomicAdd(&p.hdr->tc_fallbacks, 1ull);
      __syncthreads();
    }
    ++ord;
  }
}

size_t fallback_smem(int V, int dim) {
  return ((sizeof(FbCtl) + 15) & ~size_t(15)) + (((size_t)V * dim * 4 + 15) & ~size_t(15)) +
         (size_t)(kFbBuf + kFbNT) * 8;
}

size_t fallback_ws_bytes(int grid, int K) { return (size_t)2 * grid * K * 8; }

template <int DT>
static cudaError_t launch_fb(const FbParams& p, int grid, size_t smem, cudaStream_t st) {
  auto k = fallback_kernel<DT>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kFbNT, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  FbParams pc = p;
  void* args[] = {&pc};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), grid, kFbNT, args, smem, st);
}

cudaError_t launch_fallback(int dtype, const FbParams& p, int grid, cudaStream_t st) {
  const size_t smem = fallback_smem(p.V, p.dim);
  switch (dtype) {
    case LINR_F32: return launch_fb<LINR_F32>(p, grid, smem, st);
    case LINR_F16: return launch_fb<LINR_F16>(p, grid, smem, st);
    case LINR_BF16: return launch_fb<LINR_BF16>(p, grid, smem, st);
    case LINR_I8: return launch_fb<LINR_I8>(p, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace linr
