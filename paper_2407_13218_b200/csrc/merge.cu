// Merge of L sorted per-partition top-K key lists into the final top-K (one CTA per user).
//
// Used twice on the hot path: (a) after the scan, L = number of scan CTAs; (b) after the
// cross-GPU all-gather, L = number of shards (BASELINE.json north_star: "an NCCL allgather of K
// (score, id) pairs ... feeds a final merge"). Exact by reading R13: the union of the partitions'
// top-Ks contains the global top-K under the total key order (score desc, id asc).
//
// Pruned path when L*K does not fit in shared memory: the K-th largest key LB of the union of each
// list's top-m prefix is a lower bound of the global K-th key (those K keys exist), so only keys
// >= LB (a prefix of every sorted list) can be in the answer. For lists drawn from disjoint item
// ranges LB is usually the exact K-th key and ~K keys survive. If too many survive, a global radix
// select over all L*K keys is the (slow, exact) fallback.
#include "common.cuh"
#include "internal.h"

namespace linr {

constexpr int kMergeNT = 1024;
constexpr int kMergeCap = 16384;   // keys staged in shared memory (128 KB)

struct MergeCtl {
  SelScratch sel;
  int cnt;
  int total;
  unsigned long long lb;
  long long pass;
};

__device__ int gather_keys(uint64_t* dst, int cap, MergeCtl* ctl, int n_items,
                           const uint64_t* keys, int64_t stride_l, int K, uint64_t lb, int per_list) {
  // keys of list l at keys + l*stride_l, first per_list of them considered; keep nonzero keys >= lb
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) ctl->cnt = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n_items; i0 += kMergeNT) {   // uniform trip count: full-warp ballots
    const int i = i0 + tid;
    bool keep = false;
    uint64_t v = 0ull;
    if (i < n_items) {
      const int l = i / per_list, j = i - l * per_list;
      v = keys[(int64_t)l * stride_l + j];
      keep = v != 0ull && v >= lb;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (bal) {
      const int leader = __ffs(bal) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(&ctl->cnt, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, leader);
      const int pos = base + __popc(bal & lanemask_lt());
      if (keep && pos < cap) dst[pos] = v;
    }
  }
  __syncthreads();
  return ctl->cnt;
}

__global__ void __launch_bounds__(kMergeNT, 1) merge_kernel(const __grid_constant__ MergeParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MergeCtl* ctl = reinterpret_cast<MergeCtl*>(smem_raw);
  uint64_t* s = reinterpret_cast<uint64_t*>(smem_raw + ((sizeof(MergeCtl) + 15) & ~size_t(15)));
  int* lcnt = reinterpret_cast<int*>(s + kMergeCap);   // [L]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u = blockIdx.x;
  const int L = p.L, K = p.K;
  const uint64_t* base = p.keys + (int64_t)u * p.stride_u;

  // pass counts
  if (warp == 0) {
    long long acc = 0;
    for (int l = lane; l < L; l += 32) acc += p.pass[(int64_t)l * p.pstride_l + (int64_t)u * p.pstride_u];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ctl->pass = acc;
  }

  int n = -1;
  const int64_t total = (int64_t)L * K;
  if (total <= kMergeCap) {
    n = gather_keys(s, kMergeCap, ctl, (int)total, base, p.stride_l, K, 1ull, K);
  } else {
    const int m = p.m;
    int ns = gather_keys(s, kMergeCap, ctl, L * m, base, p.stride_l, K, 1ull, m);
    uint64_t lb = 0ull;
    if (ns >= K) lb = block_select_ge<kMergeNT>([s](int i) { return s[i]; }, ns, K, &ctl->sel);
    if (lb != 0ull) {
      // count keys >= lb per list (each list is sorted descending): binary search
      for (int l = tid; l < L; l += kMergeNT) {
        const uint64_t* lp = base + (int64_t)l * p.stride_l;
        int lo = 0, hi = K;   // first index with key < lb
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (lp[mid] >= lb) lo = mid + 1; else hi = mid;
        }
        lcnt[l] = lo;
      }
      if (tid == 0) ctl->total = 0;
      __syncthreads();
      int part = 0;
      for (int l = tid; l < L; l += kMergeNT) part += lcnt[l];
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0 && part) atomicAdd(&ctl->total, part);
      __syncthreads();
      if (ctl->total <= kMergeCap) {
        // gather the prefixes: warp per list
        if (tid == 0) ctl->cnt = 0;
        __syncthreads();
        for (int l = warp; l < L; l += kMergeNT / 32) {
          const int c = lcnt[l];
          int at = 0;
          if (lane == 0 && c) at = atomicAdd(&ctl->cnt, c);
          at = __shfl_sync(0xffffffffu, at, 0);
          const uint64_t* lp = base + (int64_t)l * p.stride_l;
          for (int j = lane; j < c; j += 32) s[at + j] = lp[j];
        }
        __syncthreads();
        n = ctl->cnt;
      }
    }
    if (n < 0) {
      // exact fallback: all nonzero keys, selected in global memory if they do not fit
      int n1 = gather_keys(s, kMergeCap, ctl, (int)total, base, p.stride_l, K, 1ull, K);
      if (n1 <= kMergeCap) {
        n = n1;
      } else {
        const int64_t sl = p.stride_l;
        const uint64_t T = block_select_ge<kMergeNT>(
            [base, sl, K](int i) { const int l = i / K; return base[(int64_t)l * sl + (i - l * K)]; },
            (int)total, K, &ctl->sel);
        n = gather_keys(s, kMergeCap, ctl, (int)total, base, p.stride_l, K, T, K);
      }
    }
  }

  if (n > K) {
    const uint64_t T = block_select_ge<kMergeNT>([s](int i) { return s[i]; }, n, K, &ctl->sel);
    n = block_compact_ge<kMergeNT>(s, n, T, &ctl->sel);
  }
  const int P2 = next_pow2(n > 1 ? n : 1);
  for (int i = n + tid; i < P2; i += kMergeNT) s[i] = 0ull;
  __syncthreads();
  block_sort_desc<kMergeNT>(s, P2);

  if (p.mode == 0) {
    for (int j = tid; j < K; j += kMergeNT) {
      const int64_t at = (int64_t)u * K + j;
      if (j < n) {
        p.out_ids[at] = key_id(s[j]);
        p.out_scores[at] = key_score(s[j]);
      } else {
        p.out_ids[at] = -1;
        p.out_scores[at] = -INFINITY;
      }
    }
  } else {
    for (int j = tid; j < K; j += kMergeNT) p.out_keys[(int64_t)u * K + j] = (j < n) ? s[j] : 0ull;
  }
  if (tid == 0 && p.out_pass) p.out_pass[u] = ctl->pass;
}

int merge_sample_size(int L, int K) {
  if ((int64_t)L * K <= kMergeCap) return K;
  int m = next_pow2((3 * K + L - 1) / L);
  if (m < 16) m = 16;
  if (m > K) m = K;
  while ((int64_t)L * m > kMergeCap && m > 1) m >>= 1;
  return m;
}

cudaError_t launch_merge(const MergeParams& p, int B, cudaStream_t st) {
  const size_t smem = ((sizeof(MergeCtl) + 15) & ~size_t(15)) + (size_t)kMergeCap * 8 + (size_t)p.L * 4;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  merge_kernel<<<B, kMergeNT, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace linr
