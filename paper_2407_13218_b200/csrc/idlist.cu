// ID-list clauses (§3.1): per item and slot a list of 64-bit
// attribute ids ("we store all clause attributes in a single matrix in practice and have an extra
// counting matrix to record the number of attributes for each item in each clause"; P:4564:
// "converted to 64-bit integers before GPU comparison"). A query clause (slot, reverse, id list)
// passes an item iff at least one of the item's ids is in the list, XOR reverse.
//
// Storage (caller-owned, position-major so a warp reads 32 consecutive items' a-th id in one
// coalesced load): ids [sum_s A_s][cap_pad] u64, counts [S][cap_pad] u8.
//
// idl_filter_kernel evaluates every ID-list clause of one query over the index into a liveness
// bitmap (live AND all ID clauses of the query); the fused scan then runs on that bitmap in place
// of the index's liveness bitmap, with the bitmask clauses still evaluated inside the scan. Per item
// and clause the ids are tested against the query's sorted list by binary search (shared memory),
// stopping at the first match ("we can stop checking early as long as one attribute is
// matched").
#include "common.cuh"
#include "internal.h"

namespace linr {

constexpr int kIdlNT = 256;

struct IdlFilterParams {
  const uint64_t* ids;          // [sumA][cap_pad]
  const uint8_t* counts;        // [S][cap_pad]
  int64_t cap_pad;
  const uint32_t* live;         // index liveness bitmap
  const DevHeader* hdr;
  int slot_off[4];              // first position row of slot s in ids
  const int* q_ncl;             // [B] ID clauses per query
  const int4* q_cl;             // [B][16] (slot, reverse, first id index, count)
  const uint64_t* q_ids;        // staged query ids (each clause's list sorted ascending, distinct)
  uint32_t* out;                // [B][words] bitmaps
  int64_t words;                // bitmap words per query (cap_pad / 32)
};

__global__ void __launch_bounds__(kIdlNT) idl_filter_kernel(const __grid_constant__ IdlFilterParams p) {
  __shared__ uint64_t sq[kIdlMaxQueryIds];
  __shared__ int4 scl[16];
  const int b = blockIdx.y;
  const int ncl = p.q_ncl[b];
  if (threadIdx.x < ncl) scl[threadIdx.x] = p.q_cl[b * 16 + threadIdx.x];
  __syncthreads();
  int nids = 0;
  if (ncl > 0) nids = scl[ncl - 1].z + scl[ncl - 1].w;
  const int first = ncl > 0 ? scl[0].z : 0;
  for (int i = threadIdx.x; i < nids - first; i += kIdlNT) sq[i] = p.q_ids[first + i];
  __syncthreads();
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int lane = threadIdx.x & 31;
  for (int64_t i = (int64_t)blockIdx.x * kIdlNT + threadIdx.x; i < p.cap_pad; i += (int64_t)gridDim.x * kIdlNT) {
    bool ok = i < hwm && ((p.live[i >> 5] >> (i & 31)) & 1u);
    for (int c = 0; c < ncl && ok; ++c) {
      const int4 k = scl[c];   // x slot, y reverse, z first id, w count
      const int cnt = p.counts[(size_t)k.x * p.cap_pad + i];
      const uint64_t* col = p.ids + (size_t)p.slot_off[k.x] * p.cap_pad + i;
      const uint64_t* lst = sq + (k.z - first);
      bool hit = false;
      for (int a = 0; a < cnt && !hit; ++a) {
        const uint64_t v = col[(size_t)a * p.cap_pad];
        int lo = 0, hi = k.w;   // binary search in the sorted query list
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (lst[mid] < v) lo = mid + 1;
          else hi = mid;
        }
        hit = lo < k.w && lst[lo] == v;
      }
      ok = hit != (k.y != 0);
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) p.out[(size_t)b * p.words + (i >> 5)] = bits;
  }
}

cudaError_t launch_idl_filter(const uint64_t* ids, const uint8_t* counts, int64_t cap_pad, const uint32_t* live,
                              const DevHeader* hdr, const int* slot_off, const int* q_ncl, const void* q_cl,
                              const uint64_t* q_ids, int B, uint32_t* out, int grid_x, cudaStream_t st) {
  IdlFilterParams p;
  p.ids = ids;
  p.counts = counts;
  p.cap_pad = cap_pad;
  p.live = live;
  p.hdr = hdr;
  for (int s = 0; s < 4; ++s) p.slot_off[s] = slot_off[s];
  p.q_ncl = q_ncl;
  p.q_cl = reinterpret_cast<const int4*>(q_cl);
  p.q_ids = q_ids;
  p.out = out;
  p.words = cap_pad / 32;
  idl_filter_kernel<<<dim3(grid_x, B), kIdlNT, 0, st>>>(p);
  return cudaGetLastError();
}

// rows: global ids (null: contiguous local rows [r0, r0+n)); ids [n][A] row-major, counts [n]
__global__ void idl_set_rows_kernel(const int64_t* rows, int64_t r0, int64_t grow0, int64_t cap, int64_t n,
                                    int A, const uint64_t* src_ids, const uint8_t* src_cnt, uint64_t* dst_ids,
                                    uint8_t* dst_cnt, int64_t cap_pad, DevHeader* hdr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = rows ? rows[i] - grow0 : r0 + i;
  if (r < 0 || r >= cap) {
    if (rows) atomicAdd(&hdr->skipped, 1ull);
    return;
  }
  for (int a = 0; a < A; ++a) dst_ids[(size_t)a * cap_pad + r] = src_ids[(size_t)i * A + a];
  dst_cnt[r] = src_cnt[i];
}

cudaError_t launch_idl_set_rows(const int64_t* rows, int64_t r0, int64_t grow0, int64_t cap, int64_t n, int A,
                                const uint64_t* src_ids, const uint8_t* src_cnt, uint64_t* dst_ids, uint8_t* dst_cnt,
                                int64_t cap_pad, DevHeader* hdr, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  idl_set_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rows, r0, grow0, cap, n, A, src_ids, src_cnt,
                                                                   dst_ids, dst_cnt, cap_pad, hdr);
  return cudaGetLastError();
}

}  // namespace linr
