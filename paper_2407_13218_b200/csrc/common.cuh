// Shared device helpers of the LiNR B200 library: result keys, CTA-wide radix select,
// CTA-wide bitonic sort, order-preserving compaction. (Not shared with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define LINR_DEV __device__ __forceinline__

namespace linr {

constexpr int kTileItems = 256;      // items per warp tile (8 per lane)
constexpr int kMaxUsers = 8;         // users per GEMV scan launch
constexpr int kMaxClauses = 16;      // clauses per user (LINR_MAX_CLAUSES)

// ---------------------------------------------------------------- keys
// key = (ordered_u32(score) << 32) | (0xFFFFFFFF - gid): larger key = higher score, then lower id
// (reading R5). -0.0 is canonicalised to +0.0. Key 0 never encodes a real result
// (gid <= 0xFFFFFFFE), so 0 is the "empty" sentinel.
LINR_DEV uint32_t ordered_u32(float s) {
  uint32_t u = __float_as_uint(s);
  if ((u << 1) == 0u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
LINR_DEV float key_score(uint64_t key) {
  uint32_t o = (uint32_t)(key >> 32);
  uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(u);
}
LINR_DEV int64_t key_id(uint64_t key) { return (int64_t)(0xFFFFFFFFu - (uint32_t)key); }
LINR_DEV uint64_t make_key(float s, uint32_t gid) {
  return ((uint64_t)ordered_u32(s) << 32) | (uint64_t)(0xFFFFFFFFu - gid);
}

LINR_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

LINR_DEV uint4 ldg_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
LINR_DEV uint64_t ldg_stream_u64(const uint64_t* p) {
  uint64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}

// ---------------------------------------------------------------- CTA-wide primitives
// Scratch used by the CTA-wide helpers (lives in shared memory).
struct SelScratch {
  int hist[256];
  int warp_cnt[32];
  int sel_digit, sel_above, sel_cnt, total;
  unsigned long long red_and, red_or;
};

// Radix select: returns T such that |{i < n : get(i) >= T}| == k exactly, for 1 <= k <= n and
// pairwise-distinct keys. Keys below T are provably outside the top-k. All threads of the CTA
// must call it (contains __syncthreads). Digits of 8 bits from the first byte where the keys
// differ; stops early once the selected digit's whole bucket belongs to the top-k.
template <int NT, typename Get>
__device__ uint64_t block_select_ge(Get get, int n, int k, SelScratch* sc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // common prefix: AND / OR over all keys
  unsigned long long a = ~0ull, o = 0ull;
  for (int i = tid; i < n; i += NT) {
    uint64_t v = get(i);
    a &= v;
    o |= v;
  }
  for (int off = 16; off; off >>= 1) {
    a &= __shfl_xor_sync(0xffffffffu, a, off);
    o |= __shfl_xor_sync(0xffffffffu, o, off);
  }
  if (tid == 0) { sc->red_and = ~0ull; sc->red_or = 0ull; }
  __syncthreads();
  if (lane == 0) { atomicAnd(&sc->red_and, a); atomicOr(&sc->red_or, o); }
  __syncthreads();
  const unsigned long long diff = sc->red_and ^ sc->red_or;
  if (diff == 0ull) return sc->red_or;   // n == 1 (distinct keys): the key itself
  const int hb = 63 - __clzll((long long)diff);
  int shift = (hb / 8) * 8;
  uint64_t prefix = sc->red_or & (shift == 56 ? 0ull : (~0ull << (shift + 8)));
  uint64_t pmask = (shift == 56 ? 0ull : (~0ull << (shift + 8)));
  int kk = k;
  __syncthreads();
  for (; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += NT) sc->hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      uint64_t v = get(i);
      if ((v & pmask) == prefix) atomicAdd(&sc->hist[(int)((v >> shift) & 255u)], 1);
    }
    __syncthreads();
    if (warp == 0) {
      int c[8], s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i] = sc->hist[255 - lane * 8 - i];
        s += c[i];
      }
      int incl = s;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      const int excl = incl - s;
      if (excl < kk && kk <= incl) {
        int acc = excl;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (acc + c[i] >= kk) {
            sc->sel_digit = 255 - lane * 8 - i;
            sc->sel_above = acc;
            sc->sel_cnt = c[i];
            break;
          }
          acc += c[i];
        }
      }
    }
    __syncthreads();
    const int d = sc->sel_digit, above = sc->sel_above, cnt = sc->sel_cnt;
    __syncthreads();
    prefix |= (uint64_t)d << shift;
    pmask |= 0xFFull << shift;
    kk -= above;
    if (cnt == kk) break;   // the whole bucket is inside the top-k
  }
  return prefix;
}

// In-place, order-preserving compaction of buf[0..n) to the keys >= T. Returns the new count.
template <int NT>
__device__ int block_compact_ge(uint64_t* buf, int n, uint64_t T, SelScratch* sc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  int running = 0;
  for (int base = 0; base < n; base += NT) {
    const int i = base + tid;
    uint64_t v = (i < n) ? buf[i] : 0ull;
    const bool keep = (i < n) && v >= T;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) sc->warp_cnt[warp] = __popc(bal);
    __syncthreads();   // all reads of this chunk done, warp counts visible
    int off = running;
    for (int w = 0; w < warp; ++w) off += sc->warp_cnt[w];
    int tot = running;
    for (int w = 0; w < NW; ++w) tot += sc->warp_cnt[w];
    if (keep) buf[off + __popc(bal & lanemask_lt())] = v;
    __syncthreads();
    running = tot;
  }
  return running;
}

// Bitonic sort, descending, of s[0..P2) (P2 a power of two). All threads call.
template <int NT>
__device__ void block_sort_desc(uint64_t* s, int P2) {
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P2; i += NT) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = s[i], b = s[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (a < b) : (a > b)) { s[i] = b; s[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
}

__host__ __device__ inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace linr
