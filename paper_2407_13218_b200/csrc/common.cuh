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
LINR_DEV uint32_t ldg_stream_u32(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
LINR_DEV uint64_t ldg_stream_u64(const uint64_t* p) {
  uint64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}

// ---------------------------------------------------------------- diagnostics
// Optional phase timers (linr_debug_timers): slot = base + idx, written by thread 0 of a CTA.
LINR_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
LINR_DEV void dbg_mark(unsigned long long* d, int slot) {
  if (d != nullptr && threadIdx.x == 0) d[slot] = gtimer();
}

// ---------------------------------------------------------------- CTA-wide primitives
// Barrier of the NT threads taking part in a CTA-wide primitive: BAR = 0 is the whole CTA
// (__syncthreads), BAR > 0 a named barrier over NT threads (a role subset of a warp-specialised CTA).
template <int BAR, int NT>
LINR_DEV void part_sync() {
  if constexpr (BAR == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
  }
}

// Scratch used by the CTA-wide helpers (lives in shared memory).
struct SelScratch {
  int hist[256];
  int warp_cnt[32];
  int sel_digit, sel_above, sel_cnt, total;
  unsigned long long red_and, red_or;
};

// Radix select: returns T such that |{i < n : get(i) >= T}| == k exactly, for 1 <= k <= n and
// pairwise-distinct keys. Keys below T are provably outside the top-k. All threads of the CTA
// must call it (contains __syncthreads). 8-bit digits starting at the highest bit where the keys
// differ (so the first digit already spreads the keys); stops early once the selected digit's
// whole bucket belongs to the top-k. Plain shared-memory atomics for the histogram: measured on
// B200 2.4x faster than warp-aggregating them with __match_any_sync.
template <int NT, int BAR = 0, typename Get>
__device__ uint64_t block_select_ge(Get get, int n, int k, SelScratch* sc, int tid = threadIdx.x) {
  const int lane = tid & 31, warp = tid >> 5;
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
  part_sync<BAR, NT>();
  if (lane == 0) { atomicAnd(&sc->red_and, a); atomicOr(&sc->red_or, o); }
  part_sync<BAR, NT>();
  const unsigned long long diff = sc->red_and ^ sc->red_or;
  const unsigned long long orv = sc->red_or;
  part_sync<BAR, NT>();
  if (diff == 0ull) return orv;   // n == 1 (distinct keys): the key itself
  const int hb = 63 - __clzll((long long)diff);
  uint64_t pmask = (hb == 63) ? 0ull : (~0ull << (hb + 1));
  uint64_t prefix = orv & pmask;  // bits above hb are common to every key
  int shift = hb - 7 > 0 ? hb - 7 : 0;
  int kk = k;
  while (true) {
    for (int i = tid; i < 256; i += NT) sc->hist[i] = 0;
    part_sync<BAR, NT>();
    for (int i = tid; i < n; i += NT) {
      const uint64_t v = get(i);
      if ((v & pmask) == prefix) atomicAdd(&sc->hist[(int)((v >> shift) & 255u)], 1);
    }
    part_sync<BAR, NT>();
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
    part_sync<BAR, NT>();
    const int d = sc->sel_digit, above = sc->sel_above, cnt = sc->sel_cnt;
    part_sync<BAR, NT>();
    prefix = (prefix & ~(0xFFull << shift)) | ((uint64_t)d << shift);
    pmask |= 0xFFull << shift;
    kk -= above;
    if (cnt == kk || shift == 0) break;   // whole bucket inside the top-k, or the key is resolved
    shift = shift - 8 > 0 ? shift - 8 : 0;
  }
  return prefix;
}

// In-place, order-preserving compaction of buf[0..n) to the keys >= T. Returns the new count.
// Two barriers per NT-key chunk; warp 0 scans the per-warp counts.
template <int NT, int BAR = 0>
__device__ int block_compact_ge(uint64_t* buf, int n, uint64_t T, SelScratch* sc, int tid = threadIdx.x) {
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  int running = 0;
  for (int base = 0; base < n; base += NT) {
    const int i = base + tid;
    const uint64_t v = (i < n) ? buf[i] : 0ull;
    const bool keep = (i < n) && v >= T;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) sc->warp_cnt[warp] = __popc(bal);
    part_sync<BAR, NT>();   // all reads of this chunk done, warp counts visible
    if (warp == 0) {
      const int c = lane < NW ? sc->warp_cnt[lane] : 0;
      int incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      if (lane < NW) sc->hist[lane] = incl - c;   // exclusive warp offsets
      if (lane == 31) sc->total = incl;
    }
    part_sync<BAR, NT>();
    if (keep) buf[running + sc->hist[warp] + __popc(bal & lanemask_lt())] = v;
    running += sc->total;
  }
  part_sync<BAR, NT>();
  return running;
}

// Bitonic compare-exchange of element i against its partner value pv for stage (k, j):
// descending overall; the lower index of a pair keeps the max inside descending blocks.
LINR_DEV uint64_t bitonic_pick(uint64_t v, uint64_t pv, int i, int k, int j) {
  const bool desc = (i & k) == 0;
  const bool lower = (i & j) == 0;
  const bool take_max = (lower == desc);
  return take_max ? (v > pv ? v : pv) : (v < pv ? v : pv);
}

LINR_DEV uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

LINR_DEV uint64_t shfl_idx_u64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
LINR_DEV uint64_t shfl_up_u64(uint64_t v, int d) {
  const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, d);
  const uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), d);
  return ((uint64_t)hi << 32) | lo;
}

// MSD bucket sort, descending: keys s[0..n) (n <= 2048) -> out[0..n). Buckets = 11 bits below the
// highest bit where the keys differ (2048 buckets, scatter by atomic cursors); buckets of <= 8
// keys are insertion-sorted by one thread, buckets of <= 64 keys by one warp in registers
// (bitonic over shuffles). Returns false (out undefined) if a bucket holds more than 64 keys;
// the caller then sorts with the general bitonic network.
struct BucketScratch {
  int hist[2048];
  int wtot[32];
  int maxb;
  int nbig;
  int big[1024];
  unsigned long long red_and, red_or;
};
template <int NT>
__device__ bool block_bucket_sort_desc(const uint64_t* s, int n, uint64_t* out, BucketScratch* sc) {
  constexpr int NW = NT / 32;
  constexpr int BPW = 2048 / NW;
  constexpr int BPL = BPW / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long a = ~0ull, o = 0ull;
  for (int i = tid; i < n; i += NT) {
    const uint64_t v = s[i];
    a &= v;
    o |= v;
  }
  for (int off = 16; off; off >>= 1) {
    a &= __shfl_xor_sync(0xffffffffu, a, off);
    o |= __shfl_xor_sync(0xffffffffu, o, off);
  }
  if (tid == 0) { sc->red_and = ~0ull; sc->red_or = 0ull; sc->maxb = 0; sc->nbig = 0; }
  for (int i = tid; i < 2048; i += NT) sc->hist[i] = 0;
  __syncthreads();
  if (lane == 0) { atomicAnd(&sc->red_and, a); atomicOr(&sc->red_or, o); }
  __syncthreads();
  const unsigned long long diff = sc->red_and ^ sc->red_or;
  const int hb = diff ? 63 - __clzll((long long)diff) : 0;
  const int shift = hb - 10 > 0 ? hb - 10 : 0;
  for (int i = tid; i < n; i += NT) atomicAdd(&sc->hist[(int)((s[i] >> shift) & 2047u)], 1);
  __syncthreads();
  // exclusive offsets in descending digit order, stored back into hist as scatter cursors
  int c[BPL], sum = 0;
#pragma unroll
  for (int i = 0; i < BPL; ++i) {
    c[i] = sc->hist[2047 - warp * BPW - lane * BPL - i];
    sum += c[i];
  }
  int incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) sc->wtot[warp] = incl;
  __syncthreads();
  int acc = incl - sum, mx = 0;
  for (int w = 0; w < warp; ++w) acc += sc->wtot[w];
#pragma unroll
  for (int i = 0; i < BPL; ++i) {
    sc->hist[2047 - warp * BPW - lane * BPL - i] = acc;
    acc += c[i];
    mx = c[i] > mx ? c[i] : mx;
  }
  for (int off = 16; off; off >>= 1) {
    const int t = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = t > mx ? t : mx;
  }
  if (lane == 0) atomicMax(&sc->maxb, mx);
  __syncthreads();
  if (sc->maxb > 64) return false;
  for (int i = tid; i < n; i += NT) {
    const uint64_t v = s[i];
    out[atomicAdd(&sc->hist[(int)((v >> shift) & 2047u)], 1)] = v;
  }
  __syncthreads();
  // bucket d spans [end(d+1), end(d)) where end = the advanced cursor
  for (int d = tid; d < 2048; d += NT) {
    const int end = sc->hist[d];
    const int start = (d == 2047) ? 0 : sc->hist[d + 1];
    if (end - start > 8) {
      sc->big[atomicAdd(&sc->nbig, 1)] = d;
      continue;
    }
    for (int i = start + 1; i < end; ++i) {
      const uint64_t x = out[i];
      int j = i - 1;
      while (j >= start && out[j] < x) {
        out[j + 1] = out[j];
        --j;
      }
      out[j + 1] = x;
    }
  }
  __syncthreads();
  for (int bi = warp; bi < sc->nbig; bi += NW) {   // warp per medium bucket (<= 64 keys)
    const int d = sc->big[bi];
    const int end = sc->hist[d];
    const int start = (d == 2047) ? 0 : sc->hist[d + 1];
    const int m = end - start;
    uint64_t x0 = lane < m ? out[start + lane] : 0ull;
    uint64_t x1 = lane + 32 < m ? out[start + lane + 32] : 0ull;
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j == 32) {
          const uint64_t mxv = x0 > x1 ? x0 : x1, mnv = x0 > x1 ? x1 : x0;
          x0 = mxv;
          x1 = mnv;
        } else {
          const uint64_t p0 = shfl_xor_u64(x0, j), p1 = shfl_xor_u64(x1, j);
          x0 = bitonic_pick(x0, p0, lane, k, j);
          x1 = bitonic_pick(x1, p1, lane + 32, k, j);
        }
      }
    }
    if (lane < m) out[start + lane] = x0;
    if (lane + 32 < m) out[start + lane + 32] = x1;
  }
  __syncthreads();
  return true;
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

// One warp sorts s[0..64) descending in registers (2 elements per lane: i = lane, lane + 32).
LINR_DEV void warp_sort64_desc(uint64_t* s) {
  const int lane = threadIdx.x & 31;
  uint64_t a = s[lane], b = s[lane + 32];
  // rolled loops: this runs once per CTA at the end of a scan, where the cold instruction fetch
  // of an unrolled network costs more than the loop overhead
#pragma unroll 1
  for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {
        const uint64_t mx = a > b ? a : b, mn = a > b ? b : a;
        a = mx;   // i = lane < 32 is the lower index and k = 64 is a descending block
        b = mn;
      } else {
        const uint64_t pa = shfl_xor_u64(a, j), pb = shfl_xor_u64(b, j);
        a = bitonic_pick(a, pa, lane, k, j);
        b = bitonic_pick(b, pb, lane + 32, k, j);
      }
    }
  }
  __syncwarp();
  s[lane] = a;
  s[lane + 32] = b;
  __syncwarp();
}

// CTA-wide bitonic sort (descending) of s[0..P2), 64 <= P2 <= 4*NT, P2 a power of two. Elements
// live in registers (element i at thread i % NT, slot i / NT); partners inside a warp are
// exchanged by shuffles, across warps through the double-buffered scratch (2*P2 keys), across
// slots in registers. Far fewer barriers than a shared-memory-only network.
template <int NT>
__device__ void block_sort_desc_reg(uint64_t* s, int P2, uint64_t* scratch) {
  constexpr int EMAX = 4;
  const int t = threadIdx.x;
  const int E = P2 > NT ? P2 / NT : 1;
  uint64_t v[EMAX];
#pragma unroll
  for (int e = 0; e < EMAX; ++e) v[e] = (e < E && t + e * NT < P2) ? s[t + e * NT] : 0ull;
  int buf = 0;
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= NT) {   // partner in another slot of the same thread
        const int ej = j / NT;
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
          if (e >= E || (e & ej)) continue;   // handle each pair once, from its lower slot
          const int i = t + e * NT;
          const uint64_t a = v[e], b = v[e + ej];
          const bool desc = (i & k) == 0;
          const uint64_t mx = a > b ? a : b, mn = a > b ? b : a;
          v[e] = desc ? mx : mn;
          v[e + ej] = desc ? mn : mx;
        }
      } else if (j >= 32) {
        uint64_t* x = scratch + buf * P2;
#pragma unroll
        for (int e = 0; e < EMAX; ++e)
          if (e < E && t + e * NT < P2) x[t + e * NT] = v[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
          const int i = t + e * NT;
          if (e < E && i < P2) v[e] = bitonic_pick(v[e], x[i ^ j], i, k, j);
        }
        buf ^= 1;
      } else {
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
          if (e < E) {   // E is uniform: every lane of the warp shuffles
            const uint64_t pv = shfl_xor_u64(v[e], j);
            v[e] = bitonic_pick(v[e], pv, t + e * NT, k, j);
          }
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < EMAX; ++e)
    if (e < E && t + e * NT < P2) s[t + e * NT] = v[e];
  __syncthreads();
}

__host__ __device__ inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace linr
