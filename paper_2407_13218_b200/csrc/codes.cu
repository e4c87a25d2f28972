// Quantised KNN on the device (§3.2 "Quantized KNN", Fig. 3 caption P:4310):
// Sign-OPORP 1-bit codes, the filtered matched-bit scan with exact selection of ANY number of
// results (the notification case: top-50M of 1B members, P:4665 -- SURVEY §8(f) NEXT-1/NEXT-3),
// and the V3 two-stage search (quantised pre-ranking keeps a fraction of the passing items, the
// kept items are re-scored at full precision).
//
// Kernels (all stream-ordered, no host synchronisation):
//   oporp_encode_kernel  one thread per (vector, 64-bit code word): bin j of the code sums
//                        sign[p] * x[src[p]] over its positions in fp64, in position order (the
//                        oracle's arithmetic, so codes are bit-exact); bit = sum >= 0.
//   code_hist_kernel     pass 1 over the index: per 256-item tile, liveness + clauses,
//                        then for the passing items m = max_v popc(~q_v ^ x) (Fig. 3: XOR with the
//                        NOT-ed query code, count matched bits); m is written to a per-user byte /
//                        u16 array, a per-warp histogram of m is kept in shared memory, and each
//                        tile's max m is recorded. Every warp owns a contiguous tile range.
//   code_offsets_kernel  per (user, m): from the histograms, the number of results to produce
//                        (K, or V3's K' = min(pass, max(K, ceil(keep*pass)))), the threshold m* and,
//                        for m >= m*, each warp's first output position of its items with that m:
//                        position = #items with larger m + #items with this m in earlier warps.
//   code_emit_kernel     pass 2 over the m arrays (tiles whose max is below m* are skipped): each
//                        candidate item goes to position off[warp][m] + its rank among the warp's
//                        earlier items with the same m -- the exact (m desc, id asc) order, i.e. a
//                        parallel counting sort; positions >= K are dropped.
//   rerank_kernel        V3 stage 3: the kept rows of each user are re-scored (fp32 FFMA over the
//                        stored dtype, max over V) into an exact per-CTA top-K (threshold +
//                        radix-select compaction), sorted; merge_kernel combines the CTAs' lists.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace linr {

constexpr int kCodeNT = 512;
constexpr int kCodeNW = kCodeNT / 32;

// ------------------------------------------------------------------ encoding
template <int DT>
LINR_DEV double code_elem(const void* base, size_t i) {
  if constexpr (DT == LINR_F32) return (double)reinterpret_cast<const float*>(base)[i];
  else if constexpr (DT == LINR_BF16) return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  else if constexpr (DT == LINR_F16) return (double)__half2float(reinterpret_cast<const __half*>(base)[i]);
  else return (double)reinterpret_cast<const int8_t*>(base)[i];
}

// rows: local row r = rows ? rows[i] - grow0 : row_begin + i (rows outside [0, cap) are skipped)
template <int DT>
__global__ void __launch_bounds__(256) oporp_encode_kernel(const void* __restrict__ x, int dim, int64_t n,
                                                           int64_t row_begin, const int64_t* __restrict__ rows,
                                                           int64_t grow0, int64_t cap, int k, int L,
                                                           const int32_t* __restrict__ src,
                                                           const int8_t* __restrict__ sign, uint64_t* codes) {
  const int words = k >> 6;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * words) return;
  const int64_t i = t / words;
  const int w = (int)(t - i * words);
  int64_t r = row_begin + i;
  if (rows) {
    r = rows[i] - grow0;
    if (r < 0 || r >= cap) return;
  }
  const int b = L / k;
  const size_t xo = (size_t)r * dim;
  uint64_t code = 0ull;
  for (int j = 0; j < 64; ++j) {
    const int p0 = (w * 64 + j) * b;
    double s = 0.0;
    for (int p = p0; p < p0 + b; ++p) {
      const int c = __ldg(src + p);
      const double v = c < 0 ? 0.0 : code_elem<DT>(x, xo + c);
      s = __dadd_rn(s, __ldg(sign + p) > 0 ? v : -v);   // fp64, position order: the oracle's sum
    }
    if (s >= 0.0) code |= 1ull << j;
  }
  codes[(size_t)r * words + w] = code;
}

cudaError_t launch_oporp_encode(int dtype, const void* x, int dim, int64_t n, int64_t row_begin, const int64_t* rows,
                                int64_t grow0, int64_t cap, int k, int L, const int32_t* src, const int8_t* sign,
                                uint64_t* codes, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t threads = n * (k / 64);
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  switch (dtype) {
    case LINR_F32: oporp_encode_kernel<LINR_F32><<<blocks, 256, 0, st>>>(x, dim, n, row_begin, rows, grow0, cap, k, L, src, sign, codes); break;
    case LINR_F16: oporp_encode_kernel<LINR_F16><<<blocks, 256, 0, st>>>(x, dim, n, row_begin, rows, grow0, cap, k, L, src, sign, codes); break;
    case LINR_BF16: oporp_encode_kernel<LINR_BF16><<<blocks, 256, 0, st>>>(x, dim, n, row_begin, rows, grow0, cap, k, L, src, sign, codes); break;
    case LINR_I8: oporp_encode_kernel<LINR_I8><<<blocks, 256, 0, st>>>(x, dim, n, row_begin, rows, grow0, cap, k, L, src, sign, codes); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ pass 1: filter + matched bits + histograms
template <int WORDS>
struct CodeGeom {
  using MT = typename std::conditional<(WORDS <= 3), uint8_t, uint16_t>::type;   // m array element
  static constexpr uint32_t kNone = WORDS <= 3 ? 0xFFu : 0xFFFFu;                  // "item not passing"
  static constexpr int IB = WORDS <= 2 ? 8 : (WORDS <= 4 ? 4 : (WORDS <= 8 ? 2 : 1));   // items per load batch
};

size_t code_hist_smem(int nu, int V, int k) {
  const size_t h = ((size_t)kCodeNW * nu * (k + 1) * 4 + 15) & ~size_t(15);
  const size_t q = ((size_t)nu * V * (k / 64) * 8 + 15) & ~size_t(15);
  const size_t t = (size_t)kCodeNW * nu * 256 * (k <= 192 ? 1 : 2);
  return h + q + t + 16;
}

template <int WORDS>
__global__ void __launch_bounds__(kCodeNT, 1) code_hist_kernel(const __grid_constant__ CodeScanParams p) {
  using Gm = CodeGeom<WORDS>;
  using MT = typename Gm::MT;
  extern __shared__ __align__(16) unsigned char csm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nu = p.nu, V = p.V, K1 = WORDS * 64 + 1;
  uint32_t* hist = reinterpret_cast<uint32_t*>(csm);   // [NW][nu][K1]
  uint64_t* snq = reinterpret_cast<uint64_t*>(csm + (((size_t)kCodeNW * nu * K1 * 4 + 15) & ~size_t(15)));   // [nu][V][WORDS]
  MT* stile = reinterpret_cast<MT*>(reinterpret_cast<unsigned char*>(snq) +
                                    (((size_t)nu * V * WORDS * 8 + 15) & ~size_t(15)));   // [NW][nu][256], 16B-aligned
  for (int i = tid; i < kCodeNW * nu * K1; i += kCodeNT) hist[i] = 0u;
  for (int i = tid; i < nu * V * WORDS; i += kCodeNT) snq[i] = ~p.qcodes[i];   // NOT(query code), Fig. 3
  __syncthreads();
  const int gw = blockIdx.x * kCodeNW + warp, GW = gridDim.x * kCodeNW;
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t ntiles = (hwm + 255) / 256;
  const int64_t t0 = ntiles * gw / GW, t1 = ntiles * (gw + 1) / GW;
  uint32_t* myhist = hist + (size_t)warp * nu * K1;
  MT* mytile = stile + (size_t)warp * nu * 256;
  const bool w0 = (p.wmask & 1u) != 0;
  uint64_t a[8], na[8];
  uint32_t lw = 0, nlw = 0;
  auto prefetch = [&](int64_t tile, uint64_t (&dst)[8], uint32_t& l) {
    const int64_t base = tile * 256;
    l = lane < 8 ? __ldg(p.live + (base >> 5) + lane) : 0u;
    if (w0) {
#pragma unroll
      for (int t = 0; t < 8; ++t) dst[t] = ldg_stream_u64(p.attr + base + t * 32 + lane);
    }
  };
  if (t0 < t1) prefetch(t0, a, lw);
  for (int64_t tile = t0; tile < t1; ++tile) {
    if (tile + 1 < t1) prefetch(tile + 1, na, nlw);
    const int64_t base = tile * 256;
    uint32_t mylive = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) mylive |= ((__shfl_sync(0xffffffffu, lw, t) >> lane) & 1u) << t;
    uint32_t pb[kCodeMaxUsers];
#pragma unroll
    for (int u = 0; u < kCodeMaxUsers; ++u) pb[u] = u < nu ? mylive : 0u;
    if (__any_sync(0xffffffffu, mylive != 0u)) {
#pragma unroll 1
      for (int w = 0; w < 4; ++w) {
        if (!((p.wmask >> w) & 1u)) continue;
        uint64_t aw[8];
        if (w == 0) {
#pragma unroll
          for (int t = 0; t < 8; ++t) aw[t] = a[t];
        } else {
#pragma unroll
          for (int t = 0; t < 8; ++t) aw[t] = ldg_stream_u64(p.attr + (size_t)w * p.cap_pad + base + t * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < kCodeMaxUsers; ++u) {
          if (u >= nu) continue;
          for (int c = 0; c < p.ncl[u]; ++c) {
            const KClause k = p.cl[u * 16 + c];
            if (k.word != (uint32_t)w) continue;
            const bool rev = k.rev != 0u;
#pragma unroll
            for (int t = 0; t < 8; ++t)
              if (((aw[t] & k.mask) != 0ull) == rev) pb[u] &= ~(1u << t);
          }
        }
      }
    }
    uint32_t anyp = 0;
#pragma unroll
    for (int u = 0; u < kCodeMaxUsers; ++u) anyp |= pb[u];
    // codes of the passing items (predicated loads: sectors of non-passing items are not fetched)
#pragma unroll
    for (int t0b = 0; t0b < 8; t0b += Gm::IB) {
      uint64_t c[Gm::IB][WORDS];
#pragma unroll
      for (int j = 0; j < Gm::IB; ++j) {
        const int t = t0b + j;
        if ((anyp >> t) & 1u) {
          const uint64_t* cp = p.codes + (size_t)(base + t * 32 + lane) * WORDS;
          if constexpr (WORDS == 1) {
            c[j][0] = ldg_stream_u64(cp);
          } else {
#pragma unroll
            for (int q = 0; q < WORDS / 2; ++q) {
              const uint4 v = ldg_stream_v4(cp + 2 * q);
              c[j][2 * q] = ((uint64_t)v.y << 32) | v.x;
              c[j][2 * q + 1] = ((uint64_t)v.w << 32) | v.z;
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < Gm::IB; ++j) {
        const int t = t0b + j;
        const int it = t * 32 + lane;
#pragma unroll
        for (int u = 0; u < kCodeMaxUsers; ++u) {
          if (u >= nu) continue;
          uint32_t m = Gm::kNone;
          if ((pb[u] >> t) & 1u) {
            int best = 0;
            for (int v = 0; v < V; ++v) {
              const uint64_t* q = snq + ((size_t)u * V + v) * WORDS;
              int s = 0;
#pragma unroll
              for (int w = 0; w < WORDS; ++w) s += __popcll(q[w] ^ c[j][w]);
              best = max(best, s);
            }
            m = (uint32_t)best;
            atomicAdd(&myhist[u * K1 + best], 1u);
          }
          mytile[u * 256 + it] = (MT)m;
        }
      }
    }
    __syncwarp();
    // coalesced write of the tile's m values + the tile max per user
#pragma unroll 1
    for (int u = 0; u < nu; ++u) {
      const MT* row = mytile + u * 256;
      constexpr int VEC = 256 * sizeof(MT) / 16;   // 16 or 32 uint4 per tile
      if (lane < VEC)
        reinterpret_cast<uint4*>(reinterpret_cast<MT*>(p.marr) + (size_t)u * p.cap_pad + base)[lane] =
            reinterpret_cast<const uint4*>(row)[lane];
      int mx = -1;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t m = row[t * 32 + lane];
        if (m != Gm::kNone) mx = max(mx, (int)m);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) p.tmax[(size_t)u * p.tmax_stride + tile] = mx < 0 ? (uint16_t)0xFFFFu : (uint16_t)mx;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 8; ++t) a[t] = na[t];
    lw = nlw;
  }
  __syncwarp();
  // per-warp histogram rows -> H[u][gw][K1]; CTA totals -> T[u][K1] (atomics)
  for (int u = 0; u < nu; ++u)
    for (int m = lane; m < K1; m += 32) p.H[((size_t)u * GW + gw) * K1 + m] = myhist[u * K1 + m];
  __syncthreads();
  for (int i = tid; i < nu * K1; i += kCodeNT) {
    unsigned long long s = 0;
    for (int w = 0; w < kCodeNW; ++w) s += hist[(size_t)w * nu * K1 + i];
    if (s) atomicAdd(&p.T[i], s);
  }
}

// ------------------------------------------------------------------ offsets: counts -> output positions
__global__ void __launch_bounds__(1024) code_offsets_kernel(const __grid_constant__ CodeOffsetParams p) {
  __shared__ unsigned long long sT[1025];
  __shared__ unsigned long long s_above;
  __shared__ int s_mstar;
  __shared__ unsigned int wsum[32];
  const int m = blockIdx.x, u = blockIdx.y, K1 = p.k + 1, tid = threadIdx.x;
  for (int i = tid; i < K1; i += 1024) sT[i] = p.T[(size_t)u * K1 + i];
  __syncthreads();
  if (tid == 0) {
    unsigned long long pass = 0;
    for (int i = 0; i < K1; ++i) pass += sT[i];
    unsigned long long want;
    if (p.keep > 0.0) {   // V3: K' = min(pass, max(K, ceil(keep * pass)))
      const double kd = ceil(p.keep * (double)pass);
      unsigned long long kk = (unsigned long long)kd;
      if (kk < (unsigned long long)p.K) kk = (unsigned long long)p.K;
      want = kk < pass ? kk : pass;
    } else {
      want = (unsigned long long)p.K < pass ? (unsigned long long)p.K : pass;
    }
    // m* = the largest m with #(items with m' >= m) >= want (K1 when want == 0: nothing to emit)
    int ms = K1;
    unsigned long long cum = 0;
    if (want > 0) {
      for (int i = K1 - 1; i >= 0; --i) {
        cum += sT[i];
        if (cum >= want) { ms = i; break; }
      }
    }
    unsigned long long above = 0;
    for (int i = m + 1; i < K1; ++i) above += sT[i];
    s_above = above;
    s_mstar = ms;
    if (m == 0) {
      p.mstar[u] = ms;
      p.kept[u] = (int64_t)want;
      if (p.pass) p.pass[u] = (int64_t)pass;
    }
  }
  __syncthreads();
  if (m < s_mstar) return;
  const unsigned long long above = s_above;
  // exclusive scan over the warps' counts of value m (ordered by warp = by item id)
  const int GW = p.GW;
  const int per = (GW + 1023) / 1024;
  const int g0 = tid * per;
  unsigned int loc = 0;
  for (int j = 0; j < per; ++j)
    if (g0 + j < GW) loc += p.H[((size_t)u * GW + g0 + j) * K1 + m];
  const int lane = tid & 31, wp = tid >> 5;
  unsigned int incl = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[wp] = incl;
  __syncthreads();
  if (wp == 0) {
    const unsigned int v = wsum[lane];
    unsigned int inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    wsum[lane] = inc - v;
  }
  __syncthreads();
  unsigned long long run = above + wsum[wp] + (incl - loc);
  for (int j = 0; j < per; ++j) {
    const int g = g0 + j;
    if (g >= GW) break;
    const unsigned int h = p.H[((size_t)u * GW + g) * K1 + m];
    p.off[((size_t)u * GW + g) * K1 + m] = (uint32_t)(run < 0xFFFFFFFFull ? run : 0xFFFFFFFFull);
    run += h;
  }
}

// ------------------------------------------------------------------ pass 2: emit in (m desc, id asc) order
template <int WORDS>
__global__ void __launch_bounds__(kCodeNT, 1) code_emit_kernel(const __grid_constant__ CodeEmitParams p) {
  using Gm = CodeGeom<WORDS>;
  using MT = typename Gm::MT;
  extern __shared__ __align__(16) unsigned char esm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nu = p.nu, K1 = WORDS * 64 + 1;
  uint32_t* cursor = reinterpret_cast<uint32_t*>(esm);   // [NW][nu][K1]
  const int gw = blockIdx.x * kCodeNW + warp, GW = gridDim.x * kCodeNW;
  uint32_t* mycur = cursor + (size_t)warp * nu * K1;
  for (int u = 0; u < nu; ++u) {
    const int ms = p.mstar[u];
    for (int m = ms + lane; m < K1; m += 32) mycur[u * K1 + m] = p.off[((size_t)u * GW + gw) * K1 + m];
  }
  __syncwarp();
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t ntiles = (hwm + 255) / 256;
  const int64_t t0 = ntiles * gw / GW, t1 = ntiles * (gw + 1) / GW;
  for (int u = 0; u < nu; ++u) {
    const uint32_t ms = (uint32_t)p.mstar[u];
    const int64_t kept = p.kept[u];
    if ((int)ms >= K1 || kept == 0) continue;
    const MT* marr = reinterpret_cast<const MT*>(p.marr) + (size_t)u * p.cap_pad;
    uint32_t* cu = mycur + u * K1;
    for (int64_t tile = t0; tile < t1; ++tile) {
      const uint32_t tm = p.tmax[(size_t)u * p.tmax_stride + tile];
      if (tm == 0xFFFFu || tm < ms) continue;   // no candidate in this tile
      const int64_t base = tile * 256;
      uint32_t mv[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mv[t] = marr[base + t * 32 + lane];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t m = mv[t];
        const bool cand = m != Gm::kNone && m >= ms;
        if (__ballot_sync(0xffffffffu, cand) == 0u) continue;
        const uint32_t peers = __match_any_sync(0xffffffffu, cand ? m : 0xFFFFFFFFu);
        uint32_t pos = 0;
        if (cand) {
          pos = cu[m] + (uint32_t)__popc(peers & lanemask_lt());
          if ((int64_t)pos < kept) {
            const int64_t at = (int64_t)u * p.out_stride + pos;
            const uint32_t lr = (uint32_t)(base + t * 32 + lane);
            if (p.out_ids) {
              p.out_ids[at] = (int64_t)(p.row0 + lr);
              p.out_m[at] = (int32_t)m;
            }
            if (p.cand) p.cand[at] = lr;
          }
        }
        __syncwarp();
        if (cand && lane == 31 - __clz(peers)) cu[m] += (uint32_t)__popc(peers);
        __syncwarp();
      }
    }
  }
}

// padding of the code search's outputs: positions [kept, K) get id -1, m -1
__global__ void code_pad_kernel(const int64_t* kept, int nu, int64_t K, int64_t* out_ids, int32_t* out_m) {
  for (int u = 0; u < nu; ++u) {
    const int64_t k0 = kept[u];
    for (int64_t j = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
      out_ids[(int64_t)u * K + j] = -1;
      out_m[(int64_t)u * K + j] = -1;
    }
  }
}

// ------------------------------------------------------------------ V3 stage 3: full-precision rerank
constexpr int kRrBuf = 8192;

struct RrCtl {
  SelScratch sel;
  BucketScratch bs;
  int count;
  unsigned long long thr;
};
struct RrGet {
  const uint64_t* b;
  __device__ uint64_t operator()(int x) const { return b[x]; }
};

template <int DT>
LINR_DEV float rr_elem(const void* base, size_t i) {
  if constexpr (DT == LINR_F32) return reinterpret_cast<const float*>(base)[i];
  else if constexpr (DT == LINR_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  else if constexpr (DT == LINR_F16) return __half2float(reinterpret_cast<const __half*>(base)[i]);
  else return (float)reinterpret_cast<const int8_t*>(base)[i];
}

// Per user, each CTA re-scores a contiguous slice of the user's kept rows and writes its sorted
// top-K list (0-padded) to lists[u][cta][K] -- the layout merge_kernel takes (each list's first
// min(K, 32) keys are its sample). One warp per row group: lanes split the dimension.
template <int DT>
__global__ void __launch_bounds__(kCodeNT, 1) rerank_kernel(const __grid_constant__ RerankParams p) {
  extern __shared__ __align__(16) unsigned char rsm[];
  RrCtl* ctl = reinterpret_cast<RrCtl*>(rsm);
  float* sq = reinterpret_cast<float*>(rsm + ((sizeof(RrCtl) + 15) & ~size_t(15)));
  uint64_t* buf = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sq) +
                                              (((size_t)p.V * p.dim * 4 + 15) & ~size_t(15)));
  const int tid = threadIdx.x, lane = tid & 31;
  const int K = p.K, dim = p.dim, V = p.V;
  for (int u = 0; u < p.nu; ++u) {
    const int64_t n = p.kept[u];
    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    for (int i = tid; i < V * dim; i += kCodeNT) sq[i] = rr_elem<DT>(p.q, (size_t)u * V * dim + i);
    if (tid == 0) { ctl->count = 0; ctl->thr = 0ull; }
    __syncthreads();
    const uint32_t* cand = p.cand + (size_t)u * p.cand_stride;
    for (int64_t b0 = lo; b0 < hi; b0 += kCodeNT) {   // uniform trip count within the CTA
      const int64_t i = b0 + tid;
      const bool ok = i < hi;
      const uint32_t myrow = ok ? cand[i] : 0u;
      uint64_t mykey = 0ull;
      uint32_t bal = __ballot_sync(0xffffffffu, ok);
      while (bal) {
        const int r = __ffs(bal) - 1;
        bal &= bal - 1u;
        const uint32_t row = __shfl_sync(0xffffffffu, myrow, r);
        float best = -INFINITY;
        for (int v = 0; v < V; ++v) {
          float acc = 0.0f;
          for (int j = lane; j < dim; j += 32) acc = fmaf(rr_elem<DT>(p.emb, (size_t)row * dim + j), sq[v * dim + j], acc);
#pragma unroll
          for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          best = fmaxf(best, acc);
        }
        if (lane == r) mykey = make_key(best, p.row0 + row);
      }
      const bool c = ok && mykey >= *(volatile unsigned long long*)&ctl->thr;
      const uint32_t cb = __ballot_sync(0xffffffffu, c);
      if (cb) {
        const int leader = __ffs(cb) - 1;
        int pos0 = 0;
        if (lane == leader) pos0 = atomicAdd(&ctl->count, __popc(cb));
        pos0 = __shfl_sync(0xffffffffu, pos0, leader);
        if (c) buf[pos0 + __popc(cb & lanemask_lt())] = mykey;
      }
      __syncthreads();
      const int cnt = ctl->count;
      if (cnt > kRrBuf) {
        const uint64_t T = block_select_ge<kCodeNT>(RrGet{buf}, cnt, K, &ctl->sel);
        block_compact_ge<kCodeNT>(buf, cnt, T, &ctl->sel);
        if (tid == 0) { ctl->count = K; ctl->thr = T; }
        __syncthreads();
      }
    }
    int cnt = ctl->count;
    if (cnt > K) {
      const uint64_t T = block_select_ge<kCodeNT>(RrGet{buf}, cnt, K, &ctl->sel);
      cnt = block_compact_ge<kCodeNT>(buf, cnt, T, &ctl->sel);
    }
    uint64_t* sorted = buf + 2048;
    if (!block_bucket_sort_desc<kCodeNT>(buf, cnt, sorted, &ctl->bs)) {
      const int P2 = next_pow2(cnt > 64 ? cnt : 64);
      for (int j = cnt + tid; j < P2; j += kCodeNT) buf[j] = 0ull;
      __syncthreads();
      block_sort_desc<kCodeNT>(buf, P2);
      sorted = buf;
    }
    uint64_t* out = p.lists + ((size_t)blockIdx.x * p.nu + u) * K;   // [cta][u][K]: merge_kernel's layout
    for (int j = tid; j < K; j += kCodeNT) out[j] = j < cnt ? sorted[j] : 0ull;
    __syncthreads();
  }
}

size_t rerank_smem(int V, int dim) {
  return ((sizeof(RrCtl) + 15) & ~size_t(15)) + (((size_t)V * dim * 4 + 15) & ~size_t(15)) +
         (size_t)(kRrBuf + kCodeNT) * 8;
}

// ------------------------------------------------------------------ launchers
template <int WORDS>
static cudaError_t launch_hist_w(const CodeScanParams& p, int grid, cudaStream_t st) {
  const size_t smem = code_hist_smem(p.nu, p.V, WORDS * 64);
  auto k = code_hist_kernel<WORDS>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kCodeNT, smem, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_code_hist(int k, const CodeScanParams& p, int grid, cudaStream_t st) {
  switch (k / 64) {
    case 1: return launch_hist_w<1>(p, grid, st);
    case 2: return launch_hist_w<2>(p, grid, st);
    case 4: return launch_hist_w<4>(p, grid, st);
    case 8: return launch_hist_w<8>(p, grid, st);
    case 16: return launch_hist_w<16>(p, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_code_offsets(const CodeOffsetParams& p, int nu, cudaStream_t st) {
  code_offsets_kernel<<<dim3(p.k + 1, nu), 1024, 0, st>>>(p);
  return cudaGetLastError();
}

template <int WORDS>
static cudaError_t launch_emit_w(const CodeEmitParams& p, int grid, cudaStream_t st) {
  const size_t smem = (size_t)kCodeNW * p.nu * (WORDS * 64 + 1) * 4;
  auto k = code_emit_kernel<WORDS>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kCodeNT, smem, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_code_emit(int k, const CodeEmitParams& p, int grid, cudaStream_t st) {
  switch (k / 64) {
    case 1: return launch_emit_w<1>(p, grid, st);
    case 2: return launch_emit_w<2>(p, grid, st);
    case 4: return launch_emit_w<4>(p, grid, st);
    case 8: return launch_emit_w<8>(p, grid, st);
    case 16: return launch_emit_w<16>(p, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_code_pad(const int64_t* kept, int nu, int64_t K, int64_t* out_ids, int32_t* out_m, int grid,
                            cudaStream_t st) {
  code_pad_kernel<<<grid, 256, 0, st>>>(kept, nu, K, out_ids, out_m);
  return cudaGetLastError();
}

template <int DT>
static cudaError_t launch_rr(const RerankParams& p, int grid, cudaStream_t st) {
  const size_t smem = rerank_smem(p.V, p.dim);
  auto k = rerank_kernel<DT>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kCodeNT, smem, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_rerank(int dtype, const RerankParams& p, int grid, cudaStream_t st) {
  switch (dtype) {
    case LINR_F32: return launch_rr<LINR_F32>(p, grid, st);
    case LINR_F16: return launch_rr<LINR_F16>(p, grid, st);
    case LINR_BF16: return launch_rr<LINR_BF16>(p, grid, st);
    case LINR_I8: return launch_rr<LINR_I8>(p, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace linr
