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

#define LINR_DEV_HOST_INLINE __host__ __device__ __forceinline__

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

// Few vectors (the queries of a search): one warp per (vector, 32 bins), lane = bin, so the
// per-bin sums run in parallel (the per-word kernel above serialises 64 bins per thread); the
// warp's 32 bits are one ballot. Same fp64 position-order sums, same bits.
template <int DT>
__global__ void __launch_bounds__(256) oporp_encode_bins_kernel(const void* __restrict__ x, int dim, int64_t n, int k,
                                                                int L, const int32_t* __restrict__ src,
                                                                const int8_t* __restrict__ sign, uint32_t* codes32) {
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int groups = k >> 5;
  const int64_t i = gwarp / groups;
  if (i >= n) return;   // warp-uniform
  const int g = (int)(gwarp - i * groups);
  const int b = L / k;
  const int p0 = (g * 32 + lane) * b;
  const size_t xo = (size_t)i * dim;
  double s = 0.0;
  for (int p = p0; p < p0 + b; ++p) {
    const int c = __ldg(src + p);
    const double v = c < 0 ? 0.0 : code_elem<DT>(x, xo + c);
    s = __dadd_rn(s, __ldg(sign + p) > 0 ? v : -v);
  }
  const uint32_t bits = __ballot_sync(0xffffffffu, s >= 0.0);
  if (lane == 0) codes32[i * groups + g] = bits;   // LSB-first: bins 32g..32g+31 = u32 half g
}

cudaError_t launch_oporp_encode(int dtype, const void* x, int dim, int64_t n, int64_t row_begin, const int64_t* rows,
                                int64_t grow0, int64_t cap, int k, int L, const int32_t* src, const int8_t* sign,
                                uint64_t* codes, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (!rows && row_begin == 0 && n * (int64_t)k <= (1 << 22)) {
    const int64_t threads = n * k;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    uint32_t* c32 = reinterpret_cast<uint32_t*>(codes);
    switch (dtype) {
      case LINR_F32: oporp_encode_bins_kernel<LINR_F32><<<blocks, 256, 0, st>>>(x, dim, n, k, L, src, sign, c32); break;
      case LINR_F16: oporp_encode_bins_kernel<LINR_F16><<<blocks, 256, 0, st>>>(x, dim, n, k, L, src, sign, c32); break;
      case LINR_BF16: oporp_encode_bins_kernel<LINR_BF16><<<blocks, 256, 0, st>>>(x, dim, n, k, L, src, sign, c32); break;
      case LINR_I8: oporp_encode_bins_kernel<LINR_I8><<<blocks, 256, 0, st>>>(x, dim, n, k, L, src, sign, c32); break;
      default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
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

// ------------------------------------------------------------------ bulk-copy (TMA) helpers
LINR_DEV uint32_t cs_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
LINR_DEV void cs_mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cs_u32(b)), "r"(count) : "memory");
}
LINR_DEV void cs_mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cs_u32(b)), "r"(bytes) : "memory");
}
LINR_DEV void cs_mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tCS_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 2000;\n\t"
      "@P1 bra CS_DONE;\n\tbra CS_WAIT;\n\tCS_DONE:\n\t}" ::"r"(cs_u32(b)),
      "r"(parity)
      : "memory");
}
LINR_DEV void cs_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   cs_u32(dst)),
               "l"(src), "r"(bytes), "r"(cs_u32(bar))
               : "memory");
}

// ------------------------------------------------------------------ pass 1: filter + matched bits + histograms
template <int WORDS>
struct CodeGeom {
  using MT = typename std::conditional<(WORDS <= 3), uint8_t, uint16_t>::type;   // m array element
  static constexpr uint32_t kNone = WORDS <= 3 ? 0xFFu : 0xFFFFu;                  // "item not passing"
  static constexpr int IB = WORDS <= 2 ? 8 : (WORDS <= 4 ? 4 : (WORDS <= 8 ? 2 : 1));   // items per load batch
};

// lane-private u16 histograms (no atomics, no conflicts) when one user's k+1 bins x 32 lanes fit
LINR_DEV_HOST_INLINE bool code_lanepriv(int nu, int k) { return nu == 1 && k <= 64; }
constexpr int kCodeStages = 3;                        // per-warp bulk-copy ring: attribute word 0 + liveness
constexpr int kCodeStageBytes = 256 * 8 + 32;         // of one 256-item tile
size_t code_hist_smem(int nu, int V, int k) {
  const size_t h = ((size_t)kCodeNW * nu * (k + 1) * 4 + 15) & ~size_t(15);
  const size_t lp = code_lanepriv(nu, k) ? (size_t)kCodeNW * (k + 1) * 32 * 2 : 0;
  const size_t q = ((size_t)nu * V * (k / 64) * 8 + 15) & ~size_t(15);
  const size_t t = (size_t)kCodeNW * nu * 256 * (k <= 192 ? 1 : 2);
  const size_t ring = (size_t)kCodeNW * kCodeStages * kCodeStageBytes + (size_t)kCodeNW * kCodeStages * 8;
  return h + lp + q + t + ring + 32;
}

template <int WORDS, int NUM>
__global__ void __launch_bounds__(kCodeNT, 1) code_hist_kernel(const __grid_constant__ CodeScanParams p) {
  using Gm = CodeGeom<WORDS>;
  using MT = typename Gm::MT;
  extern __shared__ __align__(16) unsigned char csm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nu = NUM == 1 ? 1 : p.nu, V = p.V, K1 = WORDS * 64 + 1;   // NUM: users compiled for (1 or 8)
  uint32_t* hist = reinterpret_cast<uint32_t*>(csm);   // [NW][nu][K1]
  const bool lp = WORDS <= 2 && code_lanepriv(nu, WORDS * 64);
  uint16_t* lh = reinterpret_cast<uint16_t*>(csm + (((size_t)kCodeNW * nu * K1 * 4 + 15) & ~size_t(15)));   // [NW][K1][32]
  uint64_t* snq = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(lh) +
                                              (lp ? (size_t)kCodeNW * K1 * 32 * 2 : 0));   // [nu][V][WORDS]
  MT* stile = reinterpret_cast<MT*>(reinterpret_cast<unsigned char*>(snq) +
                                    (((size_t)nu * V * WORDS * 8 + 15) & ~size_t(15)));   // [NW][nu][256], 16B-aligned
  unsigned char* ring = reinterpret_cast<unsigned char*>(stile) + (size_t)kCodeNW * nu * 256 * sizeof(MT);   // 16B-aligned
  uint64_t* rbar = reinterpret_cast<uint64_t*>(ring + (size_t)kCodeNW * kCodeStages * kCodeStageBytes);
  for (int i = tid; i < kCodeNW * nu * K1; i += kCodeNT) hist[i] = 0u;
  if (lp)
    for (int i = tid; i < kCodeNW * K1 * 16; i += kCodeNT) reinterpret_cast<uint32_t*>(lh)[i] = 0u;
  if (tid < kCodeNW * kCodeStages) cs_mbar_init(&rbar[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int i = tid; i < nu * V * WORDS; i += kCodeNT) snq[i] = ~p.qcodes[i];   // NOT(query code), Fig. 3
  __syncthreads();
  const int gw = blockIdx.x * kCodeNW + warp, GW = gridDim.x * kCodeNW;
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t ntiles = (hwm + 255) / 256;
  const int64_t t0 = ntiles * gw / GW, t1 = ntiles * (gw + 1) / GW;
  uint32_t* myhist = hist + (size_t)warp * nu * K1;
  uint16_t* mylh = lh + (size_t)warp * K1 * 32 + lane;
  MT* mytile = stile + (size_t)warp * nu * 256;
  const bool w0 = (p.wmask & 1u) != 0;
  // per-warp ring of kCodeStages tiles: attribute word 0 (2 KB) + liveness (32 B) of a tile arrive
  // by one bulk copy each (TMA, no registers held while in flight); tile t uses stage (t - t0) % S
  unsigned char* myring = ring + (size_t)warp * kCodeStages * kCodeStageBytes;
  uint64_t* mybar = rbar + warp * kCodeStages;
  auto issue = [&](int64_t tile) {
    const int st = (int)((uint32_t)(tile - t0) % kCodeStages);
    if (lane == 0) {
      unsigned char* d = myring + st * kCodeStageBytes;
      cs_mbar_expect_tx(&mybar[st], (w0 ? 2048u : 0u) + 32u);
      if (w0) cs_bulk_load(d, p.attr + tile * 256, 2048u, &mybar[st]);
      cs_bulk_load(d + 2048, p.live + tile * 8, 32u, &mybar[st]);
    }
  };
  auto fetch = [&](int64_t tile, uint64_t (&a)[8], uint32_t& lw) {   // wait for the tile's stage, read it
    const uint32_t rel = (uint32_t)(tile - t0);
    const int st = (int)(rel % kCodeStages);
    cs_mbar_wait(&mybar[st], (rel / kCodeStages) & 1u);
    const unsigned char* d = myring + st * kCodeStageBytes;
    lw = lane < 8 ? reinterpret_cast<const uint32_t*>(d + 2048)[lane] : 0u;
    if (w0) {
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] = reinterpret_cast<const uint64_t*>(d)[t * 32 + lane];
    }
    __syncwarp();   // every lane has read the stage: it may be refilled
    if (tile + kCodeStages < t1) issue(tile + kCodeStages);
  };
  // one tile: liveness + clauses, matched bits of the passing items, histogram, m array, tile max
  // Software pipeline over the warp's tiles (k <= 128: codes of 8 B / 16 B per item): phase A of
  // tile i+1 (liveness + clauses, then the predicated code loads) is issued before phase B of tile i
  // (matched bits, histogram, m array), and the attributes of tile i+2 are in flight meanwhile; two
  // register sets and a loop unrolled by two, so no register copy waits on an in-flight load.
  constexpr bool kPipe = WORDS <= 2;
  struct Stage {
    uint32_t pb[NUM];
    uint64_t c[kPipe ? 8 : 1][kPipe ? WORDS : 1];
  };
  auto load_code = [&](const uint64_t* cp, uint64_t* dst) {
    if constexpr (WORDS == 1) {
      dst[0] = ldg_stream_u64(cp);
    } else {
#pragma unroll
      for (int q = 0; q < WORDS / 2; ++q) {
        const uint4 v = ldg_stream_v4(cp + 2 * q);
        dst[2 * q] = ((uint64_t)v.y << 32) | v.x;
        dst[2 * q + 1] = ((uint64_t)v.w << 32) | v.z;
      }
    }
  };
  auto phaseA = [&](const int64_t tile, Stage& S) {
    const int64_t base = tile * 256;
    uint64_t a[8];
    uint32_t lw;
    fetch(tile, a, lw);
    uint32_t mylive = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) mylive |= ((__shfl_sync(0xffffffffu, lw, t) >> lane) & 1u) << t;
#pragma unroll
    for (int u = 0; u < NUM; ++u) S.pb[u] = u < nu ? mylive : 0u;
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
        for (int u = 0; u < NUM; ++u) {
          if (u >= nu) continue;
          for (int c = 0; c < p.ncl[u]; ++c) {
            const KClause k = p.cl[u * 16 + c];
            if (k.word != (uint32_t)w) continue;
            const bool rev = k.rev != 0u;
#pragma unroll
            for (int t = 0; t < 8; ++t)
              if (((aw[t] & k.mask) != 0ull) == rev) S.pb[u] &= ~(1u << t);
          }
        }
      }
    }
    if constexpr (kPipe) {   // codes of the passing items (predicated: sectors of non-passing items stay unread)
      uint32_t anyp = 0;
#pragma unroll
      for (int u = 0; u < NUM; ++u) anyp |= S.pb[u];
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if ((anyp >> t) & 1u) load_code(p.codes + (size_t)(base + t * 32 + lane) * WORDS, S.c[t]);
    }
  };
  auto score = [&](const int t, const uint64_t* c, const Stage& S) {
    const int it = t * 32 + lane;
#pragma unroll
    for (int u = 0; u < NUM; ++u) {
      if (u >= nu) continue;
      uint32_t m = Gm::kNone;
      if ((S.pb[u] >> t) & 1u) {
        int best = 0;
        if (V == 1) {
          const uint64_t* q = snq + (size_t)u * WORDS;
#pragma unroll
          for (int w = 0; w < WORDS; ++w) best += __popcll(q[w] ^ c[w]);
        } else {
          for (int v = 0; v < V; ++v) {
            const uint64_t* q = snq + ((size_t)u * V + v) * WORDS;
            int s = 0;
#pragma unroll
            for (int w = 0; w < WORDS; ++w) s += __popcll(q[w] ^ c[w]);
            best = max(best, s);
          }
        }
        m = (uint32_t)best;
        if (lp) mylh[best * 32] += 1;   // this lane's own counter
        else atomicAdd(&myhist[u * K1 + best], 1u);
      }
      mytile[u * 256 + it] = (MT)m;
    }
  };
  auto phaseB = [&](const int64_t tile, const Stage& S) {
    const int64_t base = tile * 256;
    if constexpr (kPipe) {
#pragma unroll
      for (int t = 0; t < 8; ++t) score(t, S.c[t], S);
    } else {
      uint32_t anyp = 0;
#pragma unroll
      for (int u = 0; u < NUM; ++u) anyp |= S.pb[u];
#pragma unroll
      for (int t0b = 0; t0b < 8; t0b += Gm::IB) {
        uint64_t c[Gm::IB][WORDS];
#pragma unroll
        for (int j = 0; j < Gm::IB; ++j)
          if ((anyp >> (t0b + j)) & 1u) load_code(p.codes + (size_t)(base + (t0b + j) * 32 + lane) * WORDS, c[j]);
#pragma unroll
        for (int j = 0; j < Gm::IB; ++j) score(t0b + j, c[j], S);
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
  };
  // pipeline: attributes + liveness kCodeStages tiles ahead (bulk copies), code loads two tiles
  // ahead (phase A of tile i+2 before phase B of tile i), three register sets, unrolled by three
  for (int64_t t = t0; t < t1 && t < t0 + kCodeStages; ++t) issue(t);
  if constexpr (WORDS == 1) {
    Stage S0, S1, S2;
    if (t0 < t1) phaseA(t0, S0);
    if (t0 + 1 < t1) phaseA(t0 + 1, S1);
    for (int64_t tile = t0; tile < t1; tile += 3) {
      if (tile + 2 < t1) phaseA(tile + 2, S2);
      phaseB(tile, S0);
      if (tile + 1 >= t1) break;
      if (tile + 3 < t1) phaseA(tile + 3, S0);
      phaseB(tile + 1, S1);
      if (tile + 2 >= t1) break;
      if (tile + 4 < t1) phaseA(tile + 4, S1);
      phaseB(tile + 2, S2);
    }
  } else {   // wider codes: code loads one tile ahead (two register sets)
    Stage S0, S1;
    if (t0 < t1) phaseA(t0, S0);
    for (int64_t tile = t0; tile < t1; tile += 2) {
      if (tile + 1 < t1) phaseA(tile + 1, S1);
      phaseB(tile, S0);
      if (tile + 1 >= t1) break;
      if (tile + 2 < t1) phaseA(tile + 2, S0);
      phaseB(tile + 1, S1);
    }
  }
  __syncwarp();
  if (lp) {   // fold the lane-private counters into the warp's histogram
    const uint16_t* base = lh + (size_t)warp * K1 * 32;
    for (int m = lane; m < K1; m += 32) {
      uint32_t c = 0;
      const uint32_t* r = reinterpret_cast<const uint32_t*>(base + (size_t)m * 32);
#pragma unroll
      for (int l = 0; l < 16; ++l) c += (r[l] & 0xFFFFu) + (r[l] >> 16);
      myhist[m] = c;
    }
    __syncwarp();
  }
  // per-warp histograms -> H[u][K1][GW] (column m of every warp contiguous for the offset scans);
  // CTA totals -> T[u][K1]
  for (int u = 0; u < nu; ++u)
    for (int m = lane; m < K1; m += 32) p.H[((size_t)u * K1 + m) * GW + gw] = myhist[u * K1 + m];
  __syncthreads();
  for (int i = tid; i < nu * K1; i += kCodeNT) {
    unsigned long long s = 0;
    for (int w = 0; w < kCodeNW; ++w) s += hist[(size_t)w * nu * K1 + i];
    if (s) atomicAdd(&p.T[i], s);
  }
  // the last CTA to finish turns the totals into the selection: per user the suffix counts
  // S[m] = #items with m' >= m, the number of results kept = min(pass, K) (V3: min(pass,
  // max(K, ceil(keep*pass)))), m* = the largest m with S[m] >= kept
  __threadfence();
  __syncthreads();
  __shared__ unsigned int s_ticket;
  if (tid == 0) s_ticket = atomicAdd(p.ticket, 1u);
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  __threadfence();
  unsigned long long* S = reinterpret_cast<unsigned long long*>(csm);   // reuse: [K1 + 1]
  for (int u = 0; u < nu; ++u) {
    if (warp == 0) {   // suffix sums, lane l owns a contiguous chunk of the reversed bins
      const int per = (K1 + 31) / 32;
      unsigned long long loc = 0;
      for (int j = 0; j < per; ++j) {
        const int m = K1 - 1 - (lane * per + j);
        if (m >= 0) loc += atomicAdd(&p.T[(size_t)u * K1 + m], 0ull);
      }
      unsigned long long incl = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      unsigned long long run = incl - loc;
      for (int j = 0; j < per; ++j) {
        const int m = K1 - 1 - (lane * per + j);
        if (m >= 0) {
          run += atomicAdd(&p.T[(size_t)u * K1 + m], 0ull);
          S[m] = run;
        }
      }
      if (lane == 0) S[K1] = 0ull;
    }
    __syncthreads();
    const unsigned long long pass = S[0];
    unsigned long long want;
    if (p.keep > 0.0) {
      unsigned long long kk = (unsigned long long)ceil(p.keep * (double)pass);
      if (kk < (unsigned long long)p.K) kk = (unsigned long long)p.K;
      want = kk < pass ? kk : pass;
    } else {
      want = (unsigned long long)p.K < pass ? (unsigned long long)p.K : pass;
    }
    if (tid == 0) {
      p.mstar[u] = K1;   // nothing to emit unless a bin below qualifies
      p.kept[u] = (int64_t)want;
      if (p.pass) p.pass[u] = (int64_t)pass;
    }
    __syncthreads();
    for (int m = tid; m < K1; m += kCodeNT) {
      p.above[(size_t)u * (K1 + 1) + m] = S[m + 1];
      if (want > 0 && S[m] >= want && S[m + 1] < want) p.mstar[u] = m;
    }
    __syncthreads();
  }
  if (tid == 0) *p.ticket = 0u;   // reusable by the next search on this workspace
}

// ------------------------------------------------------------------ offsets: counts -> output positions
// Block (m, u), m >= m*: exclusive scan over the warps (= item-id order) of their counts of value m,
// offset by the number of items with a larger m: off[u][gw][m] = first output position of warp gw's
// items with matched bits m.
__global__ void __launch_bounds__(1024) code_offsets_kernel(const __grid_constant__ CodeOffsetParams p) {
  __shared__ unsigned int wsum[32];
  const int m = blockIdx.x, u = blockIdx.y, K1 = p.k + 1, tid = threadIdx.x;
  if (m < p.mstar[u]) return;
  const unsigned long long above = p.above[(size_t)u * (K1 + 1) + m];
  const int GW = p.GW;
  const int per = (GW + 1023) / 1024;
  const int g0 = tid * per;
  const uint32_t* col = p.H + ((size_t)u * K1 + m) * GW;
  unsigned int loc = 0;
  for (int j = 0; j < per; ++j)
    if (g0 + j < GW) loc += col[g0 + j];
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
    p.off[((size_t)u * GW + g) * K1 + m] = (uint32_t)(run < 0xFFFFFFFFull ? run : 0xFFFFFFFFull);
    run += col[g];
  }
}

// ------------------------------------------------------------------ pass 2: emit in (m desc, id asc) order
// Each warp walks its own tile range (the same as in pass 1) in id order. Tiles whose max m is below
// m* are skipped (one tmax read per tile, 32 tiles per warp load); the m values of up to 2 KB of
// qualifying tiles are loaded with 16-byte vector loads in one batch (memory-level parallelism),
// staged in shared memory and read back item-major (item t*32 + lane), so the rank among equal m
// (__match_any_sync) follows item ids.
template <int WORDS>
__global__ void __launch_bounds__(kCodeNT, 1) code_emit_kernel(const __grid_constant__ CodeEmitParams p) {
  using Gm = CodeGeom<WORDS>;
  using MT = typename Gm::MT;
  constexpr int TB = 256 * (int)sizeof(MT);   // bytes of m per tile
  constexpr int G = 2048 / TB;                // tiles per load batch
  constexpr int LPT = TB / 16;                // lanes per tile load
  constexpr int TPI = 32 / LPT;               // tiles per load instruction
  constexpr int NI = G / TPI;                 // load instructions per batch
  extern __shared__ __align__(16) unsigned char esm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nu = p.nu, K1 = WORDS * 64 + 1;
  unsigned char* mybuf = esm + (size_t)warp * 2048;
  uint32_t* mylist = reinterpret_cast<uint32_t*>(esm + (size_t)kCodeNW * 2048) + (size_t)warp * 256;   // [NW][256]
  uint32_t* cursor = reinterpret_cast<uint32_t*>(esm + (size_t)kCodeNW * 3072);   // [NW][nu][K1]
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
    const unsigned char* marr = reinterpret_cast<const unsigned char*>(p.marr) + (size_t)u * p.cap_pad * sizeof(MT);
    uint32_t* cu = mycur + u * K1;
    for (int64_t chunk = t0; chunk < t1; chunk += 32) {
      const int64_t tl = chunk + lane;
      const uint32_t tm = tl < t1 ? p.tmax[(size_t)u * p.tmax_stride + tl] : 0xFFFFu;
      uint32_t q = __ballot_sync(0xffffffffu, tm != 0xFFFFu && tm >= ms);
      while (q) {
        const int ng = min(__popc(q), G);
        uint4 v[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int g = i * TPI + lane / LPT;
          if (g < ng) {
            const int j = (int)__fns(q, 0, g + 1);
            v[i] = ldg_stream_v4(marr + (size_t)(chunk + j) * TB + (lane % LPT) * 16);
          }
        }
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int g = i * TPI + lane / LPT;
          if (g < ng) *reinterpret_cast<uint4*>(mybuf + g * TB + (lane % LPT) * 16) = v[i];
        }
        __syncwarp();
        for (int g = 0; g < ng; ++g) {
          const int j = __ffs(q) - 1;
          q &= q - 1u;
          const int64_t base = (chunk + j) * 256;
          const MT* row = reinterpret_cast<const MT*>(mybuf + g * TB);
          // candidates of the tile, compacted in item order (t-major, lane-minor = id order)
          int nc = 0;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const uint32_t m = row[t * 32 + lane];
            const bool cand = m != Gm::kNone && m >= ms;
            const uint32_t bal = __ballot_sync(0xffffffffu, cand);
            if (cand) mylist[nc + __popc(bal & lanemask_lt())] = ((uint32_t)(t * 32 + lane) << 16) | m;
            nc += __popc(bal);
          }
          __syncwarp();
          // 32 candidates at a time: rank among equal m by one match, positions from the cursors
          for (int c0 = 0; c0 < nc; c0 += 32) {
            const bool valid = c0 + lane < nc;
            const uint32_t e = valid ? mylist[c0 + lane] : 0xFFFFFFFFu;
            const uint32_t m = e & 0xFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, valid ? m : 0xFFFFFFFFu);
            if (valid) {
              const uint32_t pos = cu[m] + (uint32_t)__popc(peers & lanemask_lt());
              if ((int64_t)pos < kept) {
                const int64_t at = (int64_t)u * p.out_stride + pos;
                const uint32_t lr = (uint32_t)(base + (e >> 16));
                if (p.out_ids) {
                  p.out_ids[at] = (int64_t)(p.row0 + lr);
                  p.out_m[at] = (int32_t)m;
                }
                if (p.cand) p.cand[at] = lr;
              }
            }
            __syncwarp();
            if (valid && lane == 31 - __clz(peers)) cu[m] += (uint32_t)__popc(peers);
            __syncwarp();
          }
        }
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
  auto k = p.nu == 1 ? code_hist_kernel<WORDS, 1> : code_hist_kernel<WORDS, kCodeMaxUsers>;
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
  const size_t smem = (size_t)kCodeNW * 3072 + (size_t)kCodeNW * p.nu * (WORDS * 64 + 1) * 4;
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
