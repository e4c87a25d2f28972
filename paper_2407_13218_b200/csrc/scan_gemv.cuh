// Fused pre-filter + dot-product score + CTA top-K scan (the "GEMV" path, B*V <= 8 query vectors
// per launch). PAPER.md §3.1: clause evaluation is fused into the scoring
// pass so filtered-out rows are never loaded (the V2 "explicit pre-filtering" idea, P:4284,
// without materialising a slice) and never reach top-K (reading R1: exclusion, not zero-masking).
// The fully fused filter+score+top-K kernel is the option §6 describes for regular KNN.
//
// Per warp tile of 256 items (8 per lane):
//   1. liveness bits (1 bit/item) + attribute words (8 B/item, coalesced 256 B per warp load);
//      evaluate every user's clauses -> per-(user,item) pass bits; compact passing items into a
//      per-warp list in shared memory (ballot + popc).
//   2. stream only the passing rows: LPR lanes per row, one 16-byte ld.global.nc per lane per
//      chunk, R rows in flight per lane group; fp32 FFMA (f32/f16/bf16) or exact int32 DP4A (int8)
//      against the query chunk held in registers; butterfly-reduce over the LPR lanes; max over the
//      user's V vectors (reading R12).
//   3. threshold test against the CTA's current per-user bound, warp-aggregated append of packed
//      (score,id) keys to the CTA's shared-memory buffer; when a buffer passes its soft capacity the
//      whole CTA radix-selects the K-th key and compacts (exact: keys below the K-th of K kept keys
//      can never enter the top-K).
//   4. at the end each CTA sorts its <= K survivors and writes them; the merge kernel combines the
//      per-CTA lists.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace linr {

template <int DT, int D>
struct RowGeom {
  static constexpr int ESZ = (DT == LINR_F32) ? 4 : (DT == LINR_I8 ? 1 : 2);
  static constexpr int ROWB = D * ESZ;          // bytes per row
  static constexpr int CH = ROWB / 16;          // 16-byte chunks per row
  static constexpr int LPR = CH < 32 ? CH : 32; // lanes per row
  static constexpr int CPL = CH / LPR;          // chunks per lane
  static constexpr int RPW = 32 / LPR;          // rows per warp step
  static constexpr int R = CPL >= 4 ? 1 : 4 / CPL;  // rows in flight per lane group
  static constexpr int RPI = RPW * R;           // rows per warp iteration
  static constexpr int EPC = 16 / ESZ;          // elements per chunk
  static_assert(ROWB % 16 == 0, "row must be a multiple of 16 bytes");
};

template <int DT>
struct ChunkDot;

template <>
struct ChunkDot<LINR_F32> {
  LINR_DEV static void load_q(const uint4 raw, float* q) {
    q[0] = __uint_as_float(raw.x); q[1] = __uint_as_float(raw.y);
    q[2] = __uint_as_float(raw.z); q[3] = __uint_as_float(raw.w);
  }
  LINR_DEV static float dot(const uint4 v, const float* q, float acc) {
    acc = fmaf(__uint_as_float(v.x), q[0], acc);
    acc = fmaf(__uint_as_float(v.y), q[1], acc);
    acc = fmaf(__uint_as_float(v.z), q[2], acc);
    acc = fmaf(__uint_as_float(v.w), q[3], acc);
    return acc;
  }
};

template <>
struct ChunkDot<LINR_BF16> {
  LINR_DEV static void unpack(const uint32_t w, float& lo, float& hi) {
    lo = __uint_as_float(w << 16);
    hi = __uint_as_float(w & 0xFFFF0000u);
  }
  LINR_DEV static void load_q(const uint4 raw, float* q) {
    unpack(raw.x, q[0], q[1]); unpack(raw.y, q[2], q[3]);
    unpack(raw.z, q[4], q[5]); unpack(raw.w, q[6], q[7]);
  }
  LINR_DEV static float dot(const uint4 v, const float* q, float acc) {
    float a, b;
    unpack(v.x, a, b); acc = fmaf(a, q[0], acc); acc = fmaf(b, q[1], acc);
    unpack(v.y, a, b); acc = fmaf(a, q[2], acc); acc = fmaf(b, q[3], acc);
    unpack(v.z, a, b); acc = fmaf(a, q[4], acc); acc = fmaf(b, q[5], acc);
    unpack(v.w, a, b); acc = fmaf(a, q[6], acc); acc = fmaf(b, q[7], acc);
    return acc;
  }
};

template <>
struct ChunkDot<LINR_F16> {
  LINR_DEV static void unpack(const uint32_t w, float& lo, float& hi) {
    __half2 h = *reinterpret_cast<const __half2*>(&w);
    float2 f = __half22float2(h);
    lo = f.x;
    hi = f.y;
  }
  LINR_DEV static void load_q(const uint4 raw, float* q) {
    unpack(raw.x, q[0], q[1]); unpack(raw.y, q[2], q[3]);
    unpack(raw.z, q[4], q[5]); unpack(raw.w, q[6], q[7]);
  }
  LINR_DEV static float dot(const uint4 v, const float* q, float acc) {
    float a, b;
    unpack(v.x, a, b); acc = fmaf(a, q[0], acc); acc = fmaf(b, q[1], acc);
    unpack(v.y, a, b); acc = fmaf(a, q[2], acc); acc = fmaf(b, q[3], acc);
    unpack(v.z, a, b); acc = fmaf(a, q[4], acc); acc = fmaf(b, q[5], acc);
    unpack(v.w, a, b); acc = fmaf(a, q[6], acc); acc = fmaf(b, q[7], acc);
    return acc;
  }
};

struct ScanCtl {
  SelScratch sel;
  unsigned long long thr[kMaxUsers];   // key >= thr may still enter the CTA's top-K
  int count[kMaxUsers];                // keys in each user's buffer
  unsigned int pass[kMaxUsers];        // passing items seen by this CTA
  int flag;                            // a buffer reached its soft capacity
  int done;                            // warps finished with their tiles
  int overflow;                        // appends beyond the hard capacity (must stay 0)
};

static_assert(sizeof(ScanCtl) + 16 <= 2048, "host plan reserves 2 KB for ScanCtl (api.cu kScanCtlBytes)");

LINR_DEV bool scan_flag(const ScanCtl* ctl, int lane) {
  int f = 0;
  if (lane == 0) f = *(volatile const int*)&ctl->flag;
  return __shfl_sync(0xffffffffu, f, 0) != 0;
}

template <int NT>
__device__ __noinline__ void scan_compact_all(ScanCtl* ctl, uint64_t* bufs, const ScanParams& p) {
  __syncthreads();   // every warp of the CTA is here (flag checks are warp-uniform)
  for (int u = 0; u < p.nu; ++u) {
    const int n = min(ctl->count[u], p.bufcap);
    if (n > p.K) {
      uint64_t* b = bufs + (size_t)u * p.bufcap;
      const uint64_t T = block_select_ge<NT>([b](int i) { return b[i]; }, n, p.K, &ctl->sel);
      block_compact_ge<NT>(b, n, T, &ctl->sel);
      if (threadIdx.x == 0) {
        ctl->count[u] = p.K;
        if (T > ctl->thr[u]) ctl->thr[u] = T;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) ctl->flag = 0;
  __syncthreads();
}

template <int DT, int D, int NQV, int NT>
__global__ void __launch_bounds__(NT, 1) scan_gemv_kernel(const __grid_constant__ ScanParams p) {
  using G = RowGeom<DT, D>;
  constexpr bool kInt = (DT == LINR_I8);
  using acc_t = typename std::conditional<kInt, int, float>::type;
  constexpr int NW = NT / 32;
  constexpr int NU = NQV;   // at most one user per vector

  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScanCtl* ctl = reinterpret_cast<ScanCtl*>(smem_raw);
  uint64_t* bufs = reinterpret_cast<uint64_t*>(smem_raw + ((sizeof(ScanCtl) + 15) & ~size_t(15)));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint16_t* wlist = reinterpret_cast<uint16_t*>(bufs + (size_t)p.nu * p.bufcap) + warp * kTileItems;

  if (tid < kMaxUsers) {
    ctl->thr[tid] = 0ull;
    ctl->count[tid] = 0;
    ctl->pass[tid] = 0u;
  }
  if (tid == 0) { ctl->flag = 0; ctl->done = 0; ctl->overflow = 0; }

  // ---- query chunks into registers (lane group member gl owns chunks gl + c*LPR)
  const int g = lane / G::LPR, gl = lane % G::LPR;
  const int nvec = p.nu * p.V;
  int uj[NQV];
#pragma unroll
  for (int j = 0; j < NQV; ++j) uj[j] = (j < nvec) ? j / p.V : -1;

  float qf[kInt ? 1 : NQV][kInt ? 1 : G::CPL][kInt ? 1 : G::EPC];
  uint4 qi[kInt ? NQV : 1][kInt ? G::CPL : 1];
#pragma unroll
  for (int j = 0; j < NQV; ++j) {
#pragma unroll
    for (int c = 0; c < G::CPL; ++c) {
      uint4 raw = make_uint4(0, 0, 0, 0);
      if (j < nvec)
        raw = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(p.q) + (size_t)j * G::ROWB +
                                                   (gl + c * G::LPR) * 16));
      if constexpr (kInt) {
        qi[j][c] = raw;
      } else {
        ChunkDot<DT>::load_q(raw, qf[j][c]);
      }
    }
  }
  __syncthreads();

  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t ntiles = (hwm + kTileItems - 1) / kTileItems;
  uint32_t pcnt[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) pcnt[u] = 0;

  for (int64_t tile = (int64_t)blockIdx.x * NW + warp; tile < ntiles; tile += (int64_t)gridDim.x * NW) {
    if (scan_flag(ctl, lane)) scan_compact_all<NT>(ctl, bufs, p);
    const int64_t base = tile * kTileItems;

    // ---- 1. liveness + clauses -> pass bits
    const uint32_t lw = (lane < 8) ? __ldg(p.live + (base >> 5) + lane) : 0u;
    uint32_t mylive = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) mylive |= ((__shfl_sync(0xffffffffu, lw, t) >> lane) & 1u) << t;
    uint32_t pb[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) pb[u] = (u < p.nu) ? mylive : 0u;
    if (__any_sync(0xffffffffu, mylive != 0)) {
#pragma unroll 1
      for (int w = 0; w < 4; ++w) {
        if (!((p.wmask >> w) & 1u)) continue;
        uint64_t a[8];
        const uint64_t* ap = p.attr + (size_t)w * p.cap_pad + base + lane;
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] = ldg_stream_u64(ap + t * 32);
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          if (u >= p.nu) continue;
          for (int c = 0; c < p.ncl[u]; ++c) {
            const KClause& k = p.cl[u][c];
            if (k.word != (uint32_t)w) continue;
            const unsigned long long m = k.mask;
            const bool rev = k.rev != 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const bool hit = (a[t] & m) != 0ull;
              if (hit == rev) pb[u] &= ~(1u << t);
            }
          }
        }
      }
    }

    // ---- compact passing items of the tile into the warp list
    int cnt = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      uint32_t um = 0;
#pragma unroll
      for (int u = 0; u < NU; ++u) um |= ((pb[u] >> t) & 1u) << u;
      const uint32_t bal = __ballot_sync(0xffffffffu, um != 0u);
      if (um) wlist[cnt + __popc(bal & lanemask_lt())] = (uint16_t)(((t * 32 + lane) << 8) | um);
      cnt += __popc(bal);
    }
#pragma unroll
    for (int u = 0; u < NU; ++u) pcnt[u] += __popc(pb[u]);
    __syncwarp();

    // ---- 2./3. stream passing rows, score, threshold, append
    for (int j0 = 0; j0 < cnt; j0 += G::RPI) {
      uint4 v[G::R][G::CPL];
      uint32_t ent[G::R];
#pragma unroll
      for (int r = 0; r < G::R; ++r) {
        const int idx = j0 + r * G::RPW + g;
        ent[r] = (idx < cnt) ? (uint32_t)wlist[idx] : 0u;
        const char* rowp = reinterpret_cast<const char*>(p.emb) + (size_t)(base + (ent[r] >> 8)) * G::ROWB + gl * 16;
#pragma unroll
        for (int c = 0; c < G::CPL; ++c)
          v[r][c] = ent[r] ? ldg_stream_v4(rowp + c * G::LPR * 16) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < G::R; ++r) {
        acc_t s[NQV];
#pragma unroll
        for (int j = 0; j < NQV; ++j) {
          acc_t acc = 0;
#pragma unroll
          for (int c = 0; c < G::CPL; ++c) {
            if constexpr (kInt) {
              acc = __dp4a((int)v[r][c].x, (int)qi[j][c].x, acc);
              acc = __dp4a((int)v[r][c].y, (int)qi[j][c].y, acc);
              acc = __dp4a((int)v[r][c].z, (int)qi[j][c].z, acc);
              acc = __dp4a((int)v[r][c].w, (int)qi[j][c].w, acc);
            } else {
              acc = ChunkDot<DT>::dot(v[r][c], qf[j][c], acc);
            }
          }
#pragma unroll
          for (int o = G::LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          s[j] = acc;
        }
        const uint32_t gid = p.row0 + (uint32_t)(base + (ent[r] >> 8));
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          float su = -INFINITY;
#pragma unroll
          for (int j = 0; j < NQV; ++j)
            if (uj[j] == u) su = fmaxf(su, (float)s[j]);
          bool cand = false;
          uint64_t key = 0ull;
          if (u < p.nu && gl == 0 && ((ent[r] >> u) & 1u)) {
            key = make_key(su, gid);
            cand = key >= *(volatile const unsigned long long*)&ctl->thr[u];
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, cand);
          if (bal) {
            const int leader = __ffs(bal) - 1;
            const int nb = __popc(bal);
            int pos0 = 0;
            if (lane == leader) {
              pos0 = atomicAdd(&ctl->count[u], nb);
              if (pos0 + nb >= p.C) {
                *(volatile int*)&ctl->flag = 1;
                __threadfence_block();
              }
            }
            pos0 = __shfl_sync(0xffffffffu, pos0, leader);
            if (cand) {
              const int pos = pos0 + __popc(bal & lanemask_lt());
              if (pos < p.bufcap) bufs[(size_t)u * p.bufcap + pos] = key;
              else atomicAdd(&ctl->overflow, 1);
            }
          }
        }
      }
      if (scan_flag(ctl, lane)) scan_compact_all<NT>(ctl, bufs, p);
    }
    __syncwarp();
  }

  // ---- per-CTA pass counts
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    uint32_t c = pcnt[u];
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0 && u < p.nu && c) atomicAdd(&ctl->pass[u], c);
  }

  // ---- termination: keep joining compactions until every warp is done
  if (lane == 0) atomicAdd(&ctl->done, 1);
  while (true) {
    if (scan_flag(ctl, lane)) {
      scan_compact_all<NT>(ctl, bufs, p);
      continue;
    }
    int d = 0;
    if (lane == 0) d = *(volatile int*)&ctl->done;
    d = __shfl_sync(0xffffffffu, d, 0);
    if (d == NW) break;
    __nanosleep(64);
  }
  __syncthreads();

  // ---- 4. final per-CTA top-K: select, sort descending, write
  for (int u = 0; u < p.nu; ++u) {
    uint64_t* b = bufs + (size_t)u * p.bufcap;
    int n = min(ctl->count[u], p.bufcap);
    if (n > p.K) {
      const uint64_t T = block_select_ge<NT>([b](int i) { return b[i]; }, n, p.K, &ctl->sel);
      n = block_compact_ge<NT>(b, n, T, &ctl->sel);
    }
    const int P2 = next_pow2(n > 1 ? n : 1);
    for (int i = n + tid; i < P2; i += NT) b[i] = 0ull;
    __syncthreads();
    block_sort_desc<NT>(b, P2);
    uint64_t* out = p.out_keys + ((size_t)u * gridDim.x + blockIdx.x) * p.K;
    for (int i = tid; i < p.K; i += NT) out[i] = (i < n) ? b[i] : 0ull;
    __syncthreads();
  }
  if (tid < p.nu) {
    p.out_pass[(size_t)tid * gridDim.x + blockIdx.x] = (int64_t)ctl->pass[tid];
  }
  if (tid == 0 && ctl->overflow) atomicAdd(&p.hdr->overflow, (unsigned long long)ctl->overflow);
}

template <int DT>
struct ScanDispatch {
  template <int D, int NQV>
  static constexpr int nt() {
    return (NQV >= 4 || RowGeom<DT, D>::CPL >= 2) ? 512 : 1024;
  }
  template <int D, int NQV>
  static cudaError_t go(const ScanParams& p, int grid, size_t smem, cudaStream_t st) {
    constexpr int NT = nt<D, NQV>();
    auto k = scan_gemv_kernel<DT, D, NQV, NT>;
    static size_t smem_set = 0;   // opt-in size already granted to this instance
    if (smem > smem_set) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      smem_set = smem;
    }
    k<<<grid, NT, smem, st>>>(p);
    return cudaGetLastError();
  }
  template <int D>
  static cudaError_t by_nqv(int nqv, const ScanParams& p, int grid, size_t smem, cudaStream_t st) {
    switch (nqv) {
      case 1: return go<D, 1>(p, grid, smem, st);
      case 2: return go<D, 2>(p, grid, smem, st);
      case 4: return go<D, 4>(p, grid, smem, st);
      case 8: return go<D, 8>(p, grid, smem, st);
    }
    return cudaErrorInvalidValue;
  }
  static cudaError_t launch(int dim, int nqv, const ScanParams& p, int grid, size_t smem, cudaStream_t st) {
    switch (dim) {
      case 16: return by_nqv<16>(nqv, p, grid, smem, st);
      case 32: return by_nqv<32>(nqv, p, grid, smem, st);
      case 64: return by_nqv<64>(nqv, p, grid, smem, st);
      case 128: return by_nqv<128>(nqv, p, grid, smem, st);
      case 256: return by_nqv<256>(nqv, p, grid, smem, st);
      case 512: return by_nqv<512>(nqv, p, grid, smem, st);
      case 1024: return by_nqv<1024>(nqv, p, grid, smem, st);
    }
    return cudaErrorInvalidValue;
  }
  template <int D>
  static ScanCfg cfg_d(int nqv) {
    using G = RowGeom<DT, D>;
    int nt = (nqv >= 4 || G::CPL >= 2) ? 512 : 1024;
    return ScanCfg{nt, G::RPI};
  }
  static ScanCfg cfg(int dim, int nqv) {
    switch (dim) {
      case 16: return cfg_d<16>(nqv);
      case 32: return cfg_d<32>(nqv);
      case 64: return cfg_d<64>(nqv);
      case 128: return cfg_d<128>(nqv);
      case 256: return cfg_d<256>(nqv);
      case 512: return cfg_d<512>(nqv);
      case 1024: return cfg_d<1024>(nqv);
    }
    return ScanCfg{0, 0};
  }
};

}  // namespace linr
