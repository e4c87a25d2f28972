// Fused pre-filter + dot-product score + CTA top-K scan (the "GEMV" path, B*V <= 8 query vectors
// per launch). PAPER.md §3.1: clause evaluation is fused into the scoring
// pass so filtered-out rows are never loaded (the V2 "explicit pre-filtering" idea, P:4284,
// without materialising a slice) and never reach top-K (reading R1: exclusion, not zero-masking).
// The fully fused filter+score+top-K kernel is the option §6 describes for regular KNN.
//
// One persistent CTA per SM owns a contiguous range of 256-item tiles; its warps take tiles
// dynamically. Per warp tile (8 items per lane):
//   1. liveness bits (1 bit/item) + attribute words (8 B/item, coalesced 256 B per warp load,
//      prefetched one tile ahead in registers); evaluate every user's clauses -> per-(user,item)
//      pass bits; compact passing items into a per-warp list in shared memory (ballot + popc).
//   2. gather only the passing rows with cp.async (LDGSTS, 16 B per lane, no register cost) into a
//      per-warp shared-memory ring of S stages, so S-1 row groups are in flight while one is
//      scored; LPR lanes per row, each owning CPL chunks; fp32 FFMA (f32/f16/bf16) or exact int32
//      DP4A (int8) against the query chunk held in registers; butterfly-reduce over the LPR lanes;
//      max over the user's V vectors (reading R12).
//   3. threshold test against the CTA's current per-user bound, warp-aggregated append of packed
//      (score,id) keys to the CTA's shared-memory buffer, and insertion into the warp's sorted
//      top-32 register list (warp select). When a buffer passes its soft capacity the whole CTA
//      radix-selects the K-th key and compacts (exact: keys below the K-th of K kept keys can
//      never enter the top-K).
//   4. at the end the CTA merges its warps' top-32 lists into its sorted top-32 "sample" and
//      writes the sample plus its (unsorted) buffer; merge.cu combines the CTAs: the K-th key of
//      the union of samples bounds the answer from below, so normally only samples are read.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "merge.cuh"

namespace linr {

// Row geometry. LPR lanes cooperate on one row, each owning CPL 16-byte chunks (chunk gl + c*LPR,
// so one load instruction of a row group reads LPR*16 contiguous bytes: full 32-byte sectors);
// RPW rows per warp instruction, R rows in flight per lane group. LPR = 4 keeps the per-row
// bookkeeping (butterfly reduce, key, threshold, append ballot) amortised over 8 rows per warp
// instruction while keeping 64-byte contiguous segments per row per load.
// Row geometry. LPR lanes cooperate on one row, each owning CPL 16-byte chunks (chunk gl + c*LPR,
// so one load instruction of a row group reads LPR*16 contiguous bytes: full 32-byte sectors);
// RPW rows per warp instruction, R rows in flight per lane group. Few lanes per row (LPR = 4)
// amortise the per-row bookkeeping (butterfly reduce, key, threshold, append ballot) over 8 rows
// per warp instruction; with more query vectors LPR grows so the per-lane query chunks (NQV*CPL
// chunks held in registers) stay within budget.
constexpr int geom_lpr(int CH, int NQV, int PER) {
  int lpr = CH / 4 > 4 ? CH / 4 : 4;
  if (lpr > 32) lpr = 32;
  if (lpr > CH) lpr = CH;
  while (lpr < CH && lpr < 32 && NQV * (CH / lpr) * PER > 32) lpr *= 2;
  return lpr;
}

template <int DT, int D, int NQV = 1>
struct RowGeom {
  static constexpr int ESZ = (DT == LINR_F32) ? 4 : (DT == LINR_I8 ? 1 : 2);
  static constexpr int ROWB = D * ESZ;          // bytes per row
  static constexpr int CH = ROWB / 16;          // 16-byte chunks per row
  static constexpr int EPC = 16 / ESZ;          // elements per chunk
  static constexpr int PER = (DT == LINR_I8) ? 4 : EPC;   // query registers per chunk
  static constexpr int LPR = geom_lpr(CH, NQV, PER);      // lanes per row
  static constexpr int CPL = CH / LPR;          // chunks per lane
  static constexpr int RPW = 32 / LPR;          // rows per warp step
  static constexpr int R = CPL >= 4 ? 1 : 4 / CPL;  // rows in flight per lane group
  static constexpr int RPI = RPW * R;           // rows per warp iteration
  static constexpr int STG = RPI * ROWB >= 4096 ? 2 : 4;   // cp.async ring depth (4 KB rows: 2, so 16 warps fit)
  static_assert(ROWB % 16 == 0, "row must be a multiple of 16 bytes");
  static_assert(CH % LPR == 0, "chunks must split evenly over the lanes of a row");
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
  int next_tile;                       // CTA-local dynamic tile counter
  int wcnt;                            // write counter for the final list
  int ticket;                          // fused-merge ticket of this CTA
  // warp-specialised scan (scan_ws_kernel): row-group ring bookkeeping
  int ghead;                           // row groups allocated by the producer warps
  int gtotal;                          // total groups, published when every producer is done
  int pdone;                           // warps finished filtering
  int gcons;                           // row groups claimed by scoring warps
};

static_assert(sizeof(ScanCtl) + 16 <= 2048, "host plan reserves 2 KB for ScanCtl (api.cu kScanCtlBytes)");

constexpr int kSample = kScanSample;   // sorted per-CTA sample length (merge pruning)

LINR_DEV bool scan_flag(const ScanCtl* ctl, int lane) {
  int f = 0;
  if (lane == 0) f = *(volatile const int*)&ctl->flag;
  return __shfl_sync(0xffffffffu, f, 0) != 0;
}

LINR_DEV void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}
LINR_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
LINR_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NT>
__device__ __noinline__ void scan_compact_all(ScanCtl* ctl, uint64_t* bufs, const ScanParams& p) {
  __syncthreads();   // every warp of the CTA is here (flag checks are warp-uniform)
  if (p.dbg != nullptr && threadIdx.x == 0) atomicAdd(&p.dbg[blockIdx.x * 8 + 7], 1ull);
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

// ---------------------------------------------------------------- tensor-core GEMV geometry
// bf16/f16 (mma.m16n8k16, fp32 accumulate) and int8 (mma.m16n8k32, exact s32 accumulate): a warp
// scores 16 gathered rows against up to 8 query vectors (the mma's n = 8 columns) per group. The
// rows sit in a per-warp shared-memory ring filled by cp.async with an XOR swizzle on the 16-byte
// chunk index so ldmatrix reads 8 rows at the same column without bank conflicts. The path is
// HBM-bound; the mma only replaces ~8 CUDA-core instructions per row (unpack + FFMA + butterfly)
// with ~1 (ldmatrix + mma per 16 rows x 16/32 k), cutting issue pressure. f32 (no exact tensor-core
// path) and other shapes use the FFMA geometry above.
template <int DT, int D>
struct MmaGeom {
  static constexpr bool ok = ((DT == LINR_BF16 || DT == LINR_F16) && D >= 16 && D <= 128) ||
                             (DT == LINR_I8 && D >= 32 && D <= 256);
  static constexpr int ESZ = (DT == LINR_I8) ? 1 : 2;
  static constexpr int ROWB = D * ESZ;
  static constexpr int CH = ROWB / 16;           // 16-byte chunks per row
  static constexpr int NKS = ROWB / 32;          // k-steps of 32 bytes (k16 bf16 / k32 int8)
  static constexpr int ROWS = 16;                // rows per group
  static constexpr int STAGE = ROWS * ROWB;
  static constexpr int S0 = 8192 / (STAGE > 0 ? STAGE : 1);
  static constexpr int S = S0 < 2 ? 2 : (S0 > 4 ? 4 : S0);   // ring stages
  static constexpr int CPLN = (ROWS * CH) / 32 > 0 ? (ROWS * CH) / 32 : 1;   // chunks per lane per stage
  static constexpr int SWZ_DIV = CH >= 8 ? 1 : 8 / (CH > 0 ? CH : 1);
  static constexpr int SWZ_MOD = CH >= 8 ? 8 : CH;
  LINR_DEV static int swz(int row) { return (row / SWZ_DIV) % (SWZ_MOD > 0 ? SWZ_MOD : 1); }
};

LINR_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

template <int DT>
LINR_DEV void mma16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (DT == LINR_BF16) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
}
LINR_DEV void mma32_s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NT, int NU>
struct Appender {
  // Threshold test + warp-aggregated append of candidate keys into the CTA buffer of user u.
  LINR_DEV static void append(ScanCtl* ctl, uint64_t* bufs, const ScanParams& p, int u, bool cand_in, uint64_t key) {
    const int lane = threadIdx.x & 31;
    bool cand = cand_in && key >= *(volatile const unsigned long long*)&ctl->thr[u];
    const uint32_t bal = __ballot_sync(0xffffffffu, cand);
    if (!bal) return;
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
};

template <int DT, int D, int NQV>
struct ScanGeom {
  static constexpr bool kMma = MmaGeom<DT, D>::ok && NQV <= 8;
  static constexpr int RPI = kMma ? 16 : RowGeom<DT, D, NQV>::RPI;   // rows per warp iteration
  static constexpr int RING = kMma ? MmaGeom<DT, D>::S * MmaGeom<DT, D>::STAGE
                                   : RowGeom<DT, D, NQV>::STG * RowGeom<DT, D, NQV>::RPI * RowGeom<DT, D, NQV>::ROWB;
};

// Per-CTA output (sorted top-32 sample + every kept key) and the fused merge, run by all NT
// threads of the CTA once the scan of its range is complete. rings: >= 512 idle bytes (scratch).
template <int NT>
__device__ __forceinline__ void scan_tail(ScanCtl* ctl, uint64_t* bufs, const ScanParams& p, unsigned char* rings,
                                          unsigned char* smem_raw, size_t ring_bytes) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- 4. per-CTA output: sorted top-32 sample + the whole (unsorted) buffer
  uint64_t* scratch64 = reinterpret_cast<uint64_t*>(rings);   // 64 keys (the rings are idle now)
  const size_t cta = (size_t)blockIdx.x;
  for (int u = 0; u < p.nu; ++u) {
    uint64_t* b = bufs + (size_t)u * p.bufcap;
    int n = min(ctl->count[u], p.bufcap);
    bool sample_full64 = false;   // scratch64[32..64) holds candidates too (sorted with the rest)
    if (n > p.list_cap) {
      const uint64_t T = block_select_ge<NT>([b](int i) { return b[i]; }, n, p.K, &ctl->sel);
      n = block_compact_ge<NT>(b, n, T, &ctl->sel);
    }
    // sample: the top-32 keys, sorted
    const int tail_cap = (int)min((size_t)1024, ring_bytes / 8 - 64);
    if (n > kSample && tail_cap < NT) {   // no room for the candidate pass: select over the buffer
      const uint64_t T = block_select_ge<NT>([b](int i) { return b[i]; }, n, kSample, &ctl->sel);
      if (tid == 0) ctl->wcnt = 0;
      __syncthreads();
      for (int i0 = 0; i0 < n; i0 += NT) {
        const int i = i0 + tid;
        const bool top = i < n && b[i] >= T;
        const uint32_t bal = __ballot_sync(0xffffffffu, top);
        int at = 0;
        if (lane == 0 && bal) at = atomicAdd(&ctl->wcnt, __popc(bal));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (top) scratch64[at + __popc(bal & lanemask_lt())] = b[i];
      }
      __syncthreads();
    } else if (n > kSample) {
      // T0 = the 32nd largest of the threads' local maxima bounds the CTA's 32nd key from below
      // (those 32 keys exist), so the top 32 are among the keys >= T0 -- usually a few dozen.
      // T0 comes from a warp bitonic sort of each warp's 32 maxima and a tree of top-32 bitonic
      // merges; the candidates >= T0 are sorted by one warp. Fallback: radix select.
      const int kTailCand = tail_cap;
      uint64_t* cand = scratch64 + 64;          // the rings are idle: room for kTailCand keys
      uint64_t mx = 0ull;
      for (int i = tid; i < n; i += NT) mx = b[i] > mx ? b[i] : mx;
      {   // rank sort of the warp's 32 maxima: keys are distinct, only zero maxima (threads
          // without keys) tie, and ties rank by lane
        int r = 0;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
          const uint64_t y = shfl_idx_u64(mx, j);
          r += (y > mx) || (y == mx && j < lane);
        }
        cand[warp * 32 + r] = mx;   // warp w's maxima, sorted descending, at cand[32w ..]
      }
      __syncthreads();
      constexpr int NW = NT / 32;
      for (int span = 1; span < NW; span <<= 1) {
        if ((warp & (2 * span - 1)) == 0) {
          const uint64_t x = cand[warp * 32 + lane], y = cand[(warp + span) * 32 + 31 - lane];
          uint64_t v = x > y ? x : y;   // bitonic: the top 32 of the two lists
#pragma unroll 1
          for (int j = 16; j > 0; j >>= 1) {
            const uint64_t pv = shfl_xor_u64(v, j);
            v = ((lane & j) == 0) ? (v > pv ? v : pv) : (v < pv ? v : pv);
          }
          cand[warp * 32 + lane] = v;
        }
        __syncthreads();
      }
      const uint64_t T0 = cand[31];
      if (tid == 0) ctl->wcnt = 0;
      __syncthreads();
      {   // collect the keys >= T0: count per thread, one warp scan and one atomic per warp
        int c = 0;
        for (int i = tid; i < n; i += NT) c += (b[i] >= T0) ? 1 : 0;   // keys are nonzero
        int incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += t;
        }
        int base = 0;
        if (lane == 31 && incl) base = atomicAdd(&ctl->wcnt, incl);
        int pos = __shfl_sync(0xffffffffu, base, 31) + incl - c;
        for (int i = tid; i < n && c > 0; i += NT) {
          const uint64_t v = b[i];
          if (v >= T0) {
            if (pos < kTailCand) cand[pos] = v;
            ++pos;
            --c;
          }
        }
      }
      __syncthreads();
      const int m = ctl->wcnt;
      if (m <= 64) {   // one warp sorts the candidates; the first 32 are the sample
        sample_full64 = true;
        if (warp == 0) {
          scratch64[lane] = lane < m ? cand[lane] : 0ull;
          scratch64[lane + 32] = lane + 32 < m ? cand[lane + 32] : 0ull;
        }
        __syncthreads();
      } else {
        const bool small = m <= kTailCand;
        const uint64_t T = small ? block_select_ge<NT>([cand](int i) { return cand[i]; }, m, kSample, &ctl->sel)
                                 : block_select_ge<NT>([b](int i) { return b[i]; }, n, kSample, &ctl->sel);
        if (tid == 0) ctl->wcnt = 0;
        __syncthreads();
        const int mm = small ? m : n;
        const uint64_t* src = small ? cand : b;
        for (int i0 = 0; i0 < mm; i0 += NT) {
          const int i = i0 + tid;
          const uint64_t v = i < mm ? src[i] : 0ull;
          const bool top = i < mm && v >= T && v != 0ull;
          const uint32_t bal = __ballot_sync(0xffffffffu, top);
          int at = 0;
          if (lane == 0 && bal) at = atomicAdd(&ctl->wcnt, __popc(bal));
          at = __shfl_sync(0xffffffffu, at, 0);
          if (top) scratch64[at + __popc(bal & lanemask_lt())] = v;
        }
        __syncthreads();
      }
    } else {
      for (int i = tid; i < kSample; i += NT) scratch64[i] = i < n ? b[i] : 0ull;
      __syncthreads();
    }
    if (u == 0) dbg_mark(p.dbg, blockIdx.x * 8 + 2);
    uint64_t* samp = p.out_samp + ((size_t)u * gridDim.x + cta) * kSample;
    if (warp == 0) {
      if (!sample_full64) scratch64[32 + lane] = 0ull;
      __syncwarp();
      // rank sort of <= 64 distinct nonzero keys (zeros are padding): a key's position is the
      // number of larger keys -- 32 independent broadcast steps instead of a 21-stage network
      const uint64_t x0 = scratch64[lane], x1 = scratch64[lane + 32];
      int r0 = 0, r1 = 0;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const uint64_t y0 = shfl_idx_u64(x0, j), y1 = shfl_idx_u64(x1, j);
        r0 += (y0 > x0) + (y1 > x0);
        r1 += (y0 > x1) + (y1 > x1);
      }
      samp[lane] = 0ull;
      __syncwarp();
      if (x0 != 0ull && r0 < kSample) samp[r0] = x0;
      if (x1 != 0ull && r1 < kSample) samp[r1] = x1;
    }
    if (u == 0) dbg_mark(p.dbg, blockIdx.x * 8 + 6);
    uint64_t* lst = p.out_list + ((size_t)u * gridDim.x + cta) * p.list_cap;
    for (int i = tid; i < n; i += NT) lst[i] = b[i];
    if (tid == 0) p.out_cnt[(size_t)u * gridDim.x + cta] = n;
    __syncthreads();
  }
  if (tid < p.nu) p.out_pass[(size_t)tid * gridDim.x + cta] = (int64_t)ctl->pass[tid];
  if (tid == 0 && ctl->overflow) atomicAdd(&p.hdr->overflow, (unsigned long long)ctl->overflow);
  dbg_mark(p.dbg, blockIdx.x * 8 + 3);

  // ---- 5. fused merge: the last nu CTAs to finish merge one user each (no extra launch)
  if (!p.fuse_merge) return;
  __threadfence();   // this CTA's outputs are visible before it takes a ticket
  __syncthreads();
  if (tid == 0) ctl->ticket = (int)atomicAdd(&p.hdr->done_ctas[p.fuse_slot], 1u);
  __syncthreads();
  const int ticket = ctl->ticket;
  const int first = (int)gridDim.x - p.nu;
  if (ticket < first) return;
  if (tid == 0) {   // wait until every CTA of this launch has published its outputs
    while (*(volatile unsigned int*)&p.hdr->done_ctas[p.fuse_slot] < gridDim.x) __nanosleep(64);
  }
  __syncthreads();
  __threadfence();
  merge_user<NT>(p.mp, ticket - first, smem_raw);
  if (tid == 0) {
    if (atomicAdd(&p.hdr->merged[p.fuse_slot], 1u) == (unsigned int)p.nu - 1) {   // last merger resets the slot
      p.hdr->merged[p.fuse_slot] = 0u;
      __threadfence();
      atomicExch(&p.hdr->done_ctas[p.fuse_slot], 0u);
    }
  }
}

template <int DT, int D, int NQV, int NT>
__global__ void __launch_bounds__(NT, 1) scan_gemv_kernel(const __grid_constant__ ScanParams p) {
  asm volatile("griddepcontrol.launch_dependents;");   // see scan_ws_kernel
  using G = RowGeom<DT, D, NQV>;
  using M = MmaGeom<DT, D>;
  constexpr bool kMma = ScanGeom<DT, D, NQV>::kMma;
  constexpr bool kInt = (DT == LINR_I8);
  using acc_t = typename std::conditional<kInt, int, float>::type;
  constexpr int NW = NT / 32;
  constexpr int NU = NQV;   // at most one user per vector
  constexpr int RING = ScanGeom<DT, D, NQV>::RING;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScanCtl* ctl = reinterpret_cast<ScanCtl*>(smem_raw);
  uint64_t* bufs = reinterpret_cast<uint64_t*>(smem_raw + ((sizeof(ScanCtl) + 15) & ~size_t(15)));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint16_t* wlist_all = reinterpret_cast<uint16_t*>(bufs + (size_t)p.nu * p.bufcap);
  uint16_t* wlist = wlist_all + warp * kTileItems;
  unsigned char* rings = reinterpret_cast<unsigned char*>(wlist_all + NW * kTileItems);   // 16B aligned
  unsigned char* ring = rings + (size_t)warp * RING;

  if (tid < kMaxUsers) {
    ctl->thr[tid] = (p.init_thr != nullptr && tid < p.nu) ? p.init_thr[tid] : 0ull;
    ctl->count[tid] = 0;
    ctl->pass[tid] = 0u;
  }
  if (tid == 0) { ctl->flag = 0; ctl->done = 0; ctl->overflow = 0; ctl->next_tile = 0; }

  const int nvec = p.nu * p.V;
  // ---- query registers
  // FFMA path: lane group member gl owns chunks gl + c*LPR of every query vector.
  // MMA path: B fragments; lane (g = lane/4, t = lane%4) holds vector g's k-pairs 2t, 2t+8 (bf16)
  // or k-quads 4t, 4t+16 (int8) of every k-step.
  const int g = lane / G::LPR, gl = lane % G::LPR;
  int uj[NQV];
#pragma unroll
  for (int j = 0; j < NQV; ++j) uj[j] = (j < nvec) ? j / p.V : -1;
  float qf[(kInt || kMma) ? 1 : NQV][(kInt || kMma) ? 1 : G::CPL][(kInt || kMma) ? 1 : G::EPC];
  uint4 qi[(kInt && !kMma) ? NQV : 1][(kInt && !kMma) ? G::CPL : 1];
  uint32_t bq[kMma ? M::NKS : 1][2];
  int ucol0 = -1, ucol1 = -1;   // MMA path: user of this lane's two accumulator columns
  if constexpr (kMma) {
    const int mg = lane >> 2, mt = lane & 3;
    ucol0 = (2 * mt < nvec) ? (2 * mt) / p.V : -1;
    ucol1 = (2 * mt + 1 < nvec) ? (2 * mt + 1) / p.V : -1;
    const char* qv = reinterpret_cast<const char*>(p.q) + (size_t)mg * M::ROWB;
#pragma unroll
    for (int ks = 0; ks < M::NKS; ++ks) {
      uint32_t b0 = 0, b1 = 0;
      if (mg < nvec) {
        const int o0 = kInt ? (ks * 32 + 4 * mt) : (ks * 16 + 2 * mt) * 2;
        const int o1 = kInt ? (ks * 32 + 4 * mt + 16) : (ks * 16 + 2 * mt + 8) * 2;
        b0 = __ldg(reinterpret_cast<const unsigned int*>(qv + o0));
        b1 = __ldg(reinterpret_cast<const unsigned int*>(qv + o1));
      }
      bq[ks][0] = b0;
      bq[ks][1] = b1;
    }
  } else {
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
  }
  __syncthreads();
  dbg_mark(p.dbg, blockIdx.x * 8 + 0);

  // ---- this CTA's contiguous tile range; warps take tiles from it dynamically
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t ntiles = (hwm + kTileItems - 1) / kTileItems;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  auto grab = [&]() -> int64_t {
    int t = 0;
    if (lane == 0) t = atomicAdd(&ctl->next_tile, 1);
    return t_begin + __shfl_sync(0xffffffffu, t, 0);
  };
  const bool w0 = (p.wmask & 1u) != 0;
  auto prefetch = [&](int64_t tile, uint64_t (&a)[8], uint32_t& lw) {
    const int64_t base = tile * kTileItems;
    lw = (lane < 8) ? __ldg(p.live + (base >> 5) + lane) : 0u;
    if (w0) {
      const uint64_t* ap = p.attr + base + lane;
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] = ldg_stream_u64(ap + t * 32);
    }
  };

  uint32_t pcnt[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) pcnt[u] = 0;

  // attribute words + liveness of the next two tiles are in flight while a tile is processed
  int64_t tile = grab();
  uint64_t a[8], na[8];
  uint32_t lw = 0, nlw = 0;
  if (tile < t_end) prefetch(tile, a, lw);
  int64_t next = grab();
  if (next < t_end) prefetch(next, na, nlw);
  while (tile < t_end) {
    if (scan_flag(ctl, lane)) scan_compact_all<NT>(ctl, bufs, p);
    const int64_t next2 = grab();
    uint64_t nna[8];
    uint32_t nnlw = 0;
    if (next2 < t_end) prefetch(next2, nna, nnlw);
    const int64_t base = tile * kTileItems;

    // ---- 1. liveness + clauses -> pass bits
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
        uint64_t aw[8];
        if (w == 0) {
#pragma unroll
          for (int t = 0; t < 8; ++t) aw[t] = a[t];
        } else {
          const uint64_t* ap = p.attr + (size_t)w * p.cap_pad + base + lane;
#pragma unroll
          for (int t = 0; t < 8; ++t) aw[t] = ldg_stream_u64(ap + t * 32);
        }
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
              const bool hit = (aw[t] & m) != 0ull;
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

    if constexpr (kMma) {
      // ---- 2./3. tensor-core path: 16-row groups through the swizzled cp.async ring
      const int ngrp = (cnt + M::ROWS - 1) / M::ROWS;
      // copy mapping: LPRC lanes per row, each copying CPR chunks (chunk cl + k*LPRC), so one
      // instruction moves LPRC*16 contiguous bytes of each of 32/LPRC rows (full 32-byte sectors);
      // one wlist lookup and one base address per row per lane.
      constexpr int LPRC = M::CH < 4 ? M::CH : 4;
      constexpr int RPS = 32 / LPRC;                 // rows per copy step
      constexpr int NRS = M::ROWS / RPS;             // copy steps per group
      constexpr int CPR = M::CH / LPRC;              // chunks per lane per row
      const int crow = lane / LPRC, cl = lane % LPRC;
      auto issue = [&](int gi) {
        unsigned char* st = ring + (gi % M::S) * M::STAGE;
#pragma unroll
        for (int rs = 0; rs < NRS; ++rs) {
          const int row = crow + rs * RPS;
          const int idx = gi * M::ROWS + row;
          const uint32_t e = (idx < cnt) ? (uint32_t)wlist[idx] : 0u;
          const char* src = reinterpret_cast<const char*>(p.emb) + (size_t)(base + (e >> 8)) * M::ROWB;
          unsigned char* dst = st + row * M::ROWB;
          const int sw = M::swz(row);
          const int bytes = e ? 16 : 0;
#pragma unroll
          for (int k = 0; k < CPR; ++k) {
            const int c = cl + k * LPRC;
            cp_async16(dst + ((c ^ sw) * 16), src + c * 16, bytes);
          }
        }
        cp_async_commit();
      };
#pragma unroll
      for (int gi = 0; gi < M::S - 1; ++gi) {
        if (gi < ngrp) issue(gi); else cp_async_commit();
      }
      const int mg = lane >> 2, mt = lane & 3;
      for (int gi = 0; gi < ngrp; ++gi) {
        if (gi + M::S - 1 < ngrp) issue(gi + M::S - 1); else cp_async_commit();
        cp_async_wait<M::S - 1>();
        __syncwarp();   // the group's rows were copied by every lane of the warp
        const unsigned char* st = ring + (gi % M::S) * M::STAGE;
        const uint32_t st_s = (uint32_t)__cvta_generic_to_shared(st);
        acc_t acc[4] = {0, 0, 0, 0};
        const int lrow = lane & 15, lhalf = lane >> 4;
#pragma unroll
        for (int ks = 0; ks < M::NKS; ++ks) {
          uint32_t af[4];
          const int chunk = ks * 2 + lhalf;
          ldsm_x4(st_s + lrow * M::ROWB + ((chunk ^ M::swz(lrow)) * 16), af[0], af[1], af[2], af[3]);
          if constexpr (kInt) mma32_s8(acc, af, bq[ks][0], bq[ks][1]);
          else mma16<DT>(acc, af, bq[ks][0], bq[ks][1]);
        }
        // accumulator: acc[0..1] = row mg, columns 2mt, 2mt+1; acc[2..3] = row mg+8
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = mg + 8 * h;
          const int idx = gi * M::ROWS + row;
          const uint32_t ent = (idx < cnt) ? (uint32_t)wlist[idx] : 0u;
          const uint32_t gid = p.row0 + (uint32_t)(base + (ent >> 8));
          const float v0 = (float)acc[2 * h], v1 = (float)acc[2 * h + 1];
          if constexpr (NQV == 1) {   // one user, one vector: column 0 lives in lanes mt == 0
            const bool cand = p.nu > 0 && mt == 0 && (ent & 1u);
            Appender<NT, NU>::append(ctl, bufs, p, 0, cand, cand ? make_key(v0, gid) : 0ull);
          } else {
#pragma unroll
            for (int u = 0; u < NU; ++u) {
              float m = -INFINITY;
              if (ucol0 == u) m = v0;
              if (ucol1 == u) m = fmaxf(m, v1);
              m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
              m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
              const bool cand = u < p.nu && mt == 0 && ((ent >> u) & 1u);
              Appender<NT, NU>::append(ctl, bufs, p, u, cand, cand ? make_key(m, gid) : 0ull);
            }
          }
        }
        __syncwarp();   // every lane is done reading this stage before it is refilled
        if (scan_flag(ctl, lane)) scan_compact_all<NT>(ctl, bufs, p);
      }
    } else {
      // ---- 2./3. CUDA-core path: LPR lanes per row, cp.async ring of G::STG stages
      constexpr int kStages = G::STG;
      const int n_iter = (cnt + G::RPI - 1) / G::RPI;
      constexpr int STAGE = G::RPI * G::ROWB;
      auto issue = [&](int it) {
        unsigned char* st = ring + (it % kStages) * STAGE;
#pragma unroll
        for (int r = 0; r < G::R; ++r) {
          const int slot = r * G::RPW + g;
          const int idx = it * G::RPI + slot;
          const uint32_t e = (idx < cnt) ? (uint32_t)wlist[idx] : 0u;
          const char* src = reinterpret_cast<const char*>(p.emb) + (size_t)(base + (e >> 8)) * G::ROWB + gl * 16;
#pragma unroll
          for (int c = 0; c < G::CPL; ++c)
            cp_async16(st + slot * G::ROWB + (gl + c * G::LPR) * 16, src + c * G::LPR * 16, e ? 16 : 0);
        }
        cp_async_commit();
      };
#pragma unroll
      for (int it = 0; it < kStages - 1; ++it) {
        if (it < n_iter) issue(it); else cp_async_commit();
      }
      for (int it = 0; it < n_iter; ++it) {
        if (it + kStages - 1 < n_iter) issue(it + kStages - 1); else cp_async_commit();
        cp_async_wait<kStages - 1>();   // each lane reads back only the chunks it copied
        const unsigned char* st = ring + (it % kStages) * STAGE;
#pragma unroll
        for (int r = 0; r < G::R; ++r) {
          const int slot = r * G::RPW + g;
          const int idx = it * G::RPI + slot;
          const uint32_t ent = (idx < cnt) ? (uint32_t)wlist[idx] : 0u;
          uint4 v[G::CPL];
#pragma unroll
          for (int c = 0; c < G::CPL; ++c)
            v[c] = *reinterpret_cast<const uint4*>(st + slot * G::ROWB + (gl + c * G::LPR) * 16);
          acc_t s[NQV];
#pragma unroll
          for (int j = 0; j < NQV; ++j) {
            acc_t acc = 0;
#pragma unroll
            for (int c = 0; c < G::CPL; ++c) {
              if constexpr (kInt) {
                acc = __dp4a((int)v[c].x, (int)qi[j][c].x, acc);
                acc = __dp4a((int)v[c].y, (int)qi[j][c].y, acc);
                acc = __dp4a((int)v[c].z, (int)qi[j][c].z, acc);
                acc = __dp4a((int)v[c].w, (int)qi[j][c].w, acc);
              } else {
                acc = ChunkDot<DT>::dot(v[c], qf[j][c], acc);
              }
            }
#pragma unroll
            for (int o = G::LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            s[j] = acc;
          }
          const uint32_t gid = p.row0 + (uint32_t)(base + (ent >> 8));
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            float su = -INFINITY;
#pragma unroll
            for (int j = 0; j < NQV; ++j)
              if (uj[j] == u) su = fmaxf(su, (float)s[j]);
            const bool cand = u < p.nu && gl == 0 && ((ent >> u) & 1u);
            Appender<NT, NU>::append(ctl, bufs, p, u, cand, cand ? make_key(su, gid) : 0ull);
          }
        }
        if (scan_flag(ctl, lane)) scan_compact_all<NT>(ctl, bufs, p);
      }
    }
    cp_async_wait<0>();
    __syncwarp();
    tile = next;
    next = next2;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      a[t] = na[t];
      na[t] = nna[t];
    }
    lw = nlw;
    nlw = nnlw;
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
    __nanosleep(256);
  }
  __syncthreads();
  dbg_mark(p.dbg, blockIdx.x * 8 + 1);

  scan_tail<NT>(ctl, bufs, p, rings, smem_raw, (size_t)NW * RING);
}

}  // namespace linr
