// Batched filtered top-K on the 5th-generation tensor cores (tcgen05), for query batches that make
// scoring a real GEMM (B*V >= 16 query vectors): BASELINE.json north_star "tcgen05 tensor-core
// tiles (kind::f16 and kind::i8) only when the query batch makes scoring a real GEMM".
//
// Per search (all launches on the caller's stream, no host synchronisation on the common path):
//   1. tc_scan_kernel<SAMPLE>: a few 128-item tiles per CTA, evenly spread over the index; every
//      passing (user, item) key is appended to the user's sample buffer.
//   2. tc_threshold_kernel: per user, T_u = a key with exactly r sample keys >= T_u, where r is the
//      sample count expected above the answer's K-th key plus a 6-sigma margin; T_u = 0 if the
//      sample holds fewer than r keys (no filtering).
//   3. tc_scan_kernel<MAIN>: every tile. Warp-specialised persistent CTA: warp 0 issues TMA loads
//      (128-row item tile, 128B-swizzled, + the tile's attribute words and liveness bits) into a
//      2-stage shared-memory ring; warp 1 issues tcgen05.mma (M=128 items x N=NP query vectors,
//      K=16 bf16/f16 or 32 int8 per instruction) into a double-buffered TMEM accumulator (fp32 or
//      exact s32); warps 4-7 (one TMEM lane = one item row per thread) tcgen05.ld the scores,
//      max-merge each user's V columns, compare against T_u first (cheap), evaluate the user's
//      clauses only for the rare survivors (P:4266 semantics) and append survivors' keys.
//   4. tc_finalize_kernel: per user, the K largest appended keys, sorted, decoded; a flag marks
//      users whose result cannot be certified (buffer overflow, or T_u > 0 with fewer than K keys
//      appended); 5. fallback.cu recomputes the flagged users exactly on the device.
// Exactness: every key >= T_u is appended; if at least K are, the K-th is >= T_u, so the top-K
// of the buffer is the top-K of the user's passing items (reading R13-style argument).
#include <cuda.h>

#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"

namespace linr {

constexpr int kTcThreads = 640;   // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-19 epilogue (4 column groups)
constexpr int kTcXStagesMax = 6;  // item-tile ring (released by the MMA commit): as many as shared memory holds
constexpr int kTcAStages = 8;     // attribute ring (released by the epilogue): deeper than the item ring so
                                  // the producer runs ahead of the epilogue by the item ring, not by this one
constexpr size_t kTcSmemBudget = 232448 - 1024;   // sm_100 opt-in shared memory per CTA minus the kernel's 1 KB static segment
constexpr int kTcRows = 128;

// ------------------------------------------------------------------ PTX helpers
LINR_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
LINR_DEV void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
LINR_DEV void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
LINR_DEV void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
LINR_DEV void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 2000;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
LINR_DEV void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
LINR_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
LINR_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LINR_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
LINR_DEV void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
template <int DT>
LINR_DEV void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  if constexpr (DT == LINR_I8) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
LINR_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
LINR_DEV void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// one column (x1) / a user's V aligned columns (x2, x4), maxed: the main pass re-reads hot columns
LINR_DEV uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return r;
}
LINR_DEV void tmem_ld2(uint32_t taddr, uint32_t (&v)[2]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
LINR_DEV void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
LINR_DEV void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major shared-memory matrix descriptor (canonical layout: rows of SW bytes, 8-row core groups
// SBO = 8*SW bytes apart, SW-byte swizzle; SM100 descriptor version 1).
template <int SW>
LINR_DEV uint64_t umma_desc(uint32_t saddr) {
  constexpr uint64_t layout = SW == 128 ? 2 : (SW == 64 ? 4 : 6);
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                          // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(((8 * SW) >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                          // version
  d |= layout << 61;
  return d;
}

template <int DT, int NP>
constexpr uint32_t tc_idesc() {
  // c_format [4,6): 1 = F32, 2 = S32; a/b format [7,10)/[10,13): F16 0, BF16 1, S8 signed 1;
  // K-major A and B; n_dim [17,23) = N >> 3; m_dim [24,29) = M >> 4
  uint32_t d = 0;
  if (DT == LINR_I8) {
    d |= 2u << 4;
    d |= 1u << 7;
    d |= 1u << 10;
  } else {
    d |= 1u << 4;
    const uint32_t f = (DT == LINR_BF16) ? 1u : 0u;
    d |= f << 7;
    d |= f << 10;
  }
  d |= (uint32_t)(NP >> 3) << 17;
  d |= (uint32_t)(kTcRows >> 4) << 24;
  return d;
}

template <int DT, int D>
struct TcGeom {
  static constexpr int ESZ = DT == LINR_I8 ? 1 : 2;
  static constexpr int ROWB = D * ESZ;
  static constexpr int SW = ROWB >= 128 ? 128 : ROWB;   // swizzle span = box inner bytes
  static constexpr int NATOM = ROWB / SW;                // swizzle atoms along K
  static constexpr int KSTEP_B = 32;                     // bytes of K per MMA (16 x 2B or 32 x 1B)
  static constexpr int KPA = SW / KSTEP_B;               // MMAs per atom
  static constexpr int NKS = ROWB / KSTEP_B;
  static constexpr int XBYTES = kTcRows * ROWB;
};

struct TcSmemCtl {
  uint64_t xfull[kTcXStagesMax], xempty[kTcXStagesMax], afull[kTcAStages], aempty[kTcAStages];
  uint64_t tfull[2], tempty[2], qbar;
  uint32_t tmem_base;
};

template <int CW>
LINR_DEV void tmem_ld(uint32_t taddr, uint32_t (&v)[CW]) {
  if constexpr (CW == 32) tmem_ld32(taddr, v);
  else if constexpr (CW == 16) tmem_ld16(taddr, v);
  else tmem_ld8(taddr, v);
}
// max over n (compile-time) floats: tree of 3-input maxima
template <int N>
LINR_DEV float fmax_tree(const float* a);
LINR_DEV float fmax3(float a, float b, float c);
template <int N>
LINR_DEV float fmax_tree(const float* a) {
  if constexpr (N == 1) return a[0];
  else if constexpr (N == 2) return fmaxf(a[0], a[1]);
  else if constexpr (N == 3) return fmax3(a[0], a[1], a[2]);
  else {
    constexpr int M = (N + 2) / 3;
    float b[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      if (3 * k + 2 < N) b[k] = fmax3(a[3 * k], a[3 * k + 1], a[3 * k + 2]);
      else if (3 * k + 1 < N) b[k] = fmaxf(a[3 * k], a[3 * k + 1]);
      else b[k] = a[3 * k];
    }
    return fmax_tree<M>(b);
  }
}
LINR_DEV float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
template <bool kInt>
LINR_DEV uint32_t vmax(uint32_t a, uint32_t b) {
  if (kInt) return (uint32_t)max((int)a, (int)b);
  return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b)));
}

// Shared-memory layout (byte offsets from the 1 KB-aligned base). nu users, maxc clause slots per user,
// npad = max(NP, 32) accumulator columns (a 32-column chunk never reads past the per-column tables).
struct TcLay {
  size_t q, qe, xe, x, a, astage, live, thr, ct, cq, cl, cnt, ctl, bytes;
  int xs;
};
// wmax = attribute words staged per tile (highest word any clause reads, + 1)
__host__ __device__ inline TcLay tc_lay(int np, int rowb, int nu, int maxc, int wmax) {
  TcLay l;
  const int npad = np < 32 ? 32 : np;
  l.q = 0;                                                       // NATOM x [NP][SW] queries (TMA)
  l.qe = l.q + (size_t)np * rowb;                                // [npad][32 B] threshold K-step, B side
  l.xe = (l.qe + (size_t)npad * 32 + 1023) / 1024 * 1024;        // [128][32 B] threshold K-step, A side
  l.x = l.xe + 4096;                                             // xs x NATOM x [128][SW] item tiles
  l.astage = (size_t)wmax * 1024 + 128;                          // wmax words x 1 KB + live bits (16 B)
  l.live = (size_t)wmax * 1024;
  size_t rest = (size_t)kTcAStages * l.astage;
  rest += (size_t)nu * 8 + 16 + (size_t)npad * 8 + (size_t)nu * maxc * 16;
  rest += (size_t)nu * 4 + 16;
  rest += sizeof(TcSmemCtl) + 1024;
  const size_t tile = (size_t)kTcRows * rowb;
  const size_t used = l.x + rest;
  l.xs = used >= kTcSmemBudget ? 0 : (int)((kTcSmemBudget - used) / tile);
  if (l.xs > kTcXStagesMax) l.xs = kTcXStagesMax;
  l.a = l.x + (size_t)l.xs * tile;
  l.thr = l.a + (size_t)kTcAStages * l.astage;                   // [nu] u64 threshold keys
  l.ct = (l.thr + (size_t)nu * 8 + 15) / 16 * 16;                // [npad] per-column hot-test threshold
  l.cq = l.ct + (size_t)npad * 4;                                // [npad] per-column score offset
  l.cl = l.cq + (size_t)npad * 4;                                // [nu][maxc] clauses (16 B)
  l.cnt = l.cl + (size_t)nu * maxc * 16;                         // [nu] region fill counters
  l.ctl = (l.cnt + (size_t)nu * 4 + 15) / 16 * 16;
  l.bytes = l.ctl + sizeof(TcSmemCtl) + 1024;                    // + alignment slack
  return l;
}

// 16-bit encodings of the threshold K-step (kind::f16 operands)
template <int DT>
LINR_DEV uint16_t tc_h_one() { return DT == LINR_BF16 ? (uint16_t)0x3F80u : (uint16_t)0x3C00u; }
template <int DT>
LINR_DEV uint16_t tc_h_bits(float x) {   // exact for dtype values (the split halves and their negations)
  if (DT == LINR_BF16) return __bfloat16_as_ushort(__float2bfloat16_rn(x));
  return __half_as_ushort(__float2half_rn(x));
}
template <int DT>
LINR_DEV float tc_h_rd(float x) {
  if (DT == LINR_BF16) return __bfloat162float(__float2bfloat16_rd(x));
  return __half2float(__float2half_rd(x));
}
// Conservative folded threshold t_eff = hi + lo < T: two dtype values rounded down from the f32 value
// just below T (about 16 (bf16) / 22 (f16) significant bits, so the hot band [t_eff, T) is thin).
template <int DT>
LINR_DEV void tc_h_split(float T, float* hi, float* lo) {
  const float x = nextafterf(T, -INFINITY);
  *hi = tc_h_rd<DT>(x);
  *lo = tc_h_rd<DT>(x - *hi);   // x - hi is exact (Sterbenz-range) and >= 0
}

// Does row `arow` of the attribute stage satisfy all clauses of a user? (sCl row of maxc slots;
// empty slots are always-true)
LINR_DEV bool tc_clauses(const uint4* k, int maxc, const unsigned char* ad, int arow) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (c < maxc) {
      const uint4 kr = k[c];
      const uint64_t mask = ((uint64_t)kr.y << 32) | kr.x;
      const uint64_t aw = reinterpret_cast<const uint64_t*>(ad + kr.z * 1024)[arow];
      ok = ok && (((aw & mask) != 0ull) != (kr.w != 0u));
    }
  }
  for (int c = 4; c < maxc; ++c) {
    const uint4 kr = k[c];
    const uint64_t mask = ((uint64_t)kr.y << 32) | kr.x;
    const uint64_t aw = reinterpret_cast<const uint64_t*>(ad + kr.z * 1024)[arow];
    ok = ok && (((aw & mask) != 0ull) != (kr.w != 0u));
  }
  return ok;
}

// Same, with the row's word 0 in a register when it is the only word clauses read (one = true).
LINR_DEV bool tc_clauses_reg(const uint4* k, int maxc, uint64_t w0, bool one, const unsigned char* ad, int arow) {
  if (!one) return tc_clauses(k, maxc, ad, arow);
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (c < maxc) {
      const uint4 kr = k[c];
      const uint64_t mask = ((uint64_t)kr.y << 32) | kr.x;
      ok = ok && (((w0 & mask) != 0ull) != (kr.w != 0u));
    }
  }
  for (int c = 4; c < maxc; ++c) {
    const uint4 kr = k[c];
    const uint64_t mask = ((uint64_t)kr.y << 32) | kr.x;
    ok = ok && (((w0 & mask) != 0ull) != (kr.w != 0u));
  }
  return ok;
}

// One CTA per SM, persistent over its tiles. Warp 0: TMA producer (item tile + attribute/live
// stage per tile, queries once). Warp 1: MMA issuer (NKS K-steps over the tile, plus, for the
// float kinds in the main pass, one extra K-step that adds -t_u to every column of user u so the
// accumulator holds s - t). Warp 2: TMEM allocator. Warps 4..: epilogue.
//
// Sample pass (p.sample_tiles > 0, no thresholds): every passing (row, user) pair of the sampled
// tiles is appended to the per-(user, CTA) regions (thread per row, clauses evaluated per pair).
// Main pass: a row is hot when some column of the chunk reaches its threshold (float: max of the
// folded s - t >= 0; int8: not every s - t negative). Hot rows are staged; the warp then walks
// them, lane j taking column j: exact key >= T_u, clauses, append.
template <int DT, int D, int NP>
__global__ void __launch_bounds__(kTcThreads, 1) tc_scan_kernel(const __grid_constant__ TcParams p) {
  if (p.gate != nullptr && *(volatile const int*)p.gate != p.gate_want) return;   // path not chosen
  using G = TcGeom<DT, D>;
  constexpr bool kInt = DT == LINR_I8;
  constexpr int NEPI = kTcThreads - 128;   // epilogue threads (warps 4..)
  constexpr int NPAD = NP < 32 ? 32 : NP;
  // epilogue chunk width: 32 columns, narrower for small NP so all four column groups get work
  constexpr int CW = NP >= 128 ? 32 : (NP == 64 ? 16 : 8);
  extern __shared__ __align__(1024) unsigned char smem_raw_tc[];
  // 1024-byte alignment for the 128B-swizzled TMA/UMMA tiles; indexing the extern array keeps the
  // pointers in the shared window (LDS/STS rather than generic loads)
  unsigned char* smem = smem_raw_tc + ((1024u - (smem_u32(smem_raw_tc) & 1023u)) & 1023u);
  const TcLay L = tc_lay(NP, G::ROWB, p.nu, p.maxc, p.wmax);
  const int XS = L.xs;
  unsigned char* sQ = smem + L.q;
  unsigned char* sQe = smem + L.qe;
  unsigned char* sXe = smem + L.xe;
  unsigned char* sX = smem + L.x;
  unsigned char* sA = smem + L.a;
  uint64_t* sThr = reinterpret_cast<uint64_t*>(smem + L.thr);
  uint32_t* sCT = reinterpret_cast<uint32_t*>(smem + L.ct);   // hot-test threshold per column (f32 or i32 bits)
  float* sCQ = reinterpret_cast<float*>(smem + L.cq);         // rare path: score = acc + sCQ (folded) / T (int)
  uint4* sCl = reinterpret_cast<uint4*>(smem + L.cl);
  int* sCnt = reinterpret_cast<int*>(smem + L.cnt);
  TcSmemCtl* ctl = reinterpret_cast<TcSmemCtl*>(smem + L.ctl);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t sFreeCols[8];   // main pass (folded): lead columns of users without a threshold
  __shared__ int sChunk[2][4], sChunkDone[2][4];   // dynamic chunk tickets per (accumulator, lane quarter)

  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t ntiles = (hwm + kTcRows - 1) / kTcRows;
  // tile sequence of this CTA: the sample pass takes sample_tiles distinct tiles per CTA spread
  // evenly over the index (every tile once if the index is smaller); the main pass strides.
  const bool spread = p.sample_tiles > 0;          // tile sequence of the sample passes
  const bool sample = spread && !p.sample_thr;      // epilogue: append every passing pair
  const bool fold = !kInt && !sample;
  const int V = p.V;   // 1, 2, 4 or 8
  const int lv = V == 1 ? 0 : (V == 2 ? 1 : (V == 4 ? 2 : 3));
  const int64_t stotal = (int64_t)gridDim.x * p.sample_tiles;
  int64_t nmine;
  if (spread) {
    if (ntiles > stotal) nmine = p.sample_tiles;
    else nmine = max((int64_t)0, min((int64_t)p.sample_tiles, ntiles - (int64_t)blockIdx.x * p.sample_tiles));
  } else {
    nmine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  }
  auto tile_of = [&](int64_t i) -> int64_t {
    if (spread) {
      const int64_t j = (int64_t)blockIdx.x * p.sample_tiles + i;
      return ntiles > stotal ? (j * ntiles) / stotal : j;   // distinct, evenly spread
    }
    return blockIdx.x + i * gridDim.x;
  };

  if (tid == 0) {
    for (int s = 0; s < XS; ++s) {
      mbar_init(&ctl->xfull[s], 1);
      mbar_init(&ctl->xempty[s], 1);   // released by the MMA commit
    }
    for (int s = 0; s < kTcAStages; ++s) {
      mbar_init(&ctl->afull[s], 1);
      mbar_init(&ctl->aempty[s], NEPI / 32);   // released by every epilogue warp
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&ctl->tfull[a], 1);
      mbar_init(&ctl->tempty[a], NEPI);
    }
    mbar_init(&ctl->qbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 8) {
    sFreeCols[tid] = 0u;
    (&sChunk[0][0])[tid] = 0;
    (&sChunkDone[0][0])[tid] = 0;
  }
  for (int u = tid; u < p.nu; u += kTcThreads) {
    sCnt[u] = 0;
    sThr[u] = p.thr ? p.thr[u] : 0ull;
  }
  // clause table [nu][maxc]; missing slots hold an always-true clause (empty mask, reverse)
  for (int idx = tid; idx < p.nu * p.maxc; idx += kTcThreads) {
    const int u = idx / p.maxc, c = idx - u * p.maxc;
    uint4 k = make_uint4(0u, 0u, 0u, 1u);
    if (c < p.ncl[u]) k = *reinterpret_cast<const uint4*>(p.cl + u * 16 + c);
    sCl[idx] = k;
  }
  __syncthreads();
  // per-column thresholds. Folded (float main pass): t_eff = hi + lo < T_u (tc_h_split), the MMA adds
  // -t_eff, the hot test is acc >= 0 and the rare path rebuilds s = acc + t_eff. A user without a
  // threshold (T = 0) gets t_eff = 0 and marks its chunk always-hot. Columns past the users get a
  // huge t_eff (never hot). Int8: i32 threshold ceil(T) clamped to +-2^30 (s - t never overflows).
  for (int c = tid; c < NPAD; c += kTcThreads) {
    const int u = c >> lv;
    const bool real = c < p.nvec;
    const uint64_t T = real ? sThr[u] : 0ull;
    uint32_t ct;
    float cq;
    if (kInt) {
      const float tf = T ? key_score(T) : -INFINITY;
      ct = (uint32_t)(!real ? (1 << 30) : (T ? (int)fmaxf(fminf(ceilf(tf), 1073741824.0f), -1073741824.0f) : -(1 << 30)));
      cq = real ? tf : INFINITY;
    } else if (fold) {
      float hi = 0.0f, lo = 0.0f;
      if (!real) {
        hi = DT == LINR_BF16 ? 3.0e38f : 65504.0f;
      } else if (T && fabsf(key_score(T)) < 16384.0f) {
        tc_h_split<DT>(key_score(T), &hi, &lo);
      } else {   // no threshold (or out of the 16-bit range): t_eff = 0, the column is always hot
        atomicOr(&sFreeCols[c >> 5], 1u << (c & 31));
      }
      ct = __float_as_uint(0.0f);
      cq = hi + lo;   // <= the f32 value below T: a non-hot pair rebuilds to a score < T
      uint16_t* qe = reinterpret_cast<uint16_t*>(sQe) + c * 16 + (((c >> 2) & 1) << 3);
      qe[0] = tc_h_bits<DT>(-hi);
      qe[1] = tc_h_bits<DT>(-lo);
    } else {
      ct = __float_as_uint(!real ? INFINITY : (T ? key_score(T) : -INFINITY));
      cq = 0.0f;
    }
    sCT[c] = ct;
    sCQ[c] = cq;
  }
  if (fold) {
    // threshold K-step operands in the 32-byte swizzle (16-byte chunk h of row r at h ^ ((r >> 2) & 1)):
    // A = [1, 1, 0, ...] for every item row, B = [-hi, -lo, 0, ...] per column (written above)
    for (int i = tid; i < NPAD * 16; i += kTcThreads) {
      const int c = i >> 4, e = (i & 15) - (((c >> 2) & 1) << 3);   // logical element of the slot
      if (e != 0 && e != 1) reinterpret_cast<uint16_t*>(sQe)[i] = 0;
    }
    for (int i = tid; i < kTcRows * 16; i += kTcThreads) {
      const int r = i >> 4, e = (i & 15) - (((r >> 2) & 1) << 3);
      reinterpret_cast<uint16_t*>(sXe)[i] = (e == 0 || e == 1) ? tc_h_one<DT>() : (uint16_t)0;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
  }
  // two accumulators of NP columns; a 32-column chunk load of the second stays inside (NP = 16: 64)
  constexpr uint32_t kCols = (2 * NP) <= 64 ? 64 : ((2 * NP) <= 128 ? 128 : ((2 * NP) <= 256 ? 256 : 512));
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&ctl->tmem_base)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_base;

  if (warp == 0) {
    if (lane == 0 && nmine > 0) {
      // queries once: NATOM boxes of [NP rows x SW bytes]
      mbar_expect_tx(&ctl->qbar, (uint32_t)(NP * G::ROWB));
      for (int a = 0; a < G::NATOM; ++a) tma_load_2d(sQ + (size_t)a * NP * G::SW, &p.tmq, a * G::SW, 0, &ctl->qbar);
      const uint32_t abytes = (uint32_t)p.wmax * 1024u + 16u;
      int xs = 0;
      uint32_t xph = 0;
      for (int64_t i = 0; i < nmine; ++i) {
        const int64_t t = tile_of(i);
        const int as = (int)(i % kTcAStages);
        const uint32_t aph = (uint32_t)((i / kTcAStages) & 1);
        mbar_wait(&ctl->xempty[xs], xph ^ 1u);
        unsigned char* xd = sX + (size_t)xs * G::XBYTES;
        mbar_expect_tx(&ctl->xfull[xs], (uint32_t)G::XBYTES);
        for (int a = 0; a < G::NATOM; ++a)
          tma_load_2d(xd + (size_t)a * kTcRows * G::SW, &p.tmx, a * G::SW, (int)(t * kTcRows), &ctl->xfull[xs]);
        mbar_wait(&ctl->aempty[as], aph ^ 1u);
        unsigned char* ad = sA + (size_t)as * L.astage;
        mbar_expect_tx(&ctl->afull[as], abytes);
        for (int w = 0; w < p.wmax; ++w)
          bulk_load(ad + w * 1024, p.attr + (size_t)w * p.cap_pad + t * kTcRows, 1024u, &ctl->afull[as]);
        bulk_load(ad + L.live, p.live + t * (kTcRows / 32), 16u, &ctl->afull[as]);
        if (++xs == XS) { xs = 0; xph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nmine > 0) {
      constexpr uint32_t idesc = tc_idesc<DT, NP>();
      mbar_wait(&ctl->qbar, 0);
      tc_fence_after();
      const uint32_t q_s = smem_u32(sQ);
      const uint64_t dxe = umma_desc<32>(smem_u32(sXe)), dqe = umma_desc<32>(smem_u32(sQe));
      int xs = 0;
      uint32_t xph = 0;
      for (int64_t i = 0; i < nmine; ++i) {
        const int acc = (int)(i & 1);
        const uint32_t tph = (uint32_t)((i >> 1) & 1);
        mbar_wait(&ctl->tempty[acc], tph ^ 1u);
        mbar_wait(&ctl->xfull[xs], xph);
        tc_fence_after();
        const uint32_t x_s = smem_u32(sX + (size_t)xs * G::XBYTES);
#pragma unroll
        for (int k = 0; k < G::NKS; ++k) {
          const int atom = k / G::KPA, kk = k % G::KPA;
          const uint64_t da = umma_desc<G::SW>(x_s + (uint32_t)(atom * kTcRows * G::SW + kk * G::KSTEP_B));
          const uint64_t db = umma_desc<G::SW>(q_s + (uint32_t)(atom * NP * G::SW + kk * G::KSTEP_B));
          tc_mma<DT>(tmem + (uint32_t)(acc * NP), da, db, idesc, k > 0 ? 1u : 0u);
        }
        if (fold) tc_mma<DT>(tmem + (uint32_t)(acc * NP), dxe, dqe, idesc, 1u);
        tc_commit(&ctl->xempty[xs]);  // item tile reusable once the MMAs have read it
        tc_commit(&ctl->tfull[acc]);  // accumulator ready
        if (++xs == XS) { xs = 0; xph ^= 1u; }
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: thread <-> TMEM lane (item row) (warp % 4) * 32 + lane; the epilogue
    // warpgroups split the accumulator columns in 32-column chunks (each chunk = 32/V users).
    const int row = (warp & 3) * 32 + lane;
    const int grp = (warp - 4) >> 2;
    constexpr int NGRP = NEPI / 128;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int nchunks = (p.nvec + CW - 1) / CW;
    // lead columns of the chunk (a user's first column holds the max over its V columns)
    const int cmode = (p.maxc == 2 && p.wmax == 1) ? 2 : 0;
    constexpr uint32_t kLow = CW == 32 ? 0xffffffffu : ((1u << CW) - 1u);
    const uint32_t lead_mask = kLow & (V == 1 ? 0xffffffffu : (V == 2 ? 0x55555555u : (V == 4 ? 0x11111111u : 0x01010101u)));
    for (int64_t i = 0; i < nmine; ++i) {
      const int64_t t = tile_of(i);
      const int as = (int)(i % kTcAStages);
      const uint32_t aph = (uint32_t)((i / kTcAStages) & 1);
      const int acc = (int)(i & 1);
      const uint32_t tph = (uint32_t)((i >> 1) & 1);
      mbar_wait(&ctl->tfull[acc], tph);
      mbar_wait(&ctl->afull[as], aph);
      tc_fence_after();
      const unsigned char* ad = sA + (size_t)as * L.astage;
      const uint32_t lw = reinterpret_cast<const uint32_t*>(ad + L.live)[row >> 5];
      const bool live = ((lw >> (row & 31)) & 1u) && (t * kTcRows + row < hwm);
      const uint32_t rbase = p.row0 + (uint32_t)(t * kTcRows) + (uint32_t)((warp & 3) * 32);
      const bool aw = p.wmax == 1;   // single attribute word: keep this row's word in registers
      const uint64_t aw0 = p.wmax >= 1 ? reinterpret_cast<const uint64_t*>(ad)[row] : 0ull;
      // chunk order: static (grp, grp + 4, ...) or, with p.dyn, tickets shared by the four warps of
      // this TMEM lane quarter (a warp slowed by hot columns takes fewer chunks)
      const int q4 = warp & 3;
      auto next_chunk = [&](int cur) -> int {
        if (!p.dyn) return cur + NGRP;
        int c = 0;
        if (lane == 0) c = atomicAdd(&sChunk[acc][q4], 1);
        return __shfl_sync(0xffffffffu, c, 0);
      };
      for (int ch = p.dyn ? next_chunk(0) : grp; ch < nchunks; ch = next_chunk(ch)) {
        uint32_t v[CW];
        tmem_ld<CW>(tmem + lane_base + (uint32_t)(acc * NP + ch * CW), v);
        const int c0 = ch * CW;
        if (V > 1) {   // per-user max over its V aligned columns into the user's first column
#pragma unroll
          for (int j = 0; j < CW; j += 2) v[j] = vmax<kInt>(v[j], v[j + 1]);
          if (V >= 4) {
#pragma unroll
            for (int j = 0; j < CW; j += 4) v[j] = vmax<kInt>(v[j], v[j + 2]);
          }
          if (V >= 8) {
#pragma unroll
            for (int j = 0; j < CW; j += 8) v[j] = vmax<kInt>(v[j], v[j + 4]);
          }
        }
        if (sample) {
          // ---- sample pass: thread per row. The clause bits of the chunk's users first, in a
          // rolled loop (one copy of the clause code: the unrolled append loop below stays small
          // enough for the instruction cache), then per user (warp-uniform) the passing rows
          // append with one shared-memory atomic per warp
          uint32_t pmask = 0u;
          if (live) {
            if (cmode == 2) {   // <= 2 clauses on word 0: branch-free test per user
#pragma unroll 1
              for (int j = 0; j < CW; j += V) {
                if (c0 + j >= p.nvec) break;
                const int u = (c0 + j) >> lv;
                const uint4 k0 = sCl[u * 2], k1 = sCl[u * 2 + 1];
                const uint64_t m0 = ((uint64_t)k0.y << 32) | k0.x, m1 = ((uint64_t)k1.y << 32) | k1.x;
                const bool ok = (((aw0 & m0) != 0ull) != (k0.w != 0u)) && (((aw0 & m1) != 0ull) != (k1.w != 0u));
                pmask |= (ok ? 1u : 0u) << j;
              }
            } else {
#pragma unroll 1
              for (int j = 0; j < CW; j += V) {
                if (c0 + j >= p.nvec) break;
                const int u = (c0 + j) >> lv;
                if (tc_clauses_reg(sCl + u * p.maxc, p.maxc, aw0, aw, ad, row)) pmask |= 1u << j;
              }
            }
          }
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            if ((j & (V - 1)) != 0 || c0 + j >= p.nvec) continue;
            const int u = (c0 + j) >> lv;
            const bool ok = (pmask >> j) & 1u;
            const uint32_t m = __ballot_sync(0xffffffffu, ok);
            if (m == 0u) continue;
            const int leader = __ffs(m) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&sCnt[u], __popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (ok) {
              const int pos = base + __popc(m & lanemask_lt());
              const float sj = kInt ? (float)(int)v[j] : __uint_as_float(v[j]);
              if (pos < p.cap) p.buf[((size_t)u * gridDim.x + blockIdx.x) * p.cap + pos] = make_key(sj, rbase + lane);
            }
          }
          continue;
        }
        // ---- main pass: per thread (item row), the mask of the chunk's lead columns whose score
        // reaches the user's threshold, one funnel shift per column: float (folded) -- the sign bit
        // of s - t_eff (acc = +-0 rebuilds to t_eff < T and is rejected below either way); int8 --
        // the sign bit of s - t. Columns past the users never reach theirs.
        // four independent 8-column chains (bit j of chain g = column 8g + j), then combined
        uint32_t nq[4] = {0u, 0u, 0u, 0u};
        if (kInt) {
          const uint4* ct4 = reinterpret_cast<const uint4*>(sCT + c0);
#pragma unroll
          for (int j4 = CW / 4 - 1; j4 >= 0; --j4) {
            const uint4 t4 = ct4[j4];
            uint32_t& n = nq[(4 * j4) >> 3];
            n = __funnelshift_l((uint32_t)((int)v[4 * j4 + 3] - (int)t4.w), n, 1);
            n = __funnelshift_l((uint32_t)((int)v[4 * j4 + 2] - (int)t4.z), n, 1);
            n = __funnelshift_l((uint32_t)((int)v[4 * j4 + 1] - (int)t4.y), n, 1);
            n = __funnelshift_l((uint32_t)((int)v[4 * j4] - (int)t4.x), n, 1);
          }
        } else {
#pragma unroll
          for (int j = CW - 1; j >= 0; --j) nq[j >> 3] = __funnelshift_l(v[j], nq[j >> 3], 1);
        }
        const uint32_t neg = nq[0] | (nq[1] << 8) | (nq[2] << 16) | (nq[3] << 24);
        uint32_t hm = ~neg & lead_mask;
        if (fold) hm |= (sFreeCols[c0 >> 5] >> (c0 & 31)) & lead_mask;   // users without a threshold
        hm = live ? hm : 0u;
        uint32_t cols = __reduce_or_sync(0xffffffffu, hm);
        // rare: every hot lead column of the warp's 32 rows, one at a time (warp-uniform): re-read the
        // column (the user's V columns, maxed) from TMEM; the rows where it is hot rebuild the exact
        // key, check it against T_u and the user's clauses (row's word 0 in a register), append.
        while (cols) {
          const int j = __ffs(cols) - 1;
          cols &= cols - 1u;
          const int cj = c0 + j;
          const int uj = cj >> lv;
          // the user's clauses first (the row's attribute word is in a register): most hot pairs
          // fail them (the hot test is on unfiltered scores), and then the column is not re-read
          bool cand = ((hm >> j) & 1u) != 0u;
          if (cmode == 2) {   // common case: <= 2 clauses on word 0 (missing slots are always-true)
            const uint4 k0 = sCl[uj * 2], k1 = sCl[uj * 2 + 1];
            const uint64_t m0 = ((uint64_t)k0.y << 32) | k0.x, m1 = ((uint64_t)k1.y << 32) | k1.x;
            cand = cand && (((aw0 & m0) != 0ull) != (k0.w != 0u)) && (((aw0 & m1) != 0ull) != (k1.w != 0u));
          } else if (cand) {
            cand = tc_clauses_reg(sCl + uj * p.maxc, p.maxc, aw0, aw, ad, row);
          }
          if (!__any_sync(0xffffffffu, cand)) continue;
          const uint32_t ta = tmem + lane_base + (uint32_t)(acc * NP + cj);
          uint32_t raw;
          if (V == 1) {
            raw = tmem_ld1(ta);
          } else if (V == 2) {
            uint32_t w[2];
            tmem_ld2(ta, w);
            raw = vmax<kInt>(w[0], w[1]);
          } else if (V == 4) {
            uint32_t w[4];
            tmem_ld4(ta, w);
            raw = vmax<kInt>(vmax<kInt>(w[0], w[1]), vmax<kInt>(w[2], w[3]));
          } else {
            uint32_t w[8];
            tmem_ld8(ta, w);
            raw = vmax<kInt>(vmax<kInt>(vmax<kInt>(w[0], w[1]), vmax<kInt>(w[2], w[3])),
                             vmax<kInt>(vmax<kInt>(w[4], w[5]), vmax<kInt>(w[6], w[7])));
          }
          bool ok = false;
          uint64_t key = 0ull;
          if (cand) {
            const float sj = kInt ? (float)(int)raw : __uint_as_float(raw) + sCQ[cj];
            key = make_key(sj, rbase + (uint32_t)lane);
            ok = key >= sThr[uj];
          }
          const uint32_t m = __ballot_sync(0xffffffffu, ok);
          if (m) {
            const int leader = __ffs(m) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&sCnt[uj], __popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            const int pos = base + __popc(m & lanemask_lt());
            if (ok && pos < p.cap) p.buf[((size_t)uj * gridDim.x + blockIdx.x) * p.cap + pos] = key;
          }
        }
      }
      if (p.dyn && lane == 0) {   // the quarter's last warp resets its tickets for tile i + 2
        if (atomicAdd(&sChunkDone[acc][q4], 1) == NGRP - 1) {
          sChunk[acc][q4] = 0;
          sChunkDone[acc][q4] = 0;
        }
      }
      tc_fence_before();
      mbar_arrive(&ctl->tempty[acc]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl->aempty[as]);   // one arrival per epilogue warp
    }
  }
  tc_fence_before();
  __syncthreads();
  for (int u = tid; u < p.nu; u += kTcThreads) p.cnt[(size_t)u * gridDim.x + blockIdx.x] = sCnt[u];
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols) : "memory");
  }
}

// ------------------------------------------------------------------ per-user region gather
// Keys of user u live in grid regions buf[(u*grid + c)*cap + 0..min(cnt[u*grid+c], cap)). Gather at
// most `room` of them into dst (shared memory). Returns the number gathered; *total = all keys
// (including any beyond the region capacity: total > gathered means an overflowed region).
template <int NT>
__device__ int gather_regions(const uint64_t* buf, const int* cnt, int grid, int cap, int u, uint64_t* dst, int room,
                              int* s_n, long long* s_total, long long* total, long long* clamped = nullptr) {
  // all region counts at once (thread per region, grid <= NT), an exclusive scan of the clamped
  // counts, then every thread copies a strided slice of the concatenation: all loads in flight
  // (round 1 walked the regions one warp-atomic at a time: ~20 us of dependent L2 round trips)
  __shared__ int s_off[NT + 1];
  __shared__ int s_wsum[NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { *s_n = 0; *s_total = 0; }
  __syncthreads();
  const int raw = tid < grid ? cnt[(size_t)u * grid + tid] : 0;
  const int m = raw < cap ? raw : cap;
  long long rt = raw;
  for (int o = 16; o; o >>= 1) rt += __shfl_xor_sync(0xffffffffu, rt, o);
  if (lane == 0 && rt) atomicAdd((unsigned long long*)s_total, (unsigned long long)rt);
  int incl = m;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += s_wsum[w];
  s_off[tid] = base + incl - m;
  if (tid == NT - 1) s_off[NT] = base + incl;
  __syncthreads();
  const int n = s_off[grid] < room ? s_off[grid] : room;
  int c = 0;
  for (int i0 = tid; i0 < n; i0 += 8 * NT) {   // eight independent loads in flight per thread
    uint64_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * NT;
      v[k] = 0ull;
      if (i < n) {
        while (s_off[c + 1] <= i) ++c;   // region of concatenated position i (monotone in i)
        v[k] = buf[((size_t)u * grid + c) * cap + (i - s_off[c])];
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i0 + k * NT < n) dst[i0 + k * NT] = v[k];
  }
  __syncthreads();
  *total = *s_total;
  if (clamped) *clamped = s_off[grid];   // keys present in the regions (each clamped to cap)
  if (tid == 0) *s_n = n;
  return n;
}

// ------------------------------------------------------------------ thresholds from the sample
constexpr int kTcGatherCap = 16384;
// finalize: a user's main-pass keys (>= T_u). ~2-5K on 10M-row shards, but the threshold loosens as
// the sample fraction shrinks (100M rows: ~6K +- a lot), and a user past the cap is recomputed
// exactly by the fallback (100M int8 B = 256 with 8192: 774 ms per step); 16384 keys (160 KB)
constexpr int kTcFinCap = 16384;
constexpr double kTcSigma = 4.0;
__global__ void __launch_bounds__(512, 1) tc_threshold_kernel(const uint64_t* sbuf, const int* scnt, int scap,
                                                              int grid, int nu, int K, int sample_items,
                                                              const DevHeader* hdr, uint64_t* thr,
                                                              const uint64_t* floor) {
  extern __shared__ __align__(16) unsigned char tsm[];
  SelScratch* sc = reinterpret_cast<SelScratch*>(tsm);
  int* s_n = reinterpret_cast<int*>(sc + 1);
  long long* s_total = reinterpret_cast<long long*>(s_n + 2);
  uint64_t* keys = reinterpret_cast<uint64_t*>(tsm + ((sizeof(SelScratch) + 32 + 15) & ~size_t(15)));
  const int u = blockIdx.x;
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&hdr->hwm);
  long long total = 0;
  // regions (and the gather) keep the first passers in row order: a subset of the sample whose
  // size fraction n/total scales the expected count of global top-K keys it holds
  const int n = gather_regions<512>(sbuf, scnt, grid, scap, u, keys, kTcGatherCap, s_n, s_total, &total);
  double frac = hwm > 0 ? (double)sample_items / (double)hwm : 1.0;
  frac = frac < 1.0 ? frac : 1.0;
  if (total > n && total > 0) frac *= (double)n / (double)total;
  // lam = expected sample keys among the global top K; r sits kTcSigma deviations above it, so the
  // r-th sample key is below the global K-th key except with a small probability (caught exactly by
  // the finalisation's certification, which sends the user to the exact GEMV path)
  const double lam = (double)K * frac;
  const int r = (int)ceil(lam + kTcSigma * sqrt(lam) + 3.0);
  // floor (second-stage sample): the keys were collected at >= floor[u], so the r-th of them is
  // >= floor[u]; with fewer than r of them the first-stage threshold stands
  const uint64_t F = floor ? floor[u] : 0ull;
  uint64_t T = F;
  if (n >= r) T = block_select_ge<512>([keys](int i) { return keys[i]; }, n, r, sc);
  if (threadIdx.x == 0) thr[u] = T > F ? T : F;
}

// ------------------------------------------------------------------ per-user finalisation
struct FinSmem {
  SelScratch sel;
  BucketScratch bs;
  int n;
  long long total;
};
__global__ void __launch_bounds__(512, 1) tc_finalize_kernel(const uint64_t* buf, const int* cnt, int cap, int grid,
                                                             const uint64_t* thr, int K, int64_t* out_ids,
                                                             float* out_scores, uint64_t* out_keys, int* flags,
                                                             unsigned int* fb_bar, int room, const int* gate) {
  if (gate != nullptr && *(volatile const int*)gate != 1) return;   // union path chosen instead
  extern __shared__ __align__(16) unsigned char fsm[];
  FinSmem* f = reinterpret_cast<FinSmem*>(fsm);
  uint64_t* s = reinterpret_cast<uint64_t*>(fsm + ((sizeof(FinSmem) + 15) & ~size_t(15)));
  uint64_t* s2 = s + kTcFinCap;   // 4096 keys
  const int u = blockIdx.x, tid = threadIdx.x;
  if (u == 0 && tid == 0) *fb_bar = 0u;   // the fallback kernel's grid barrier starts from zero
  long long total = 0, present = 0;
  int n = gather_regions<512>(buf, cnt, grid, cap, u, s, room, &f->n, &f->total, &total, &present);
  // a region that overflowed lost keys: flagged, recomputed exactly by the fallback
  const bool overflow = total > present;
  if (!overflow && present > n) {
    // every key is in the regions but more than fit in shared memory (a loose threshold on a large
    // shard): the exact K-th largest straight from the regions in global memory (zero padding
    // sorts below every key), then the K keys >= it (keys are distinct) -- no fallback needed
    auto get = [=](int i) -> uint64_t {
      const int c = i / cap, j = i - c * cap;
      const int m = min(cnt[(size_t)u * grid + c], cap);
      return j < m ? buf[((size_t)u * grid + c) * cap + j] : 0ull;
    };
    const uint64_t TK = block_select_ge<512>(get, grid * cap, K, &f->sel);
    if (tid == 0) f->n = 0;
    __syncthreads();
    for (int i = tid; i < grid * cap; i += 512) {
      const uint64_t v = get(i);
      if (v != 0ull && v >= TK) s[atomicAdd(&f->n, 1)] = v;
    }
    __syncthreads();
    n = f->n < kTcFinCap ? f->n : kTcFinCap;
  }
  if (n > K) {
    const uint64_t T = block_select_ge<512>([s](int i) { return s[i]; }, n, K, &f->sel);
    n = block_compact_ge<512>(s, n, T, &f->sel);
  }
  const uint64_t* sorted = s2;
  if (!block_bucket_sort_desc<512>(s, n, s2, &f->bs)) {
    const int P2 = next_pow2(n > 64 ? n : 64);
    for (int i = n + tid; i < P2; i += 512) s[i] = 0ull;
    __syncthreads();
    block_sort_desc<512>(s, P2);
    sorted = s;
  }
  for (int j = tid; j < K; j += 512) {
    const int64_t at = (int64_t)u * K + j;
    if (out_keys) {
      out_keys[at] = j < n ? sorted[j] : 0ull;
    } else if (j < n) {
      out_ids[at] = key_id(sorted[j]);
      out_scores[at] = key_score(sorted[j]);
    } else {
      out_ids[at] = -1;
      out_scores[at] = -INFINITY;
    }
  }
  if (tid == 0) flags[u] = (overflow || (thr[u] != 0ull && n < K)) ? 1 : 0;
}

// ------------------------------------------------------------------ pass counts (batched path, on request)
// One warp per 32-item group: each attribute word and liveness word is read once, then per user
// (warp-uniform) the ballot of the clause predicates; user u's running count lives in lane u % 32
// (register block u / 32), so the attribute stream is read once for all users.
__global__ void __launch_bounds__(256) tc_count_kernel(const uint64_t* attr, int64_t cap_pad, const uint32_t* live,
                                                       const DevHeader* hdr, const KClause* cl, const int* ncl,
                                                       int nu, unsigned long long* counts) {
  const int lane = threadIdx.x & 31;
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&hdr->hwm);
  const int64_t ngroups = (hwm + 31) / 32;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int kBlk = 8;   // nu <= 256 users
  unsigned long long tot[kBlk];
#pragma unroll
  for (int b = 0; b < kBlk; ++b) tot[b] = 0ull;
  for (int64_t g = gw; g < ngroups; g += nw) {
    const int64_t i = g * 32 + lane;
    const bool lv = (live[g] >> lane) & 1u;
    uint64_t aw[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) aw[w] = 0ull;
    aw[0] = attr[i];
#pragma unroll
    for (int b = 0; b < kBlk; ++b) {
      if (b * 32 >= nu) break;
      for (int j = 0; j < 32 && b * 32 + j < nu; ++j) {
        const int u = b * 32 + j;
        bool ok = lv;
        for (int c = 0; c < ncl[u]; ++c) {
          const KClause k = cl[u * 16 + c];
          const uint64_t a = k.word == 0 ? aw[0] : attr[(size_t)k.word * cap_pad + i];
          if (((a & k.mask) != 0ull) == (k.rev != 0)) ok = false;
        }
        const unsigned long long c = (unsigned long long)__popc(__ballot_sync(0xffffffffu, ok));
        if (lane == j) tot[b] += c;
      }
    }
  }
#pragma unroll
  for (int b = 0; b < kBlk; ++b)
    if (b * 32 + lane < nu && tot[b]) atomicAdd(&counts[b * 32 + lane], tot[b]);
}

cudaError_t launch_tc_count(const uint64_t* attr, int64_t cap_pad, const uint32_t* live, const DevHeader* hdr,
                            const KClause* cl, const int* ncl, int nu, unsigned long long* counts, int grid,
                            cudaStream_t st) {
  tc_count_kernel<<<grid, 256, 0, st>>>(attr, cap_pad, live, hdr, cl, ncl, nu, counts);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

bool tc_encode_map(CUtensorMap* m, const void* base, int64_t rows, int rowbytes, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const int sw = rowbytes >= 128 ? 128 : rowbytes;
  cuuint64_t dims[2] = {(cuuint64_t)rowbytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)rowbytes};
  cuuint32_t box[2] = {(cuuint32_t)sw, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle swz = sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                           : (sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int DT, int D, int NP>
static cudaError_t launch_tc_np(const TcParams& p, int grid, cudaStream_t st) {
  const size_t smem = tc_lay(NP, TcGeom<DT, D>::ROWB, p.nu, p.maxc, p.wmax).bytes;
  auto k = tc_scan_kernel<DT, D, NP>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) {
    set_error_detail("tc_scan_kernel smem " + std::to_string(smem));
    return e;
  }
  k<<<grid, kTcThreads, smem, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) set_error_detail("tc_scan_kernel launch, smem " + std::to_string(smem));
  return e;
}

template <int DT, int D>
static cudaError_t launch_tc_d(int np, const TcParams& p, int grid, cudaStream_t st) {
  switch (np) {
    case 16: return launch_tc_np<DT, D, 16>(p, grid, st);
    case 32: return launch_tc_np<DT, D, 32>(p, grid, st);
    case 64: return launch_tc_np<DT, D, 64>(p, grid, st);
    case 128: return launch_tc_np<DT, D, 128>(p, grid, st);
    case 256: return launch_tc_np<DT, D, 256>(p, grid, st);
  }
  return cudaErrorInvalidValue;
}

bool tc_supported(int dtype, int dim, int nvec, int V) {
  if (nvec < 1 || nvec > 256) return false;
  if (V != 1 && V != 2 && V != 4 && V != 8) return false;   // a user's columns stay inside a 32-column chunk
  if (dtype == LINR_BF16 || dtype == LINR_F16) return dim == 64 || dim == 128;
  if (dtype == LINR_I8) return dim == 64 || dim == 128;
  return false;
}
int tc_np(int nvec) {
  int np = 16;
  while (np < nvec) np <<= 1;
  return np;
}
size_t tc_smem_bytes(int dtype, int dim, int np, int nu, int maxc, int wmax) {
  const int esz = dtype == LINR_I8 ? 1 : 2;
  const TcLay l = tc_lay(np, dim * esz, nu, maxc, wmax);
  return l.xs >= 2 ? l.bytes : (size_t)-1;   // at least double-buffered item tiles
}

cudaError_t launch_tc_scan(int dtype, int dim, int np, const TcParams& p, int grid, cudaStream_t st) {
  if (dtype == LINR_BF16) return dim == 128 ? launch_tc_d<LINR_BF16, 128>(np, p, grid, st)
                                            : launch_tc_d<LINR_BF16, 64>(np, p, grid, st);
  if (dtype == LINR_F16) return dim == 128 ? launch_tc_d<LINR_F16, 128>(np, p, grid, st)
                                           : launch_tc_d<LINR_F16, 64>(np, p, grid, st);
  if (dtype == LINR_I8) return dim == 128 ? launch_tc_d<LINR_I8, 128>(np, p, grid, st)
                                          : launch_tc_d<LINR_I8, 64>(np, p, grid, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_tc_threshold(const uint64_t* sbuf, const int* scnt, int scap, int grid, int nu, int K,
                                int sample_items, const DevHeader* hdr, uint64_t* thr, cudaStream_t st, const uint64_t* floor) {
  const size_t smem = ((sizeof(SelScratch) + 32 + 15) & ~size_t(15)) + (size_t)kTcGatherCap * 8;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(tc_threshold_kernel), smem);
  if (e != cudaSuccess) return e;
  tc_threshold_kernel<<<nu, 512, smem, st>>>(sbuf, scnt, scap, grid, nu, K, sample_items, hdr, thr, floor);
  return cudaGetLastError();
}

// Device-side choice for small batches (union path): 1 = every user has a sample threshold (the
// dense tcgen05 pass wins), 0 = some user has none (low pass rate: the union scan wins).
// The dense pass tests every (row, user) pair against T_u BEFORE the clauses, so its hot pairs grow
// as 1 / pass rate: it is chosen only when every user has a threshold AND passes >= 1/25 of the
// sampled rows (c2 B = 8: HIGH 11.7 % -> tcgen05 0.44 ms; LOW 0.24 % -> union 0.20 ms).
__global__ void tc_decide_kernel(const uint64_t* thr, const int* scnt, int grid, int64_t sample_rows,
                                 const DevHeader* hdr, int nu, int* gate) {
  const int u = threadIdx.x;
  bool ok = true;
  if (u < nu) {
    long long passed = 0;
    for (int c = 0; c < grid; ++c) passed += scnt[(size_t)u * grid + c];
    const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&hdr->hwm);
    const int64_t rows = sample_rows < hwm ? sample_rows : hwm;
    ok = thr[u] != 0ull && passed * 25 >= rows;
  }
  const int all = __syncthreads_and(ok);
  if (u == 0) *gate = all ? 1 : 0;
}
cudaError_t launch_tc_decide(const uint64_t* thr, const int* scnt, int grid, int64_t sample_rows, const DevHeader* hdr,
                             int nu, int* gate, cudaStream_t st) {
  tc_decide_kernel<<<1, 256, 0, st>>>(thr, scnt, grid, sample_rows, hdr, nu, gate);
  return cudaGetLastError();
}

cudaError_t launch_tc_finalize(const uint64_t* buf, const int* cnt, int cap, int grid, const uint64_t* thr, int nu,
                               int K, int64_t* out_ids, float* out_scores, uint64_t* out_keys, int* flags,
                               unsigned int* fb_bar, cudaStream_t st, const int* gate) {
  const size_t smem = ((sizeof(FinSmem) + 15) & ~size_t(15)) + (size_t)(kTcFinCap + 4096) * 8;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(tc_finalize_kernel), smem);
  if (e != cudaSuccess) return e;
  // LINR_TC_FIN_ROOM (test knob): a smaller gather room forces the exact global-memory selection
  const int room = std::max(K, std::min(kTcFinCap, env_int("LINR_TC_FIN_ROOM", kTcFinCap)));
  tc_finalize_kernel<<<nu, 512, smem, st>>>(buf, cnt, cap, grid, thr, K, out_ids, out_scores, out_keys, flags,
                                            fb_bar, room, gate);
  return cudaGetLastError();
}

}  // namespace linr
