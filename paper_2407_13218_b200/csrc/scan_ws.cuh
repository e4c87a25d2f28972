// Warp-specialised fused pre-filter + score + CTA top-K scan: the GEMV path (B*V <= 8 query
// vectors per launch) for row formats the tensor cores take (bf16/f16 d <= 128, int8 d <= 256).
// Same computation as scan_gemv_kernel (§3.1: clause evaluation fused into
// the scoring pass so filtered rows are never loaded nor ranked, reading R1), organised so that
// HBM latency never sits on a warp's critical path:
//
//   producer warps (NPW): per 256-item tile, liveness + attribute words (prefetched two tiles
//     ahead in registers) -> every user's clauses -> ballot compaction of the passing rows into
//     the warp's pending list. Every 16 pending rows form a *row group*: the warp takes the next
//     slot of a CTA-wide ring (waits for its release), gathers the 16 rows with cp.async (16 B per
//     lane, 64 contiguous bytes per row per instruction, XOR-swizzled for ldmatrix) and arrives on
//     the slot's "full" mbarrier through cp.async.mbarrier.arrive (the arrival lands when the
//     copies do). Groups span tile boundaries, so almost every group is full.
//   consumer warps (NCW): take groups in ring order (group g -> consumer g mod NCW), ldmatrix +
//     mma.sync (m16n8k16 bf16/f16 -> fp32, m16n8k32 int8 -> exact s32) against the query
//     fragments held in registers, max over each user's vectors (reading R12), key, threshold
//     test, warp-aggregated append to the CTA's per-user key buffer; release the slot.
//
// Slot hand-over: "full" is an mbarrier per slot (parity waits are unambiguous because group g and
// g - R belong to the same consumer when R % NCW == 0, so a consumer is never two phases ahead);
// "released" is a monotonic per-slot counter (a producer may hold a group index several rounds
// ahead of a slot's oldest pending use, which a parity wait could not tell apart).
//
// The ring holds up to ~128 KB of rows in flight per SM, independent of how many warps score.
// Buffer compactions (exact radix select of the K-th key) involve only the consumer warps (named
// barrier 1); producers never touch the key buffers. The per-CTA output and the fused merge are
// the same as the per-warp kernel's (scan_tail).
#pragma once
#include <climits>

#include "scan_gemv.cuh"

namespace linr {

constexpr int kWsPcap = 2 * kTileItems + 32;   // pending-row list of a producer warp (<= 2 tiles + a group)

LINR_DEV uint32_t ws_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
LINR_DEV void ws_bar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ws_su32(b)), "r"(count) : "memory");
}
LINR_DEV void ws_bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ws_su32(b)) : "memory");
}
// arrival triggered when every cp.async this thread issued so far has landed (counted in init)
LINR_DEV void ws_cp_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ws_su32(b)) : "memory");
}
LINR_DEV void ws_bar_inval(uint64_t* b) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(ws_su32(b)) : "memory");
}
LINR_DEV int ws_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(ws_su32(p)) : "memory");
  return v;
}
LINR_DEV void ws_st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(ws_su32(p)), "r"(v) : "memory");
}
LINR_DEV bool ws_bar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(ws_su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}

// as ws_bar_test, but the thread may sleep up to ~1 us in the hardware until the phase completes
LINR_DEV bool ws_bar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, 1000;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(ws_su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <int DT, int D>
struct WsGeom {
  using M = MmaGeom<DT, D>;
  static constexpr int NPW = 8;                  // producer warps (filter + gather)
  static constexpr int NCW = 8;                  // consumer warps (score + select)
  static constexpr int NT = 32 * (NPW + NCW);
  // rows per group: 32 for short rows (<= 128 B: the per-group scoring cost is amortised over
  // as many bytes as a 16-row group of 256 B rows), 16 otherwise
  static constexpr int GR = M::ROWB <= 128 ? 32 : 16;
  static constexpr int GSTAGE = GR * M::ROWB;    // bytes of rows per group
  static constexpr int SLOT = GSTAGE + GR * 5 + 16;   // rows + row ids + user masks + barrier + counter
  static constexpr int FIXED = 2048 + NPW * kWsPcap * 5 + 256;
};

// compaction of every user's buffer to its K best keys, by the NTC consumer threads (barrier 1)
template <int NTC>
__device__ __noinline__ void ws_compact(ScanCtl* ctl, uint64_t* bufs, const ScanParams& p, int ctid) {
  part_sync<1, NTC>();
  if (p.dbg != nullptr && ctid == 0) atomicAdd(&p.dbg[blockIdx.x * 8 + 7], 1ull);
  for (int u = 0; u < p.nu; ++u) {
    const int n = min(ctl->count[u], p.bufcap);
    if (n > p.K) {
      uint64_t* b = bufs + (size_t)u * p.bufcap;
      const uint64_t T = block_select_ge<NTC, 1>([b](int i) { return b[i]; }, n, p.K, &ctl->sel, ctid);
      block_compact_ge<NTC, 1>(b, n, T, &ctl->sel, ctid);
      if (ctid == 0) {
        ctl->count[u] = p.K;
        if (T > ctl->thr[u]) ctl->thr[u] = T;
      }
    }
    part_sync<1, NTC>();
  }
  if (ctid == 0) ctl->flag = 0;
  part_sync<1, NTC>();
}

template <int DT, int D, int NQV>
__global__ void __launch_bounds__(WsGeom<DT, D>::NT, 1) scan_ws_kernel(const __grid_constant__ ScanParams p) {
  using M = MmaGeom<DT, D>;
  using W = WsGeom<DT, D>;
  constexpr int NT = W::NT, NPW = W::NPW, NCW = W::NCW, NU = NQV;
  constexpr bool kInt = (DT == LINR_I8);
  using acc_t = typename std::conditional<kInt, int, float>::type;
  if (p.gate != nullptr && *(volatile const int*)p.gate != p.gate_want) return;   // path not chosen
  // programmatic dependent launch: the merge kernel queued behind this scan may be scheduled now
  // (it waits in griddepcontrol.wait for this grid to complete and its writes to be visible)
  asm volatile("griddepcontrol.launch_dependents;");
  static_assert(M::ok, "warp-specialised scan needs a tensor-core row format");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  ScanCtl* ctl = reinterpret_cast<ScanCtl*>(smem_raw);
  uint64_t* bufs = reinterpret_cast<uint64_t*>(smem_raw + 2048);
  unsigned char* cur = smem_raw + 2048 + (size_t)p.nu * p.bufcap * 8;
  uint32_t* plist = reinterpret_cast<uint32_t*>(cur);
  cur += NPW * kWsPcap * 4;
  uint8_t* pmk = cur;
  cur += NPW * kWsPcap;
  const int R = p.ring;                  // a power of two, multiple of NCW
  const int rshift = __ffs(R) - 1;
  uint32_t* mrow = reinterpret_cast<uint32_t*>(cur);
  cur += (size_t)R * W::GR * 4;
  uint8_t* mmask = cur;
  cur += (size_t)R * W::GR;
  uint64_t* fullb = reinterpret_cast<uint64_t*>(cur);
  int* rel = reinterpret_cast<int*>(fullb + R);   // times each slot was released by its consumer
  cur += (size_t)R * 16;
  unsigned char* ring = reinterpret_cast<unsigned char*>(((uintptr_t)cur + 127) & ~(uintptr_t)127);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kMaxUsers) {
    ctl->thr[tid] = (p.init_thr != nullptr && tid < p.nu) ? p.init_thr[tid] : 0ull;
    ctl->count[tid] = 0;
    ctl->pass[tid] = 0u;
  }
  if (tid == 0) {
    ctl->flag = 0; ctl->done = 0; ctl->overflow = 0; ctl->next_tile = 0;
    ctl->ghead = 0; ctl->gtotal = INT_MAX; ctl->pdone = 0; ctl->gcons = 0;
  }
  for (int s = tid; s < R; s += NT) {
    ws_bar_init(&fullb[s], 33);   // 32 cp.async arrivals + the producer's metadata arrival
    rel[s] = 0;
  }
  __syncthreads();
  dbg_mark(p.dbg, blockIdx.x * 8 + 0);

  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t ntiles = (hwm + kTileItems - 1) / kTileItems;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;

  if (warp < NPW) {
    // ================================================================ producer: filter + gather
    uint32_t* prow = plist + warp * kWsPcap;
    uint8_t* pm = pmk + warp * kWsPcap;
    auto grab = [&]() -> int64_t {
      int t = 0;
      if (lane == 0) t = atomicAdd(&ctl->next_tile, 1);
      return t_begin + __shfl_sync(0xffffffffu, t, 0);
    };
    const bool w0 = (p.wmask & 1u) != 0;
    auto prefetch = [&](int64_t tile, uint64_t (&a)[8], uint32_t& lw) {
      const int64_t base = tile * kTileItems;
      lw = (lane < 8) ? ldg_stream_u32(p.live + (base >> 5) + lane) : ~0u;
      if (w0) {
        const uint64_t* ap = p.attr + base + lane;
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] = ldg_stream_u64(ap + t * 32);
      }
    };
    constexpr int LPRC = M::CH < 4 ? M::CH : 4;   // lanes per row in a copy step
    constexpr int RPS = 32 / LPRC;                 // rows per copy step
    constexpr int NRS = W::GR / RPS;               // copy steps per group
    constexpr int CPR = M::CH / LPRC;              // chunks per lane per row
    const int crow = lane / LPRC, cl = lane % LPRC;
    // one row group from pending entries [o, o+n), n <= 16 (rows past n are zero-filled, mask 0)
    auto emit = [&](int o, int n) {
      int idx = 0;
      if (lane == 0) idx = atomicAdd(&ctl->ghead, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      const int rnd = idx >> rshift, slot = idx & (R - 1);
      if (rnd > 0)
        while (ws_ld_acquire(&rel[slot]) < rnd) __nanosleep(32);
      unsigned char* st = ring + (size_t)slot * W::GSTAGE;
#pragma unroll
      for (int rs = 0; rs < NRS; ++rs) {
        const int row = crow + rs * RPS;
        const bool valid = row < n;
        const uint32_t r = valid ? prow[o + row] : 0u;
        const char* src = reinterpret_cast<const char*>(p.emb) + (size_t)r * M::ROWB;
        unsigned char* dst = st + row * M::ROWB;
        const int sw = M::swz(row);
#pragma unroll
        for (int k = 0; k < CPR; ++k) {
          const int c = cl + k * LPRC;
          cp_async16(dst + ((c ^ sw) * 16), src + c * 16, valid ? 16 : 0);
        }
      }
      if (lane < W::GR) {
        mrow[slot * W::GR + lane] = lane < n ? prow[o + lane] : 0u;
        mmask[slot * W::GR + lane] = lane < n ? pm[o + lane] : (uint8_t)0;
      }
      ws_cp_arrive(&fullb[slot]);
      __syncwarp();
      if (lane == 0) ws_bar_arrive(&fullb[slot]);
    };

    uint32_t pcnt[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) pcnt[u] = 0;
    int pc = 0;   // pending rows (warp-uniform)
    // One tile: clauses on its prefetched attribute words, pending-list append, full groups to
    // the ring; then the same registers are refilled with the tile three ahead. Three register
    // sets rotate through an unrolled loop (no register moves, which would wait for the loads).
    // clause evaluation of one attribute word: pass bits of every user for the lane's 8 items
    auto clauses_on = [&](const uint64_t (&aw)[8], uint32_t w, uint32_t (&pb)[NU]) {
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        if (u >= p.nu) continue;
        for (int c = 0; c < p.ncl[u]; ++c) {
          const KClause& k = p.cl[u][c];
          if (k.word != w) continue;
          const unsigned long long m = k.mask;
          const uint32_t rev = k.rev ? 0xFFu : 0u;
          uint32_t hit = 0;
#pragma unroll
          for (int t = 0; t < 8; ++t) hit |= ((aw[t] & m) != 0ull ? 1u : 0u) << t;
          pb[u] &= hit ^ rev;
        }
      }
    };
    const bool only_w0 = p.wmask == 1u;
    // clause evaluation of two tiles' word-0 attributes in one pass over the clause list (two
    // independent dependency chains per clause: twice the ILP of one tile)
    auto clauses_on2 = [&](const uint64_t (&a)[8], const uint64_t (&b)[8], uint32_t (&pa)[NU], uint32_t (&pbb)[NU]) {
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        if (u >= p.nu) continue;
        for (int c = 0; c < p.ncl[u]; ++c) {
          const KClause& k = p.cl[u][c];
          const unsigned long long m = k.mask;
          const uint32_t rev = k.rev ? 0xFFu : 0u;
          uint32_t ha = 0, hb = 0;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            ha |= ((a[t] & m) != 0ull ? 1u : 0u) << t;
            hb |= ((b[t] & m) != 0ull ? 1u : 0u) << t;
          }
          pa[u] &= ha ^ rev;
          pbb[u] &= hb ^ rev;
        }
      }
    };
    auto live_bits = [&](uint32_t lw) -> uint32_t {   // bit t = item base + 32 t + lane
      uint32_t mylive = 0xFFu;
      if (!__all_sync(0xffffffffu, lw == ~0u)) {
        mylive = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) mylive |= ((__shfl_sync(0xffffffffu, lw, t) >> lane) & 1u) << t;
      }
      return mylive;
    };
    auto clauses_generic = [&](const uint64_t (&a)[8], int64_t base, uint32_t (&pb)[NU]) {
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
        clauses_on(aw, (uint32_t)w, pb);
      }
    };
    // Two tiles (A, B with tb > ta): clauses on their prefetched attribute words, refill the
    // registers with the tiles four ahead (four register sets rotate through an unrolled loop:
    // no register moves, which would wait for the loads), one pending-list append for both,
    // full groups to the ring.
    auto step2 = [&](int64_t& ta, uint64_t (&a)[8], uint32_t& la, int64_t& tb, uint64_t (&b)[8],
                     uint32_t& lb) -> bool {
      if (ta >= t_end) return false;
      const bool hasb = tb < t_end;
      const int64_t base_a = ta * kTileItems, base_b = tb * kTileItems;
      const uint32_t live_a = live_bits(la), live_b = hasb ? live_bits(lb) : 0u;
      uint32_t pa[NU], pbb[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        pa[u] = (u < p.nu) ? live_a : 0u;
        pbb[u] = (u < p.nu) ? live_b : 0u;
      }
      if (only_w0) {
        clauses_on2(a, b, pa, pbb);
      } else {
        clauses_generic(a, base_a, pa);
        if (hasb) clauses_generic(b, base_b, pbb);
      }
      // the registers are free: refill them with the tiles four ahead
      ta = grab();
      if (ta < t_end) prefetch(ta, a, la);
      tb = grab();
      if (tb < t_end) prefetch(tb, b, lb);
      // ---- append the passing rows of both tiles (order is irrelevant: keys carry ids)
      uint32_t any = 0;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        any |= pa[u] | (pbb[u] << 8);
        pcnt[u] += __popc(pa[u]) + __popc(pbb[u]);
      }
      const int mine = __popc(any);
      int incl = mine;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      int pos = pc + incl - mine;
      while (any) {
        const int t = __ffs(any) - 1;
        any &= any - 1;
        const bool inb = t >= 8;
        const int tt = t & 7;
        uint32_t um = 0;
#pragma unroll
        for (int u = 0; u < NU; ++u) um |= (((inb ? pbb[u] : pa[u]) >> tt) & 1u) << u;
        prow[pos] = (uint32_t)((inb ? base_b : base_a) + tt * 32 + lane);
        pm[pos] = (uint8_t)um;
        ++pos;
      }
      pc += __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();
      // ---- full groups go to the ring; the remainder (< GR) moves to the front of the list
      int o = 0;
      while (pc - o >= W::GR) {
        emit(o, W::GR);
        o += W::GR;
      }
      if (o > 0) {
        const int n = pc - o;
        uint32_t r = 0;
        uint8_t m = 0;
        if (lane < n) { r = prow[o + lane]; m = pm[o + lane]; }
        __syncwarp();
        if (lane < n) { prow[lane] = r; pm[lane] = m; }
        __syncwarp();
        pc = n;
      }
      return true;
    };
    auto step = [&](int64_t& tile, uint64_t (&a)[8], uint32_t& lw) -> bool {
      if (tile >= t_end) return false;
      const int64_t base = tile * kTileItems;
      // ---- liveness: bit t of mylive = item base + 32 t + lane (fast path: the whole tile live)
      uint32_t mylive = 0xFFu;
      if (!__all_sync(0xffffffffu, lw == ~0u)) {
        mylive = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) mylive |= ((__shfl_sync(0xffffffffu, lw, t) >> lane) & 1u) << t;
      }
      uint32_t pb[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) pb[u] = (u < p.nu) ? mylive : 0u;
      if (only_w0) {
        clauses_on(a, 0u, pb);
      } else if (__any_sync(0xffffffffu, mylive != 0)) {
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
          clauses_on(aw, (uint32_t)w, pb);
        }
      }
      // the registers are free: refill them with the tile three ahead
      tile = grab();
      if (tile < t_end) prefetch(tile, a, lw);
      // ---- append the passing rows to the pending list (order is irrelevant: keys carry ids)
      uint32_t any = 0;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        any |= pb[u];
        pcnt[u] += __popc(pb[u]);
      }
      const int mine = __popc(any);
      int incl = mine;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      int pos = pc + incl - mine;
      while (any) {
        const int t = __ffs(any) - 1;
        any &= any - 1;
        uint32_t um = 0;
#pragma unroll
        for (int u = 0; u < NU; ++u) um |= ((pb[u] >> t) & 1u) << u;
        prow[pos] = (uint32_t)(base + t * 32 + lane);
        pm[pos] = (uint8_t)um;
        ++pos;
      }
      pc += __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();
      // ---- full groups go to the ring; the remainder (< 16) moves to the front of the list
      int o = 0;
      while (pc - o >= W::GR) {
        emit(o, W::GR);
        o += W::GR;
      }
      if (o > 0) {
        const int n = pc - o;
        uint32_t r = 0;
        uint8_t m = 0;
        if (lane < n) { r = prow[o + lane]; m = pm[o + lane]; }
        __syncwarp();
        if (lane < n) { prow[lane] = r; pm[lane] = m; }
        __syncwarp();
        pc = n;
      }
      return true;
    };
    if constexpr (W::GR == 32) {
      // short rows: the producers are the bottleneck (filter per item), two tiles per step
      int64_t t0 = grab(), t1 = grab(), t2 = grab(), t3 = grab();
      uint64_t a0[8], a1[8], a2[8], a3[8];
      uint32_t l0 = ~0u, l1 = ~0u, l2 = ~0u, l3 = ~0u;
      if (t0 < t_end) prefetch(t0, a0, l0);
      if (t1 < t_end) prefetch(t1, a1, l1);
      if (t2 < t_end) prefetch(t2, a2, l2);
      if (t3 < t_end) prefetch(t3, a3, l3);
      while (step2(t0, a0, l0, t1, a1, l1) && step2(t2, a2, l2, t3, a3, l3)) {
      }
    } else {
      int64_t t0 = grab(), t1 = grab(), t2 = grab();
      uint64_t a0[8], a1[8], a2[8];
      uint32_t l0 = ~0u, l1 = ~0u, l2 = ~0u;
      if (t0 < t_end) prefetch(t0, a0, l0);
      if (t1 < t_end) prefetch(t1, a1, l1);
      if (t2 < t_end) prefetch(t2, a2, l2);
      while (step(t0, a0, l0) && step(t1, a1, l1) && step(t2, a2, l2)) {
      }
    }
    if (pc > 0) emit(0, pc);
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      uint32_t c = pcnt[u];
      for (int o2 = 16; o2; o2 >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o2);
      if (lane == 0 && u < p.nu && c) atomicAdd(&ctl->pass[u], c);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const int order = atomicAdd(&ctl->pdone, 1);
      if (p.dbg != nullptr && (order == 0 || order == NPW - 1)) p.dbg[blockIdx.x * 8 + (order == 0 ? 4 : 5)] = gtimer();
      if (order == NPW - 1) {   // every group has been allocated
        const int total = atomicAdd(&ctl->ghead, 0);
        atomicExch(&ctl->gtotal, total);
      }
    }
  } else {
    // ================================================================ consumer: score + select
    const int cw = warp - NPW, ctid = tid - NPW * 32;
    const int nvec = p.nu * p.V;
    const int mg = lane >> 2, mt = lane & 3;
    const int ucol0 = (2 * mt < nvec) ? (2 * mt) / p.V : -1;
    const int ucol1 = (2 * mt + 1 < nvec) ? (2 * mt + 1) / p.V : -1;
    uint32_t bq[M::NKS][2];
    {
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
    }
    const int lrow = lane & 15, lhalf = lane >> 4;
    int slot = cw, rnd = 0;   // group idx = rnd * R + slot (R % NCW == 0)
    for (int idx = cw;; idx += NCW, slot += NCW) {
      if (slot >= R) {
        slot -= R;
        ++rnd;
      }
      bool have = false;
      while (true) {
        if (__all_sync(0xffffffffu, ws_bar_test(&fullb[slot], (uint32_t)rnd & 1u))) { have = true; break; }
        __nanosleep(20);
        int tot = 0;
        if (lane == 0) tot = *(volatile int*)&ctl->gtotal;
        if (idx >= __shfl_sync(0xffffffffu, tot, 0)) break;
        if (scan_flag(ctl, lane)) ws_compact<NCW * 32>(ctl, bufs, p, ctid);
      }
      if (!have) break;
      const unsigned char* st = ring + (size_t)slot * W::GSTAGE;
      const uint32_t st_s = ws_su32(st);
      constexpr int NSUB = W::GR / 16;   // m16 tiles per group
      acc_t accs[NSUB][4];
#pragma unroll
      for (int sb = 0; sb < NSUB; ++sb) {
        // two independent accumulator chains (even / odd k-steps) halve the dependent mma latency
        acc_t acc[4] = {0, 0, 0, 0}, acc2[4] = {0, 0, 0, 0};
        const int row = sb * 16 + lrow;
#pragma unroll
        for (int ks = 0; ks < M::NKS; ++ks) {
          uint32_t af[4];
          const int chunk = ks * 2 + lhalf;
          ldsm_x4(st_s + row * M::ROWB + ((chunk ^ M::swz(row)) * 16), af[0], af[1], af[2], af[3]);
          acc_t (&c)[4] = (ks & 1) ? acc2 : acc;
          if constexpr (kInt) mma32_s8(c, af, bq[ks][0], bq[ks][1]);
          else mma16<DT>(c, af, bq[ks][0], bq[ks][1]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) accs[sb][i] = acc[i] + acc2[i];
      }
      // accumulator of tile sb: [0..1] = row sb*16 + mg, columns 2mt, 2mt+1; [2..3] = row + 8
      if constexpr (NQV == 1) {
        // one user, one vector: column 0 lives in lanes mt == 0; move row r's score to lane r so
        // the group's rows take one threshold test and one append
        const uint32_t ent = lane < W::GR ? (uint32_t)mmask[slot * W::GR + lane] : 0u;
        const uint32_t lr = lane < W::GR ? mrow[slot * W::GR + lane] : 0u;
        __syncwarp();
        if (lane == 0) ws_st_release(&rel[slot], rnd + 1);   // the slot's rows and metadata are consumed
        const int src = (lane & 7) * 4;
        acc_t xv = 0;
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb) {
          const acc_t x0 = __shfl_sync(0xffffffffu, accs[sb][0], src);
          const acc_t x2 = __shfl_sync(0xffffffffu, accs[sb][2], src);
          if ((lane >> 4) == sb) xv = (lane & 8) ? x2 : x0;
        }
        const float v = (float)xv;
        const bool cand = p.nu > 0 && (ent & 1u);
        Appender<NT, NU>::append(ctl, bufs, p, 0, cand, cand ? make_key(v, p.row0 + lr) : 0ull);
        if (scan_flag(ctl, lane)) ws_compact<NCW * 32>(ctl, bufs, p, ctid);
        continue;
      }
      if (NQV > 1 && p.nu == 1) {
        // one user with V > 1 vectors (c5 U = 1): the max over the user's columns (lanes mt = 0..3
        // hold columns 2mt, 2mt+1; columns >= V are padding) by two butterfly shuffles, then the
        // same row transposition as above -- one threshold test and one append per row group
        const uint32_t ent = lane < W::GR ? (uint32_t)mmask[slot * W::GR + lane] : 0u;
        const uint32_t lr = lane < W::GR ? mrow[slot * W::GR + lane] : 0u;
        __syncwarp();
        if (lane == 0) ws_st_release(&rel[slot], rnd + 1);   // the slot's rows and metadata are consumed
        const int src = (lane & 7) * 4;
        const bool ok0 = 2 * mt < p.V, ok1 = 2 * mt + 1 < p.V;
        float xv = -INFINITY;
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb) {
          float m0 = fmaxf(ok0 ? (float)accs[sb][0] : -INFINITY, ok1 ? (float)accs[sb][1] : -INFINITY);
          float m2 = fmaxf(ok0 ? (float)accs[sb][2] : -INFINITY, ok1 ? (float)accs[sb][3] : -INFINITY);
          m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
          m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, 1));
          m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
          m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, 2));
          const float x0 = __shfl_sync(0xffffffffu, m0, src);
          const float x2 = __shfl_sync(0xffffffffu, m2, src);
          if ((lane >> 4) == sb) xv = (lane & 8) ? x2 : x0;
        }
        const bool cand = (ent & 1u) != 0u;
        Appender<NT, NU>::append(ctl, bufs, p, 0, cand, cand ? make_key(xv, p.row0 + lr) : 0ull);
        if (scan_flag(ctl, lane)) ws_compact<NCW * 32>(ctl, bufs, p, ctid);
        continue;
      }
      uint32_t ent[NSUB][2], lr[NSUB][2];
#pragma unroll
      for (int sb = 0; sb < NSUB; ++sb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          ent[sb][h] = mmask[slot * W::GR + sb * 16 + mg + 8 * h];
          lr[sb][h] = mrow[slot * W::GR + sb * 16 + mg + 8 * h];
        }
      __syncwarp();
      if (lane == 0) ws_st_release(&rel[slot], rnd + 1);   // the slot's rows and metadata are consumed
#pragma unroll
      for (int sb = 0; sb < NSUB; ++sb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t gid = p.row0 + lr[sb][h];
        const float v0 = (float)accs[sb][2 * h], v1 = (float)accs[sb][2 * h + 1];
        if (p.V == 1) {
          // one vector per user: this lane's two accumulator columns ARE (row, user) pairs, so
          // each lane tests its own pairs against the users' thresholds; the per-user appends run
          // only when some lane of the warp has a candidate (rare once the thresholds are up)
          const uint64_t k0 = make_key(v0, gid), k1 = make_key(v1, gid);
          const bool c0 = ucol0 >= 0 && ucol0 < p.nu && ((ent[sb][h] >> ucol0) & 1u) &&
                          k0 >= *(volatile const unsigned long long*)&ctl->thr[ucol0];
          const bool c1 = ucol1 >= 0 && ucol1 < p.nu && ((ent[sb][h] >> ucol1) & 1u) &&
                          k1 >= *(volatile const unsigned long long*)&ctl->thr[ucol1];
          if (__any_sync(0xffffffffu, c0 || c1)) {
#pragma unroll 1
            for (int u = 0; u < NU; ++u) {   // rolled: rare path, keep the code small (i-cache)
              if (u >= p.nu) break;
              const bool cand = (c0 && ucol0 == u) || (c1 && ucol1 == u);
              Appender<NT, NU>::append(ctl, bufs, p, u, cand, (c0 && ucol0 == u) ? k0 : k1);
            }
          }
          continue;
        }
#pragma unroll 1
        for (int u = 0; u < NU; ++u) {   // rolled: the unrolled copies overflowed the instruction cache
          if (u >= p.nu) break;   // warp-uniform: one user with V vectors runs one append, not NQV
          float m = -INFINITY;
          if (ucol0 == u) m = v0;
          if (ucol1 == u) m = fmaxf(m, v1);
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
          const bool cand = u < p.nu && mt == 0 && ((ent[sb][h] >> u) & 1u);
          Appender<NT, NU>::append(ctl, bufs, p, u, cand, cand ? make_key(m, gid) : 0ull);
        }
      }
      if (scan_flag(ctl, lane)) ws_compact<NCW * 32>(ctl, bufs, p, ctid);
    }
    // keep joining compactions until every consumer is done
    if (lane == 0) atomicAdd(&ctl->done, 1);
    while (true) {
      if (scan_flag(ctl, lane)) {
        ws_compact<NCW * 32>(ctl, bufs, p, ctid);
        continue;
      }
      int d = 0;
      if (lane == 0) d = *(volatile int*)&ctl->done;
      d = __shfl_sync(0xffffffffu, d, 0);
      if (d == NCW) break;
      __nanosleep(128);
    }
  }
  __syncthreads();
  for (int s = tid; s < R; s += NT) ws_bar_inval(&fullb[s]);   // the tail reuses this memory
  __syncthreads();
  dbg_mark(p.dbg, blockIdx.x * 8 + 1);
  scan_tail<NT>(ctl, bufs, p, ring, smem_raw, (size_t)R * W::GSTAGE);
}

}  // namespace linr
