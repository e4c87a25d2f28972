// Row-gather bandwidth micro-benchmark (not part of the library): what does B200 HBM deliver for
// the scan's access pattern -- a dense 8 B/item attribute stream plus 256 B rows of ~11.7% of the
// items, randomly placed? Modes:
//   0 dense LDG.128 stream of the whole row matrix (calibration)
//   1 gather of a precomputed sorted id list (rows only)
//   2 attribute stream only (8 B/item)
//   3 fused: attribute stream -> select -> ballot compaction -> row gather (the scan's shape)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>

constexpr int ROWB = 256;

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint64_t ldg64(const uint64_t* p) {
  uint64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}

__global__ void dense(const unsigned char* x, long long n16, unsigned* sink) {
  const uint4* p = reinterpret_cast<const uint4*>(x);
  unsigned acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ldg_nc(p + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  for (; i < n16; i += stride) { uint4 v = ldg_nc(p + i); acc ^= v.x ^ v.w; }
  if (acc == 0x12345678u) *sink = acc;
}

// U rows in flight per half-warp: one LDG.128 per lane per row (16 lanes x 16 B = 256 B row)
template <int U>
__global__ void gather_list(const unsigned char* x, const uint32_t* ids, long long nids, unsigned* sink) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned acc = 0;
  for (long long b = gw * 2 * U; b < nids; b += nw * 2 * U) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long j = b + 2 * k + half;
      const uint32_t id = j < nids ? __ldg(ids + j) : 0u;
      v[k] = ldg_nc(x + (size_t)id * ROWB + hl * 16);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

// fused: per warp a 256-item tile: attrs (8/lane) -> select -> ballot list in smem -> gather rows
template <int U, bool GATHER, bool CONTIG = false>
__global__ void fused(const unsigned char* x, const uint64_t* attr, long long n, uint64_t mask_lt,
                      unsigned* sink) {
  __shared__ uint16_t lists[32][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* L = lists[warp];
  const int half = lane >> 4, hl = lane & 15;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long ntiles_all = n / 256;
  // CONTIG: each CTA owns a contiguous tile range, its warps interleave inside it
  const long long tb = CONTIG ? ntiles_all * blockIdx.x / gridDim.x : 0;
  const long long ntiles = CONTIG ? ntiles_all * (blockIdx.x + 1) / gridDim.x : ntiles_all;
  const long long tstep = CONTIG ? (blockDim.x >> 5) : nw;
  unsigned acc = 0;
  long long t = CONTIG ? tb + warp : gw;
  uint64_t a[8], na[8];
  if (t < ntiles)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = ldg64(attr + t * 256 + k * 32 + lane);
  for (; t < ntiles; t += tstep) {
    const long long tn = t + tstep;
    if (tn < ntiles)
#pragma unroll
      for (int k = 0; k < 8; ++k) na[k] = ldg64(attr + tn * 256 + k * 32 + lane);
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool s = (a[k] & 0xFF) < mask_lt;
      const unsigned bal = __ballot_sync(0xffffffffu, s);
      if (s) L[cnt + __popc(bal & ((1u << lane) - 1))] = (uint16_t)(k * 32 + lane);
      cnt += __popc(bal);
    }
    __syncwarp();
    if (GATHER) {
      for (int b = 0; b < cnt; b += 2 * U) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int j = b + 2 * k + half;
          const int id = j < cnt ? L[j] : 0;
          v[k] = j < cnt ? ldg_nc(x + (size_t)(t * 256 + id) * ROWB + hl * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
      }
    } else {
      acc += cnt;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = na[k];
  }
  if (acc == 0x12345678u) *sink = acc;
}

__device__ __forceinline__ void cpa16(void* d, const void* s, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(d)),
               "l"(s), "r"(bytes) : "memory");
}
// cp.async ring like the library scan: S stages of 16 rows per warp; LPRC lanes per row
template <int S, int LPRC>
__global__ void fused_cpa(const unsigned char* x, const uint64_t* attr, long long n, uint64_t mask_lt,
                          unsigned* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* L = reinterpret_cast<uint16_t*>(sm) + warp * 256;
  unsigned char* ring = sm + (blockDim.x >> 5) * 512 + warp * S * 4096;
  const long long ntiles_all = n / 256;
  const long long tb = ntiles_all * blockIdx.x / gridDim.x, ntiles = ntiles_all * (blockIdx.x + 1) / gridDim.x;
  const long long tstep = blockDim.x >> 5;
  unsigned acc = 0;
  long long t = tb + warp;
  uint64_t a[8], na[8];
  if (t < ntiles)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = ldg64(attr + t * 256 + k * 32 + lane);
  constexpr int RPS = 32 / LPRC, NRS = 16 / RPS, CPR = 16 / LPRC;
  const int crow = lane / LPRC, cl = lane % LPRC;
  for (; t < ntiles; t += tstep) {
    const long long tn = t + tstep;
    if (tn < ntiles)
#pragma unroll
      for (int k = 0; k < 8; ++k) na[k] = ldg64(attr + tn * 256 + k * 32 + lane);
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool s = (a[k] & 0xFF) < mask_lt;
      const unsigned bal = __ballot_sync(0xffffffffu, s);
      if (s) L[cnt + __popc(bal & ((1u << lane) - 1))] = (uint16_t)(k * 32 + lane);
      cnt += __popc(bal);
    }
    __syncwarp();
    const int ngrp = (cnt + 15) / 16;
    auto issue = [&](int gi) {
      unsigned char* st = ring + (gi % S) * 4096;
#pragma unroll
      for (int rs = 0; rs < NRS; ++rs) {
        const int row = crow + rs * RPS, idx = gi * 16 + row;
        const int e = idx < cnt ? L[idx] : 0;
        const unsigned char* src = x + (size_t)(t * 256 + e) * ROWB;
#pragma unroll
        for (int k = 0; k < CPR; ++k) cpa16(st + row * 256 + (cl + k * LPRC) * 16, src + (cl + k * LPRC) * 16, idx < cnt ? 16 : 0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int gi = 0; gi < S - 1; ++gi) { if (gi < ngrp) issue(gi); else asm volatile("cp.async.commit_group;" ::: "memory"); }
    for (int gi = 0; gi < ngrp; ++gi) {
      if (gi + S - 1 < ngrp) issue(gi + S - 1); else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
      __syncwarp();
      acc ^= *reinterpret_cast<const unsigned*>(ring + (gi % S) * 4096 + lane * 128);
      __syncwarp();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = na[k];
  }
  if (acc == 0x12345678u) *sink = acc;
}

void run_ws_ring(const unsigned char* x, const uint32_t* ids, long long nid, int nsm, unsigned* sink);
static uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main() {
  const long long n = 10000000;
  unsigned char* x;
  uint64_t* attr;
  uint32_t* ids;
  unsigned* sink;
  cudaMalloc(&x, (size_t)n * ROWB);
  cudaMalloc(&attr, (size_t)n * 8);
  cudaMalloc(&ids, (size_t)n * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(x, 1, (size_t)n * ROWB);
  std::vector<uint64_t> ha(n);
  std::vector<uint32_t> hid;
  const uint64_t lt = 30;   // 30/256 = 11.7%
  for (long long i = 0; i < n; ++i) {
    ha[i] = sm64(i);
    if ((ha[i] & 0xFF) < lt) hid.push_back((uint32_t)i);
  }
  cudaMemcpy(attr, ha.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ids, hid.data(), hid.size() * 4, cudaMemcpyHostToDevice);
  const long long nid = (long long)hid.size();
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    const int R = 20;
    for (int i = 0; i < R; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("%-44s %8.1f us  %7.1f GB/s  (%s)\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  const double rows_b = (double)nid * ROWB, attr_b = (double)n * 8;
  printf("selected %lld rows (%.2f%%)\n", nid, 100.0 * nid / n);
  if (getenv("WS_ONLY")) { run_ws_ring(x, ids, nid, nsm, sink); return 0; }
  for (int bpsm : {1, 2, 4})
    for (int nt : {256, 512, 1024}) {
      char nm[64];
      snprintf(nm, 64, "dense grid=%dx%d nt=%d", nsm, bpsm, nt);
      timeit(nm, (double)n * ROWB, [&] { dense<<<nsm * bpsm, nt>>>(x, n * ROWB / 16, sink); });
    }
  for (int nt : {512, 1024}) {
    char nm[64];
    snprintf(nm, 64, "gather_list U=4 nt=%d", nt);
    timeit(nm, rows_b, [&] { gather_list<4><<<nsm, nt>>>(x, ids, nid, sink); });
    snprintf(nm, 64, "gather_list U=8 nt=%d", nt);
    timeit(nm, rows_b, [&] { gather_list<8><<<nsm, nt>>>(x, ids, nid, sink); });
    snprintf(nm, 64, "gather_list U=16 nt=%d", nt);
    timeit(nm, rows_b, [&] { gather_list<16><<<nsm, nt>>>(x, ids, nid, sink); });
  }
  for (int nt : {512, 1024}) {
    char nm[64];
    snprintf(nm, 64, "attr only nt=%d", nt);
    timeit(nm, attr_b, [&] { fused<4, false><<<nsm, nt>>>(x, attr, n, lt, sink); });
    snprintf(nm, 64, "fused U=4 nt=%d", nt);
    timeit(nm, attr_b + rows_b, [&] { fused<4, true><<<nsm, nt>>>(x, attr, n, lt, sink); });
    snprintf(nm, 64, "fused U=8 nt=%d", nt);
    timeit(nm, attr_b + rows_b, [&] { fused<8, true><<<nsm, nt>>>(x, attr, n, lt, sink); });
    snprintf(nm, 64, "fused U=16 nt=%d", nt);
    timeit(nm, attr_b + rows_b, [&] { fused<16, true><<<nsm, nt>>>(x, attr, n, lt, sink); });
  }
  for (int nt : {512, 1024}) {
    char nm[64];
    snprintf(nm, 64, "fused CONTIG U=8 nt=%d", nt);
    timeit(nm, attr_b + rows_b, [&] { fused<8, true, true><<<nsm, nt>>>(x, attr, n, lt, sink); });
  }
  {
    auto k2 = fused_cpa<2, 4>; auto k3 = fused_cpa<3, 4>; auto k2b = fused_cpa<2, 16>;
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k2b, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    timeit("cp.async S=2 LPRC=4 nt=512", attr_b + rows_b, [&] { k2<<<nsm, 512, 16 * 512 + 16 * 2 * 4096>>>(x, attr, n, lt, sink); });
    timeit("cp.async S=2 LPRC=16 nt=512", attr_b + rows_b, [&] { k2b<<<nsm, 512, 16 * 512 + 16 * 2 * 4096>>>(x, attr, n, lt, sink); });
    timeit("cp.async S=3 LPRC=4 nt=512", attr_b + rows_b, [&] { k3<<<nsm, 512, 16 * 512 + 16 * 3 * 4096>>>(x, attr, n, lt, sink); });
    timeit("cp.async S=2 LPRC=4 nt=768", attr_b + rows_b, [&] { k2<<<nsm, 768, 24 * 512 + 24 * 2 * 4096>>>(x, attr, n, lt, sink); });
    timeit("cp.async S=2 LPRC=16 nt=768", attr_b + rows_b, [&] { k2b<<<nsm, 768, 24 * 512 + 24 * 2 * 4096>>>(x, attr, n, lt, sink); });
  }
  return 0;
}
// ---------------------------------------------------------------------------------------------
// Warp-specialised ring micro (appended): producers gather 16-row groups of the id list into a
// CTA-wide ring, consumers read each group and release it. MODE 0: cp.async + noinc mbarrier
// arrival; MODE 1: one cp.async.bulk (TMA, 256 B) per row with complete_tx.
__device__ __forceinline__ uint32_t su32b(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool bar_test(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
               : "=r"(ok) : "r"(su32b(b)), "r"(par) : "memory");
  return ok != 0;
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) ws_ring(const unsigned char* x, const uint32_t* ids, long long nids,
                                                  int R, int NPW, unsigned* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int RB = MODE == 1 ? 272 : 256;   // padded row stride for linear TMA writes
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  int* rel = reinterpret_cast<int*>(sm + 8 * 64);
  int* ctl = rel + 64;   // [0] ghead
  unsigned char* ring = sm + 1024;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  if (tid < R) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32b(&full[tid])), "r"(MODE == 1 ? 1 : 33) : "memory");
    rel[tid] = 0;
  }
  if (tid == 0) ctl[0] = 0;
  __syncthreads();
  // this CTA's share of the id list, in groups of 16
  const long long ng_all = (nids + 15) / 16;
  const long long g0 = ng_all * blockIdx.x / gridDim.x, g1 = ng_all * (blockIdx.x + 1) / gridDim.x;
  const int ng = (int)(g1 - g0);
  unsigned acc = 0;
  if (warp < NPW) {
    // row ids of this lane's rows, prefetched one group ahead (MODE 0: rows crow, crow+8; MODE 1: row lane)
    auto ld_ids = [&](int k, uint32_t& i0, uint32_t& i1) {
      const long long gb = (g0 + k) * 16;
      const long long j0 = MODE == 0 ? gb + lane / 4 : gb + (lane & 15), j1 = gb + lane / 4 + 8;
      i0 = (k < ng && j0 < nids) ? __ldg(ids + j0) : 0u;
      i1 = (k < ng && j1 < nids) ? __ldg(ids + j1) : 0u;
    };
    uint32_t ni0, ni1;
    ld_ids(warp, ni0, ni1);
    for (int k = warp; k < ng; k += NPW) {
      const uint32_t ci0 = ni0, ci1 = ni1;
      ld_ids(k + NPW, ni0, ni1);
      int idx = 0;
      if (lane == 0) idx = atomicAdd(&ctl[0], 1);
      idx = __shfl_sync(~0u, idx, 0);
      const int rnd = idx / R, slot = idx - rnd * R;
      if (rnd > 0) {
        while (true) {
          int v;
          asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(su32b(&rel[slot])) : "memory");
          if (v >= rnd) break;
        }
      }
      unsigned char* st = ring + (size_t)slot * 16 * RB;
      const long long gb = (g0 + k) * 16;
      if (MODE == 0) {
        const int crow = lane / 4, cl = lane % 4;
        for (int rs = 0; rs < 2; ++rs) {
          const int row = crow + rs * 8;
          const long long j = gb + row;
          const uint32_t id = rs == 0 ? ci0 : ci1;
          for (int kk = 0; kk < 4; ++kk) {
            const int c = cl + kk * 4;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32b(st + row * 256 + ((c ^ (row & 7)) * 16))),
                         "l"(x + (size_t)id * 256 + c * 16), "r"(j < nids ? 16 : 0) : "memory");
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32b(&full[slot])) : "memory");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32b(&full[slot])) : "memory");
      } else {
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32b(&full[slot])), "r"(16 * 256) : "memory");
        __syncwarp();
        if (lane < 16) {
          const uint32_t id = ci0;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                           su32b(st + lane * RB)), "l"(x + (size_t)id * 256), "r"(su32b(&full[slot])) : "memory");
        }
      }
    }
  } else {
    const int cw = warp - NPW, NCW = NW - NPW;
    for (int idx = cw; idx < ng; idx += NCW) {
      const int rnd = idx / R, slot = idx - rnd * R;
      while (!__all_sync(~0u, bar_test(&full[slot], rnd & 1))) {
      }
      acc ^= *reinterpret_cast<const unsigned*>(ring + (size_t)slot * 16 * RB + (lane & 15) * RB + (lane >> 4) * 128);
      __syncwarp();
      if (lane == 0) asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(su32b(&rel[slot])), "r"(rnd + 1) : "memory");
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

void run_ws_ring(const unsigned char* x, const uint32_t* ids, long long nid, int nsm, unsigned* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto k0 = ws_ring<0>;
  auto k1 = ws_ring<1>;
  cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int R : {16, 24, 32, 48})
      for (int npw : {4, 8, 12}) {
        if (R % (16 - npw)) continue;   // consumer of group g must also own g - R
        const int RB = mode ? 272 : 256;
        const size_t smem = 1024 + (size_t)R * 16 * RB;
        auto go = [&] {
          if (mode == 0) k0<<<nsm, 512, smem>>>(x, ids, nid, R, npw, sink);
          else k1<<<nsm, 512, smem>>>(x, ids, nid, R, npw, sink);
        };
        for (int i = 0; i < 3; ++i) go();
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) go();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 20;
        printf("ws_ring mode=%d R=%d npw=%2d  %8.1f us  %7.1f GB/s (%s)\n", mode, R, npw, ms * 1e3,
               nid * 256.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
}
