// Microbenchmark of candidate CTA-wide select / compact / sort variants (clock64, one CTA).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include "../../paper_2407_13218_b200/csrc/common.cuh"
using namespace linr;

struct Scr {
  int hist[2048];
  int wtot[32];
  int sel_digit, sel_above, sel_cnt, maxb;
  unsigned long long red_and, red_or;
  int cnt;
};

// 11-bit radix select, plain smem atomics, all-warps two-level scan
template <int NT, typename Get>
__device__ uint64_t select11(Get get, int n, int k, Scr* sc) {
  constexpr int NW = NT / 32;
  constexpr int BPW = 2048 / NW;   // bins per warp
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long a = ~0ull, o = 0ull;
  for (int i = tid; i < n; i += NT) { uint64_t v = get(i); a &= v; o |= v; }
  for (int off = 16; off; off >>= 1) { a &= __shfl_xor_sync(~0u, a, off); o |= __shfl_xor_sync(~0u, o, off); }
  if (tid == 0) { sc->red_and = ~0ull; sc->red_or = 0ull; }
  __syncthreads();
  if (lane == 0) { atomicAnd(&sc->red_and, a); atomicOr(&sc->red_or, o); }
  __syncthreads();
  const unsigned long long diff = sc->red_and ^ sc->red_or, orv = sc->red_or;
  if (diff == 0ull) return orv;
  const int hb = 63 - __clzll((long long)diff);
  uint64_t pmask = (hb == 63) ? 0ull : (~0ull << (hb + 1));
  uint64_t prefix = orv & pmask;
  int shift = hb - 10 > 0 ? hb - 10 : 0;
  int kk = k;
  while (true) {
    for (int i = tid; i < 2048; i += NT) sc->hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      const uint64_t v = get(i);
      if ((v & pmask) == prefix) atomicAdd(&sc->hist[(int)((v >> shift) & 2047u)], 1);
    }
    __syncthreads();
    // warp w owns bins [2047 - w*BPW - (BPW-1) .. 2047 - w*BPW] in descending digit order
    int c[BPW / 32], s = 0;
#pragma unroll
    for (int i = 0; i < BPW / 32; ++i) { c[i] = sc->hist[2047 - warp * BPW - lane * (BPW / 32) - i]; s += c[i]; }
    int incl = s;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) { int t = __shfl_up_sync(~0u, incl, off); if (lane >= off) incl += t; }
    if (lane == 31) sc->wtot[warp] = incl;
    __syncthreads();
    int wex = 0;
    for (int w = 0; w < warp; ++w) wex += sc->wtot[w];
    const int excl = wex + incl - s;
    if (excl < kk && kk <= excl + s) {
      int acc = excl;
#pragma unroll
      for (int i = 0; i < BPW / 32; ++i) {
        if (acc + c[i] >= kk) { sc->sel_digit = 2047 - warp * BPW - lane * (BPW / 32) - i; sc->sel_above = acc; sc->sel_cnt = c[i]; break; }
        acc += c[i];
      }
    }
    __syncthreads();
    const int d = sc->sel_digit, above = sc->sel_above, cnt = sc->sel_cnt;
    __syncthreads();
    prefix = (prefix & ~(0x7FFull << shift)) | ((uint64_t)d << shift);
    pmask |= 0x7FFull << shift;
    kk -= above;
    if (cnt == kk || shift == 0) break;
    shift = shift - 11 > 0 ? shift - 11 : 0;
  }
  return prefix;
}

// plain-atomic 8-bit variant (current code without match_any)
template <int NT, typename Get>
__device__ uint64_t select8p(Get get, int n, int k, Scr* sc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long a = ~0ull, o = 0ull;
  for (int i = tid; i < n; i += NT) { uint64_t v = get(i); a &= v; o |= v; }
  for (int off = 16; off; off >>= 1) { a &= __shfl_xor_sync(~0u, a, off); o |= __shfl_xor_sync(~0u, o, off); }
  if (tid == 0) { sc->red_and = ~0ull; sc->red_or = 0ull; }
  __syncthreads();
  if (lane == 0) { atomicAnd(&sc->red_and, a); atomicOr(&sc->red_or, o); }
  __syncthreads();
  const unsigned long long diff = sc->red_and ^ sc->red_or, orv = sc->red_or;
  if (diff == 0ull) return orv;
  const int hb = 63 - __clzll((long long)diff);
  uint64_t pmask = (hb == 63) ? 0ull : (~0ull << (hb + 1));
  uint64_t prefix = orv & pmask;
  int shift = hb - 7 > 0 ? hb - 7 : 0;
  int kk = k;
  while (true) {
    for (int i = tid; i < 256; i += NT) sc->hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      const uint64_t v = get(i);
      if ((v & pmask) == prefix) atomicAdd(&sc->hist[(int)((v >> shift) & 255u)], 1);
    }
    __syncthreads();
    if (warp == 0) {
      int c[8], s = 0;
      for (int i = 0; i < 8; ++i) { c[i] = sc->hist[255 - lane * 8 - i]; s += c[i]; }
      int incl = s;
      for (int off = 1; off < 32; off <<= 1) { int t = __shfl_up_sync(~0u, incl, off); if (lane >= off) incl += t; }
      const int excl = incl - s;
      if (excl < kk && kk <= incl) {
        int acc = excl;
        for (int i = 0; i < 8; ++i) { if (acc + c[i] >= kk) { sc->sel_digit = 255 - lane * 8 - i; sc->sel_above = acc; sc->sel_cnt = c[i]; break; } acc += c[i]; }
      }
    }
    __syncthreads();
    const int d = sc->sel_digit, above = sc->sel_above, cnt = sc->sel_cnt;
    __syncthreads();
    prefix = (prefix & ~(0xFFull << shift)) | ((uint64_t)d << shift);
    pmask |= 0xFFull << shift;
    kk -= above;
    if (cnt == kk || shift == 0) break;
    shift = shift - 8 > 0 ? shift - 8 : 0;
  }
  return prefix;
}

// compaction through registers (order not preserved), n <= 32*NT
template <int NT>
__device__ int compact_reg(uint64_t* buf, int n, uint64_t T, Scr* sc) {
  const int tid = threadIdx.x, lane = tid & 31;
  uint64_t r[32];
  const int per = (n + NT - 1) / NT;
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = (j < per && tid + j * NT < n) ? buf[tid + j * NT] : 0ull;
  if (tid == 0) sc->cnt = 0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (j >= per) break;
    const bool keep = r[j] != 0ull && r[j] >= T && (tid + j * NT < n);
    const uint32_t bal = __ballot_sync(~0u, keep);
    int at = 0;
    if (lane == 0 && bal) at = atomicAdd(&sc->cnt, __popc(bal));
    at = __shfl_sync(~0u, at, 0);
    if (keep) buf[at + __popc(bal & lanemask_lt())] = r[j];
  }
  __syncthreads();
  return sc->cnt;
}

// MSD bucket sort (descending) of s[0..n), n <= 2048, into out; buckets of 11 bits below the
// highest differing bit, then insertion sort per bucket. Returns false if a bucket > 64 keys.
template <int NT>
__device__ bool bucket_sort(const uint64_t* s, int n, uint64_t* out, Scr* sc) {
  constexpr int NW = NT / 32;
  constexpr int BPW = 2048 / NW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long a = ~0ull, o = 0ull;
  for (int i = tid; i < n; i += NT) { uint64_t v = s[i]; a &= v; o |= v; }
  for (int off = 16; off; off >>= 1) { a &= __shfl_xor_sync(~0u, a, off); o |= __shfl_xor_sync(~0u, o, off); }
  if (tid == 0) { sc->red_and = ~0ull; sc->red_or = 0ull; sc->maxb = 0; }
  for (int i = tid; i < 2048; i += NT) sc->hist[i] = 0;
  __syncthreads();
  if (lane == 0) { atomicAnd(&sc->red_and, a); atomicOr(&sc->red_or, o); }
  __syncthreads();
  const unsigned long long diff = sc->red_and ^ sc->red_or;
  const int hb = diff ? 63 - __clzll((long long)diff) : 0;
  const int shift = hb - 10 > 0 ? hb - 10 : 0;
  for (int i = tid; i < n; i += NT) atomicAdd(&sc->hist[(int)((s[i] >> shift) & 2047u)], 1);
  __syncthreads();
  // exclusive offsets in descending digit order, written back into hist as cursors
  int c[BPW / 32], sum = 0;
#pragma unroll
  for (int i = 0; i < BPW / 32; ++i) { c[i] = sc->hist[2047 - warp * BPW - lane * (BPW / 32) - i]; sum += c[i]; }
  int incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) { int t = __shfl_up_sync(~0u, incl, off); if (lane >= off) incl += t; }
  if (lane == 31) sc->wtot[warp] = incl;
  __syncthreads();
  int wex = 0;
  for (int w = 0; w < warp; ++w) wex += sc->wtot[w];
  int acc = wex + incl - sum, mx = 0;
#pragma unroll
  for (int i = 0; i < BPW / 32; ++i) { sc->hist[2047 - warp * BPW - lane * (BPW / 32) - i] = acc; acc += c[i]; mx = max(mx, c[i]); }
  for (int off = 16; off; off >>= 1) mx = max(mx, __shfl_xor_sync(~0u, mx, off));
  if (lane == 0) atomicMax(&sc->maxb, mx);
  __syncthreads();
  if (sc->maxb > 64) return false;
  for (int i = tid; i < n; i += NT) {
    const uint64_t v = s[i];
    const int pos = atomicAdd(&sc->hist[(int)((v >> shift) & 2047u)], 1);
    out[pos] = v;
  }
  __syncthreads();
  // bucket d now spans [hist[d] - cnt_d, hist[d]); bucket start = end of the previous (higher) digit
  for (int d = tid; d < 2048; d += NT) {
    const int end = sc->hist[d];
    const int start = (d == 2047) ? 0 : sc->hist[d + 1];
    for (int i = start + 1; i < end; ++i) {   // insertion sort, descending
      const uint64_t x = out[i];
      int j = i - 1;
      while (j >= start && out[j] < x) { out[j + 1] = out[j]; --j; }
      out[j + 1] = x;
    }
  }
  __syncthreads();
  return true;
}

template <int NT>
__global__ void bench(const uint64_t* in, int n, int k, long long* out, uint64_t* res) {
  extern __shared__ __align__(16) unsigned char sm[];
  Scr* sc = (Scr*)sm;
  uint64_t* s = (uint64_t*)(sm + 16384);
  uint64_t* s2 = s + 16384;
  SelScratch* ss = (SelScratch*)(s2 + 4096);
  for (int i = threadIdx.x; i < n; i += NT) s[i] = in[i];
  __syncthreads();
  long long t0 = clock64();
  uint64_t T1 = block_select_ge<NT>([s](int i) { return s[i]; }, n, k, ss);
  __syncthreads();
  long long t1 = clock64();
  uint64_t T2 = select8p<NT>([s](int i) { return s[i]; }, n, k, sc);
  __syncthreads();
  long long t2 = clock64();
  uint64_t T3 = select11<NT>([s](int i) { return s[i]; }, n, k, sc);
  __syncthreads();
  long long t3 = clock64();
  int m = compact_reg<NT>(s, n, T3, sc);
  long long t4 = clock64();
  bool ok = bucket_sort<NT>(s, m, s2, sc);
  long long t5 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = m; out[6] = (T1 == T2 && T2 == T3) + 2 * ok; }
  for (int i = threadIdx.x; i < m; i += NT) res[i] = s2[i];
}

int main() {
  for (int n : {1500, 4736, 8000, 16000}) {
    int k = 1000;
    std::vector<uint64_t> h(n);
    srand(1);
    for (int i = 0; i < n; ++i) {
      float sc = 0.3f + 0.4f * (rand() / (float)RAND_MAX);
      uint32_t u; memcpy(&u, &sc, 4); u |= 0x80000000u;
      h[i] = ((uint64_t)u << 32) | (0xFFFFFFFFu - (uint32_t)i);
    }
    uint64_t *d, *r; long long* o;
    cudaMalloc(&d, n * 8); cudaMalloc(&r, 16384 * 8); cudaMalloc(&o, 64);
    cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
    size_t smem = 16384 + 16384 * 8 + 4096 * 8 + 2048;
    cudaFuncSetAttribute(bench<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int nt : {512, 1024}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (nt == 1024) bench<1024><<<1, 1024, smem>>>(d, n, k, o, r);
        else bench<512><<<1, 512, smem>>>(d, n, k, o, r);
      }
      long long ho[7]; cudaMemcpy(ho, o, 56, cudaMemcpyDeviceToHost);
      std::vector<uint64_t> hr(k); cudaMemcpy(hr.data(), r, k * 8, cudaMemcpyDeviceToHost);
      std::vector<uint64_t> ref = h; std::sort(ref.begin(), ref.end(), std::greater<uint64_t>());
      bool ok = true; for (int i = 0; i < k; ++i) ok &= (hr[i] == ref[i]);
      printf("n=%5d NT=%4d sel_match %6lld sel8plain %6lld sel11 %6lld compact_reg %6lld bucket_sort %6lld (m=%lld flags=%lld) %s\n", n, nt, ho[0], ho[1], ho[2], ho[3], ho[4], ho[5], ho[6], ok ? "OK" : "WRONG");
    }
  }
  cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
}
