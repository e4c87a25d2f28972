// Index maintenance kernels: bulk load layout transform, live row update / delete
// (§4.3 "Model Live Update": Upsert/Delete on pre-allocated tensors with a
// high-water mark), and the device-side synthetic data generator (benchmark plumbing that fills
// 1B-row shards in place; same recipe as datagen/ in Python, implemented independently).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"

namespace linr {

// ---------------------------------------------------------------- load / update / delete
__global__ void attr_soa_kernel(const uint64_t* __restrict__ src, int64_t n, int W, uint64_t* __restrict__ dst,
                                int64_t cap_pad, int64_t r0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int w = 0; w < W; ++w) dst[(int64_t)w * cap_pad + r0 + i] = src[i * W + w];
}

__global__ void set_live_range_kernel(uint32_t* live, DevHeader* hdr, int64_t r0, int64_t n) {
  const int64_t w0 = r0 >> 5, w1 = (r0 + n - 1) >> 5;
  const int64_t w = w0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w > w1) return;
  uint32_t m = 0xFFFFFFFFu;
  if (w == w0) m &= 0xFFFFFFFFu << (r0 & 31);
  if (w == w1) m &= 0xFFFFFFFFu >> (31 - ((r0 + n - 1) & 31));
  atomicOr(&live[w], m);
  if (w == w0) atomicMax(&hdr->hwm, (unsigned long long)(r0 + n));
}

// one warp per updated row: copy the row (16-byte chunks), its attribute words, then publish it.
// An id that repeats within one call is written once, by its LAST occurrence (last writer wins:
// the warp of entry i skips if any later entry carries the same id), so a row is never a mix of
// two copies.
__global__ void update_rows_kernel(const int64_t* __restrict__ rows, int64_t n, int64_t grow0, int64_t cap,
                                   int rowbytes, const uint4* __restrict__ emb_src,
                                   const uint64_t* __restrict__ attr_src, int W, uint4* emb, uint64_t* attr,
                                   int64_t cap_pad, uint32_t* live, DevHeader* hdr) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t gid = rows[i];
  const int64_t r = gid - grow0;
  if (r < 0 || r >= cap) {
    if (lane == 0) atomicAdd(&hdr->skipped, 1ull);
    return;
  }
  bool later = false;
  for (int64_t b = i + 1; b < n; b += 32) {   // warp-uniform trip count
    const int64_t j = b + lane;
    later = later || (j < n && rows[j] == gid);
    if (__any_sync(0xffffffffu, later)) return;
  }
  const int ch = rowbytes / 16;
  for (int c = lane; c < ch; c += 32) emb[r * ch + c] = emb_src[i * ch + c];
  if (lane < W) attr[(int64_t)lane * cap_pad + r] = attr_src[i * W + lane];
  __syncwarp();
  if (lane == 0) {
    atomicOr(&live[r >> 5], 1u << (r & 31));
    atomicMax(&hdr->hwm, (unsigned long long)(r + 1));
  }
}

__global__ void delete_rows_kernel(const int64_t* __restrict__ rows, int64_t n, int64_t grow0, int64_t cap,
                                   uint32_t* live, DevHeader* hdr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = rows[i] - grow0;
  if (r < 0 || r >= cap) {
    atomicAdd(&hdr->skipped, 1ull);
    return;
  }
  atomicAnd(&live[r >> 5], ~(1u << (r & 31)));
}

static unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_attr_soa(const uint64_t* src, int64_t n, int W, uint64_t* dst_soa, int64_t cap_pad, int64_t r0,
                            cudaStream_t st) {
  attr_soa_kernel<<<blocks_for(n, 256), 256, 0, st>>>(src, n, W, dst_soa, cap_pad, r0);
  return cudaGetLastError();
}
cudaError_t launch_set_live_range(uint32_t* live, DevHeader* hdr, int64_t r0, int64_t n, cudaStream_t st) {
  const int64_t words = ((r0 + n - 1) >> 5) - (r0 >> 5) + 1;
  set_live_range_kernel<<<blocks_for(words, 256), 256, 0, st>>>(live, hdr, r0, n);
  return cudaGetLastError();
}
cudaError_t launch_update_rows(const int64_t* rows, int64_t n, int64_t grow0, int64_t cap, int rowbytes,
                               const void* emb_src, const uint64_t* attr_src, int W, void* emb, uint64_t* attr,
                               int64_t cap_pad, uint32_t* live, DevHeader* hdr, cudaStream_t st) {
  update_rows_kernel<<<blocks_for(n * 32, 256), 256, 0, st>>>(rows, n, grow0, cap, rowbytes,
                                                              (const uint4*)emb_src, attr_src, W, (uint4*)emb,
                                                              attr, cap_pad, live, hdr);
  return cudaGetLastError();
}
cudaError_t launch_delete_rows(const int64_t* rows, int64_t n, int64_t grow0, int64_t cap, uint32_t* live,
                               DevHeader* hdr, cudaStream_t st) {
  delete_rows_kernel<<<blocks_for(n, 256), 256, 0, st>>>(rows, n, grow0, cap, live, hdr);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- generator
namespace gen {
constexpr uint64_t kG = 0x9E3779B97F4A7C15ull, kM1 = 0xBF58476D1CE4E5B9ull, kM2 = 0x94D049BB133111EBull,
                   kSC = 0xD6E8FEB86659FD93ull;
constexpr uint64_t S_CLUSTER = 1, S_CENTER = 2, S_NOISE = 3, S_ATTR = 4;

__host__ __device__ inline uint64_t sm64(uint64_t z) {
  z += kG;
  z = (z ^ (z >> 30)) * kM1;
  z = (z ^ (z >> 27)) * kM2;
  return z ^ (z >> 31);
}
__device__ inline uint64_t h1(uint64_t base, uint64_t a) { return sm64(base ^ a); }
__device__ inline uint64_t h2(uint64_t base, uint64_t a, uint64_t b) { return sm64(h1(base, a) ^ (b * kG)); }

struct Bases {
  uint64_t cluster, center, noise, attr;
};

__device__ inline int int8_value(const Bases& B, uint64_t row, uint64_t cl, int j) {
  const uint64_t hc = h2(B.center, cl, (uint64_t)(j >> 3));
  const uint64_t hn = h2(B.noise, row, (uint64_t)(j >> 3));
  const int cen = (int)((hc >> (8 * (j & 7))) & 0x7F) - 64;
  const int noi = (int)((hn >> (8 * (j & 7))) & 0x3F) - 32;
  int v = cen + noi;
  return v < -127 ? -127 : (v > 127 ? 127 : v);
}

__device__ inline float dense_value(const Bases& B, uint64_t row, uint64_t cl, int j) {
  const uint64_t hc = h2(B.center, cl, (uint64_t)(j >> 1));
  const uint32_t c24 = (uint32_t)((hc >> (32 * (j & 1))) & 0xFFFFFFull);
  const float c = __fsub_rn(__fmul_rn((float)c24, 5.9604644775390625e-08f), 0.5f);   // 2^-24
  const uint64_t hn = h2(B.noise, row, (uint64_t)(j >> 2));
  const uint32_t n16 = (uint32_t)((hn >> (16 * (j & 3))) & 0xFFFFull);
  const float n = __fsub_rn(__fmul_rn((float)n16, 7.62939453125e-06f), 0.25f);        // 2^-17
  return __fadd_rn(c, n);
}

__device__ inline uint16_t f32_to_bf16_rne(float x) {
  uint32_t u = __float_as_uint(x);
  u = u + 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// one thread per (row, element j)
__global__ void gen_rows_kernel(int dtype, int dim, int W, Bases B, int mode, int64_t row_begin, int64_t n,
                                void* emb, int64_t emb_row_offset, uint64_t* attrs, int64_t attr_stride,
                                bool soa) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = t / dim;
  const int j = (int)(t - i * dim);
  if (i >= n) return;
  const uint64_t row = (uint64_t)(row_begin + i);
  const uint64_t cl = h1(B.cluster, row) & 1023ull;
  if (emb) {
    const int64_t at = (emb_row_offset + i) * dim + j;
    if (dtype == LINR_I8) {
      ((int8_t*)emb)[at] = (int8_t)int8_value(B, row, cl, j);
    } else {
      float x;
      if (mode == 0) x = __fmul_rn((float)int8_value(B, row, cl, j), 0.0078125f);   // k * 2^-7
      else x = dense_value(B, row, cl, j);
      if (dtype == LINR_F32) ((float*)emb)[at] = x;
      else if (dtype == LINR_F16) ((__half*)emb)[at] = __float2half_rn(x);
      else ((uint16_t*)emb)[at] = f32_to_bf16_rne(x);
    }
  }
  if (attrs && j < W) {
    const uint64_t h = h2(B.attr, row, (uint64_t)j);
    uint64_t word;
    if (j == 0) {
      const uint64_t geo = ((h & 0xFFFFull) * 24ull) >> 16;
      const uint64_t com = (((h >> 16) & 0xFFFFull) * 16ull) >> 16;
      const uint64_t tit = (((h >> 32) & 0xFFFFull) * 16ull) >> 16;
      const uint64_t lev = (((h >> 48) & 0xFFFFull) * 8ull) >> 16;
      word = (1ull << geo) | (1ull << (24 + com)) | (1ull << (40 + tit)) | (1ull << (56 + lev));
    } else {
      word = h;
    }
    if (soa) attrs[(int64_t)j * attr_stride + emb_row_offset + i] = word;
    else attrs[i * W + j] = word;
  }
}
}  // namespace gen

cudaError_t launch_generate(int dtype, int dim, int W, uint64_t seed, int mode, int64_t row_begin, int64_t n,
                            void* emb, int64_t emb_row_offset, uint64_t* attrs, int64_t attr_stride_rows,
                            bool attrs_soa, cudaStream_t st) {
  gen::Bases B;
  B.cluster = gen::sm64(seed ^ (gen::S_CLUSTER * gen::kSC));
  B.center = gen::sm64(seed ^ (gen::S_CENTER * gen::kSC));
  B.noise = gen::sm64(seed ^ (gen::S_NOISE * gen::kSC));
  B.attr = gen::sm64(seed ^ (gen::S_ATTR * gen::kSC));
  if (n <= 0) return cudaSuccess;
  const int64_t threads = n * (int64_t)dim;
  gen::gen_rows_kernel<<<blocks_for(threads, 256), 256, 0, st>>>(dtype, dim, W, B, mode, row_begin, n, emb,
                                                                 emb_row_offset, attrs, attr_stride_rows,
                                                                 attrs_soa);
  return cudaGetLastError();
}

}  // namespace linr
