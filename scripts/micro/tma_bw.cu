// TMA streaming bandwidth micro-benchmark (not part of the library): how fast can 148 persistent
// CTAs stream a 2.56 GB item matrix into shared memory with a stage ring, per box shape?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}

constexpr int TILE = 32768;
struct Args {
  CUtensorMap tm;
  const unsigned char* base;
  long long ntiles;
  int mode, stages, boxrows;
};

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* buf = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
  __shared__ uint64_t full[8], empty[8];
  const int S = a.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long mine = a.ntiles > blockIdx.x ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    int s = 0; uint32_t ph = 0;
    for (long long i = 0; i < mine; ++i) {
      const long long t = blockIdx.x + i * gridDim.x;
      wait(&empty[s], ph ^ 1u);
      unsigned char* d = buf + (size_t)s * TILE;
      expect_tx(&full[s], TILE);
      if (a.mode == 0 || a.mode == 3) {          // [rows][256 B]: 2 boxes {128 B, 128 rows}
        tma2d(d, &a.tm, 0, (int)(t * 128), &full[s]);
        tma2d(d + 16384, &a.tm, 128, (int)(t * 128), &full[s]);
      } else if (a.mode == 1) {                   // [2*rows][128 B]: boxes {128 B, boxrows} contiguous
        for (int k = 0; k < 256 / a.boxrows; ++k)
          tma2d(d + k * a.boxrows * 128, &a.tm, 0, (int)(t * 256 + k * a.boxrows), &full[s]);
      } else if (a.mode == 2) {                   // plain bulk copy, 32 KB contiguous
        bulk(d, a.base + (size_t)t * TILE, TILE, &full[s]);
      } else if (a.mode == 4) {                   // 4 bulk copies of 8 KB
        for (int k = 0; k < 4; ++k) bulk(d + k * 8192, a.base + (size_t)t * TILE + k * 8192, 8192, &full[s]);
      }
      if (++s == S) { s = 0; ph ^= 1u; }
    }
  } else if (threadIdx.x == 32) {
    int s = 0; uint32_t ph = 0;
    unsigned acc = 0;
    for (long long i = 0; i < mine; ++i) {
      wait(&full[s], ph);
      acc += buf[(size_t)s * TILE + (i & 1023)];
      arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1u; }
    }
    if (acc == 0xFFFFFFFFu) printf("x");
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long rows = 10000000, bytes = rows * 256;
  unsigned char* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * TILE + 1024);
  struct Cfg { int mode, boxrows; CUtensorMapL2promotion prom; const char* name; };
  Cfg cfgs[] = {{0, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "2 boxes {128B,128 rows} stride 256B, promo 256B"},
                {3, 128, CU_TENSOR_MAP_L2_PROMOTION_NONE, "2 boxes {128B,128 rows} stride 256B, promo none"},
                {1, 256, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "1 box {128B,256 rows} contiguous"},
                {1, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "2 boxes {128B,128 rows} contiguous"},
                {2, 0, CU_TENSOR_MAP_L2_PROMOTION_NONE, "bulk 32 KB"},
                {4, 0, CU_TENSOR_MAP_L2_PROMOTION_NONE, "4 x bulk 8 KB"}};
  for (const Cfg& c : cfgs) {
    Args a{};
    a.base = d;
    a.ntiles = bytes / TILE;
    a.mode = c.mode;
    a.boxrows = c.boxrows;
    if (c.mode == 0 || c.mode == 3) {
      cuuint64_t dims[2] = {256, (cuuint64_t)rows}, str[1] = {256};
      cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
      enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, c.prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else if (c.mode == 1) {
      cuuint64_t dims[2] = {128, (cuuint64_t)rows * 2}, str[1] = {128};
      cuuint32_t box[2] = {128, (cuuint32_t)c.boxrows}, es[2] = {1, 1};
      enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, c.prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int S = 4; S <= 6; S += 2) {
      a.stages = S;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      stream<<<sms, 64, S * TILE + 1024>>>(a);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) stream<<<sms, 64, S * TILE + 1024>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-52s stages %d: %.3f ms  %.0f GB/s  (%s)\n", c.name, S, ms / 5, bytes / (ms / 5) / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
