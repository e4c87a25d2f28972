// Short-row gather micro-benchmark (not part of the library): what does a gather of isolated
// 64 B rows (int8 d = 64, the c4 shard) cost in DRAM traffic and time on B200, and does the L2's
// maximum fetch granularity (cudaLimitMaxL2FetchGranularity) change it?
// 125M rows x 64 B = 8 GB; ~11.7 % of the rows, randomly placed, gathered from a sorted id list
// (4 lanes x 16 B per row).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather64 gather64.cu
// run under ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum to see the traffic.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__host__ __device__ inline uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int ROWB, int U>
__global__ void gather(const unsigned char* x, const uint32_t* ids, long long nid, unsigned* sink) {
  constexpr int LPR = ROWB / 16;               // lanes per row
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  constexpr int RPW = 32 / LPR;                // rows per warp instruction
  unsigned acc = 0;
  for (long long base = gw * RPW * U; base < nid; base += nw * RPW * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long r = base + u * RPW + lane / LPR;
      v[u] = r < nid ? ldg_nc(x + (size_t)ids[r] * ROWB + (lane % LPR) * 16) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 125000000;
  const int rowb = argc > 2 ? atoi(argv[2]) : 64;
  unsigned char* x;
  uint32_t* ids;
  unsigned* sink;
  if (cudaMalloc(&x, (size_t)n * rowb) != cudaSuccess) return 1;
  cudaMalloc(&ids, (size_t)n * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(x, 1, (size_t)n * rowb);
  std::vector<uint32_t> hid;
  for (long long i = 0; i < n; ++i)
    if ((sm64(i) & 0xFF) < 30) hid.push_back((uint32_t)i);
  cudaMemcpy(ids, hid.data(), hid.size() * 4, cudaMemcpyHostToDevice);
  const long long nid = (long long)hid.size();
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  size_t g0 = 0;
  cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity);
  printf("rows %lld x %d B, selected %lld (%.2f%%), default L2 fetch granularity %zu B\n", n, rowb, nid,
         100.0 * nid / n, g0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int gran : {-1, 32, 64, 128}) {
    if (gran > 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    auto launch = [&] {
      if (rowb == 64) gather<64, 8><<<nsm * 4, 512>>>(x, ids, nid, sink);
      else gather<128, 8><<<nsm * 4, 512>>>(x, ids, nid, sink);
    };
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    const int R = 10;
    for (int i = 0; i < R; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    const double b = (double)nid * rowb;
    printf("granularity %3zu B: %8.1f us  %7.1f GB/s of row bytes  (%s)\n", g, ms * 1e3, b / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
