// Microbenchmark of the CTA-wide primitives in csrc/common.cuh (clock64 per phase, one CTA).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_2407_13218_b200/csrc/common.cuh"
using namespace linr;

template <int NT>
__global__ void bench(const uint64_t* in, int n, int k, long long* out, uint64_t* res) {
  extern __shared__ __align__(16) unsigned char sm[];
  SelScratch* sc = (SelScratch*)sm;
  uint64_t* s = (uint64_t*)(sm + 2048);
  uint64_t* scratch = s + 16384;
  for (int i = threadIdx.x; i < n; i += NT) s[i] = in[i];
  __syncthreads();
  long long t0 = clock64();
  uint64_t T = block_select_ge<NT>([s](int i) { return s[i]; }, n, k, sc);
  __syncthreads();
  long long t1 = clock64();
  int m = block_compact_ge<NT>(s, n, T, sc);
  __syncthreads();
  long long t2 = clock64();
  int P2 = next_pow2(m); if (P2 < 64) P2 = 64;
  for (int i = m + threadIdx.x; i < P2; i += NT) s[i] = 0;
  __syncthreads();
  long long t3 = clock64();
  block_sort_desc_reg<NT>(s, P2, scratch);
  long long t4 = clock64();
  for (int i = m + threadIdx.x; i < P2; i += NT) s[i] = 0;
  __syncthreads();
  long long t5 = clock64();
  block_sort_desc<NT>(s, P2);
  long long t6 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t4 - t3; out[3] = t6 - t5; out[4] = m; }
  for (int i = threadIdx.x; i < P2; i += NT) res[i] = s[i];
}

int main() {
  for (int n : {4736, 8000, 24000}) {
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
    size_t smem = 2048 + 16384 * 8 + 4096 * 8;
    cudaFuncSetAttribute(bench<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int nt : {512, 1024}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (nt == 1024) bench<1024><<<1, 1024, smem>>>(d, n, k, o, r);
        else bench<512><<<1, 512, smem>>>(d, n, k, o, r);
      }
      long long ho[5]; cudaMemcpy(ho, o, 40, cudaMemcpyDeviceToHost);
      std::vector<uint64_t> hr(1024); cudaMemcpy(hr.data(), r, 1024 * 8, cudaMemcpyDeviceToHost);
      std::vector<uint64_t> ref = h; std::sort(ref.begin(), ref.end(), std::greater<uint64_t>());
      bool ok = true; for (int i = 0; i < k; ++i) ok &= (hr[i] == ref[i]);
      printf("n=%d NT=%d select %lld compact %lld sort_reg %lld sort_smem %lld cycles (m=%lld) %s\n", n, nt, ho[0], ho[1], ho[2], ho[3], ho[4], ok ? "OK" : "WRONG");
    }
  }
  cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
}
