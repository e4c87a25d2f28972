// Learned similarity scorers in the filtered exhaustive search (§3.3, P:4316-4329;
// SURVEY §8(f) NEXT-4): Hadamard MLP and Mixture-of-Logits with synthetic weights.
//
// Both scorers split into an item-side linear map (query-independent) and a per-query part:
//   Hadamard  s = w2 . ReLU(W1 (h_q (.) h_x) + b1) + b2        with h_x = Wi x + bi
//             = w2 . ReLU(U y + b1) + b2,   y = h_x,  U = W1 diag(h_q)   (h_q = Wm q + bm)
//   MoL       s = sum_k softmax(Wo ReLU(Wgx x + c) + bo)_k <f_k, g_k(x)>,  c = Wgu u + bg
//             y = [g_1(x) .. g_K(x), Wgx x]   (f_k = Fk u per query)
// so the item side y(x) is computed once per row when the scorer is attached and whenever a row
// is loaded or upserted (feature_kernel, stream-ordered like the rows themselves), the query side
// once per search (query_prep_kernel), and the scan (scorer_scan_kernel) reads y for the rows that
// pass the liveness + clause filter and keeps an exact CTA top-K (threshold + radix-select
// compaction); merge_kernel combines the CTAs. fp32 arithmetic throughout.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"

namespace linr {

constexpr int kScNT = 512;
constexpr int kScBuf = 8192;

template <int DT>
LINR_DEV float sc_elem(const void* base, size_t i) {
  if constexpr (DT == LINR_F32) return reinterpret_cast<const float*>(base)[i];
  else if constexpr (DT == LINR_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  else if constexpr (DT == LINR_F16) return __half2float(reinterpret_cast<const __half*>(base)[i]);
  else return (float)reinterpret_cast<const int8_t*>(base)[i];
}

// ------------------------------------------------------------------ item features y(x)
// thread per (row, feature f): y[r][f] = sum_j M[f][j] x[r][j] (+ bias[f] if given)
template <int DT>
__global__ void __launch_bounds__(256) feature_kernel(const void* __restrict__ emb, int dim, int64_t n, int64_t r_begin,
                                                      const int64_t* __restrict__ rows, int64_t grow0, int64_t cap,
                                                      const float* __restrict__ M, const float* __restrict__ bias,
                                                      int F, int Fp, float* y) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * Fp) return;
  const int64_t i = t / Fp;
  const int f = (int)(t - i * Fp);
  int64_t r = r_begin + i;
  if (rows) {
    r = rows[i] - grow0;
    if (r < 0 || r >= cap) return;
  }
  float acc = 0.0f;
  if (f < F) {
    const float* m = M + (size_t)f * dim;
    for (int j = 0; j < dim; ++j) acc = fmaf(__ldg(m + j), sc_elem<DT>(emb, (size_t)r * dim + j), acc);
    if (bias) acc += __ldg(bias + f);
  }
  y[(size_t)r * Fp + f] = acc;
}

cudaError_t launch_features(int dtype, const void* emb, int dim, int64_t n, int64_t r_begin, const int64_t* rows,
                            int64_t grow0, int64_t cap, const float* M, const float* bias, int F, int Fp, float* y,
                            cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((n * Fp + 255) / 256);
  switch (dtype) {
    case LINR_F32: feature_kernel<LINR_F32><<<blocks, 256, 0, st>>>(emb, dim, n, r_begin, rows, grow0, cap, M, bias, F, Fp, y); break;
    case LINR_F16: feature_kernel<LINR_F16><<<blocks, 256, 0, st>>>(emb, dim, n, r_begin, rows, grow0, cap, M, bias, F, Fp, y); break;
    case LINR_BF16: feature_kernel<LINR_BF16><<<blocks, 256, 0, st>>>(emb, dim, n, r_begin, rows, grow0, cap, M, bias, F, Fp, y); break;
    case LINR_I8: feature_kernel<LINR_I8><<<blocks, 256, 0, st>>>(emb, dim, n, r_begin, rows, grow0, cap, M, bias, F, Fp, y); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ query side, one block per user
// Output per user (floats, stride sc_param_floats): Hadamard: U [H][Fp], b1 [H], w2 [H], b2;
// MoL: f [K*dc], c [G], Wo [K][G], bo [K].
template <int DT>
__global__ void __launch_bounds__(256) query_prep_kernel(const __grid_constant__ ScorerDev w, const void* q, int dim,
                                                         float* out, int stride) {
  const int u = blockIdx.x, tid = threadIdx.x;
  __shared__ float sq[1024];
  __shared__ float hq[256];
  for (int j = tid; j < dim; j += 256) sq[j] = sc_elem<DT>(q, (size_t)u * dim + j);
  __syncthreads();
  float* o = out + (size_t)u * stride;
  if (w.kind == 1) {
    for (int f = tid; f < w.F; f += 256) {
      float a = w.bm[f];
      for (int j = 0; j < dim; ++j) a = fmaf(w.Wm[(size_t)f * dim + j], sq[j], a);
      hq[f] = a;
    }
    __syncthreads();
    for (int i = tid; i < w.H * w.Fp; i += 256) {
      const int h = i / w.Fp, f = i - h * w.Fp;
      o[i] = f < w.F ? w.W1[h * w.F + f] * hq[f] : 0.0f;
    }
    for (int h = tid; h < w.H; h += 256) {
      o[w.H * w.Fp + h] = w.b1[h];
      o[w.H * w.Fp + w.H + h] = w.w2[h];
    }
    if (tid == 0) o[w.H * w.Fp + 2 * w.H] = w.b2[0];
  } else {
    const int KD = w.K * w.dc;
    for (int r = tid; r < KD + w.G; r += 256) {
      float a = 0.0f;
      if (r < KD) {
        for (int j = 0; j < dim; ++j) a = fmaf(w.Fk[(size_t)r * dim + j], sq[j], a);
      } else {
        const int h = r - KD;
        a = w.bg[h];
        for (int j = 0; j < dim; ++j) a = fmaf(w.Wgu[(size_t)h * dim + j], sq[j], a);
      }
      o[r] = a;
    }
    for (int i = tid; i < w.K * w.G; i += 256) o[KD + w.G + i] = w.Wo[i];
    for (int k = tid; k < w.K; k += 256) o[KD + w.G + w.K * w.G + k] = w.bo[k];
  }
}

int sc_param_floats(const ScorerDev& w) {
  if (w.kind == 1) return w.H * w.Fp + 2 * w.H + 1;
  return w.K * w.dc + w.G + w.K * w.G + w.K;
}

cudaError_t launch_query_prep(int dtype, const ScorerDev& w, const void* q, int dim, int B, float* out, int stride,
                              cudaStream_t st) {
  switch (dtype) {
    case LINR_F32: query_prep_kernel<LINR_F32><<<B, 256, 0, st>>>(w, q, dim, out, stride); break;
    case LINR_F16: query_prep_kernel<LINR_F16><<<B, 256, 0, st>>>(w, q, dim, out, stride); break;
    case LINR_BF16: query_prep_kernel<LINR_BF16><<<B, 256, 0, st>>>(w, q, dim, out, stride); break;
    case LINR_I8: query_prep_kernel<LINR_I8><<<B, 256, 0, st>>>(w, q, dim, out, stride); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ the scan
struct ScCtl {
  SelScratch sel;
  BucketScratch bs;
  int count;
  unsigned long long thr;
  unsigned int pass;
};
struct ScGet {
  const uint64_t* b;
  __device__ uint64_t operator()(int x) const { return b[x]; }
};

// score of feature row y (Fp floats) under the user's parameters P (shared memory)
template <int KIND>
LINR_DEV float sc_score(const float* __restrict__ y, const float* P, const ScorerDev& w) {
  if constexpr (KIND == 1) {
    const int H = w.H, Fp = w.Fp;
    float s = P[H * Fp + 2 * H];
    for (int h = 0; h < H; ++h) {
      const float* Uh = P + h * Fp;
      float z = P[H * Fp + h];
      for (int f = 0; f < Fp; f += 4) {
        const float4 v = *reinterpret_cast<const float4*>(y + f);
        z = fmaf(Uh[f], v.x, z);
        z = fmaf(Uh[f + 1], v.y, z);
        z = fmaf(Uh[f + 2], v.z, z);
        z = fmaf(Uh[f + 3], v.w, z);
      }
      s = fmaf(P[H * Fp + H + h], fmaxf(z, 0.0f), s);
    }
    return s;
  } else {
    const int K = w.K, dc = w.dc, G = w.G, KD = K * dc;
    float delta[8], lg[8];
    float mx = -INFINITY;
    for (int k = 0; k < K; ++k) {
      float dk = 0.0f;
      for (int c = 0; c < dc; c += 4) {
        const float4 v = *reinterpret_cast<const float4*>(y + k * dc + c);
        dk = fmaf(P[k * dc + c], v.x, dk);
        dk = fmaf(P[k * dc + c + 1], v.y, dk);
        dk = fmaf(P[k * dc + c + 2], v.z, dk);
        dk = fmaf(P[k * dc + c + 3], v.w, dk);
      }
      delta[k] = dk;
      lg[k] = P[KD + G + K * G + k];
    }
    for (int h = 0; h < G; ++h) {
      const float a = fmaxf(y[KD + h] + P[KD + h], 0.0f);
      for (int k = 0; k < K; ++k) lg[k] = fmaf(P[KD + G + k * G + h], a, lg[k]);
    }
    for (int k = 0; k < K; ++k) mx = fmaxf(mx, lg[k]);
    float den = 0.0f, num = 0.0f;
    for (int k = 0; k < K; ++k) {
      const float e = __expf(lg[k] - mx);
      den += e;
      num = fmaf(e, delta[k], num);
    }
    return num / den;
  }
}

template <int KIND>
__global__ void __launch_bounds__(kScNT, 1) scorer_scan_kernel(const __grid_constant__ ScorerScanParams p) {
  extern __shared__ __align__(16) unsigned char ssm[];
  ScCtl* ctl = reinterpret_cast<ScCtl*>(ssm);
  float* P = reinterpret_cast<float*>(ssm + ((sizeof(ScCtl) + 15) & ~size_t(15)));
  uint64_t* buf = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(P) +
                                              (((size_t)p.param_stride * 4 + 15) & ~size_t(15)));
  const int tid = threadIdx.x, lane = tid & 31;
  const int K = p.K;
  const int64_t hwm = (int64_t)(*(volatile const unsigned long long*)&p.hdr->hwm);
  const int64_t lo = hwm * blockIdx.x / gridDim.x, hi = hwm * (blockIdx.x + 1) / gridDim.x;
  for (int u = 0; u < p.nu; ++u) {
    for (int i = tid; i < p.param_stride; i += kScNT) P[i] = p.params[(size_t)u * p.param_stride + i];
    if (tid == 0) { ctl->count = 0; ctl->thr = 0ull; ctl->pass = 0u; }
    __syncthreads();
    const int ncl = p.ncl[u];
    const KClause* cl = p.cl + (size_t)u * 16;
    unsigned int mypass = 0;
    for (int64_t b0 = lo; b0 < hi; b0 += kScNT) {   // uniform trip count within the CTA
      const int64_t i = b0 + tid;
      bool ok = i < hi && ((p.live[i >> 5] >> (i & 31)) & 1u);
      for (int c = 0; c < ncl && ok; ++c) {
        const KClause k = cl[c];
        const bool hit = (p.attr[(size_t)k.word * p.cap_pad + i] & k.mask) != 0ull;
        if (hit == (k.rev != 0u)) ok = false;
      }
      mypass += ok ? 1u : 0u;
      uint64_t key = 0ull;
      if (ok) key = make_key(sc_score<KIND>(p.y + (size_t)i * p.w.Fp, P, p.w), p.row0 + (uint32_t)i);
      const bool c = ok && key >= *(volatile unsigned long long*)&ctl->thr;
      const uint32_t cb = __ballot_sync(0xffffffffu, c);
      if (cb) {
        const int leader = __ffs(cb) - 1;
        int pos0 = 0;
        if (lane == leader) pos0 = atomicAdd(&ctl->count, __popc(cb));
        pos0 = __shfl_sync(0xffffffffu, pos0, leader);
        if (c) buf[pos0 + __popc(cb & lanemask_lt())] = key;
      }
      __syncthreads();
      const int cnt = ctl->count;
      if (cnt > kScBuf) {
        const uint64_t T = block_select_ge<kScNT>(ScGet{buf}, cnt, K, &ctl->sel);
        block_compact_ge<kScNT>(buf, cnt, T, &ctl->sel);
        if (tid == 0) { ctl->count = K; ctl->thr = T; }
        __syncthreads();
      }
    }
    for (int o = 16; o; o >>= 1) mypass += __shfl_xor_sync(0xffffffffu, mypass, o);
    if (lane == 0 && mypass) atomicAdd(&ctl->pass, mypass);
    __syncthreads();
    int cnt = ctl->count;
    if (cnt > K) {
      const uint64_t T = block_select_ge<kScNT>(ScGet{buf}, cnt, K, &ctl->sel);
      cnt = block_compact_ge<kScNT>(buf, cnt, T, &ctl->sel);
    }
    uint64_t* sorted = buf + 2048;
    if (!block_bucket_sort_desc<kScNT>(buf, cnt, sorted, &ctl->bs)) {
      const int P2 = next_pow2(cnt > 64 ? cnt : 64);
      for (int j = cnt + tid; j < P2; j += kScNT) buf[j] = 0ull;
      __syncthreads();
      block_sort_desc<kScNT>(buf, P2);
      sorted = buf;
    }
    uint64_t* out = p.lists + ((size_t)blockIdx.x * p.nu + u) * K;   // [cta][u][K]
    for (int j = tid; j < K; j += kScNT) out[j] = j < cnt ? sorted[j] : 0ull;
    if (tid == 0) p.pass[(size_t)blockIdx.x * p.nu + u] = (int64_t)ctl->pass;
    __syncthreads();
  }
}

size_t scorer_scan_smem(int param_floats) {
  return ((sizeof(ScCtl) + 15) & ~size_t(15)) + (((size_t)param_floats * 4 + 15) & ~size_t(15)) +
         (size_t)(kScBuf + kScNT) * 8;
}

cudaError_t launch_scorer_scan(const ScorerScanParams& p, int grid, cudaStream_t st) {
  const size_t smem = scorer_scan_smem(p.param_stride);
  const void* k = p.w.kind == 1 ? reinterpret_cast<const void*>(scorer_scan_kernel<1>)
                                : reinterpret_cast<const void*>(scorer_scan_kernel<2>);
  cudaError_t e = ensure_smem(k, smem);
  if (e != cudaSuccess) return e;
  if (p.w.kind == 1) scorer_scan_kernel<1><<<grid, kScNT, smem, st>>>(p);
  else scorer_scan_kernel<2><<<grid, kScNT, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace linr
