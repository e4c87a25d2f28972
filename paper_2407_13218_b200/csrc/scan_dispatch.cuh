// Per-dtype dispatch of the GEMV-path scan kernels: the warp-specialised tensor-core kernel
// (scan_ws.cuh) where the row format allows it, the per-warp fused kernel (scan_gemv.cuh) otherwise.
#pragma once
#include "scan_gemv.cuh"
#include "scan_ws.cuh"

namespace linr {

template <int DT>
struct ScanDispatch {
  template <int D, int NQV>
  static constexpr int nt() {
    return 512;   // 16 warps x 128 registers: query chunks + next-tile prefetch stay in registers
  }
  template <int D, int NQV>
  static cudaError_t go(const ScanParams& p, int grid, size_t smem, cudaStream_t st) {
    if constexpr (ScanGeom<DT, D, NQV>::kMma) {
      if (p.ring > 0) {   // warp-specialised kernel (the plan sized its ring)
        auto k = scan_ws_kernel<DT, D, NQV>;
        cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
        if (e != cudaSuccess) return e;
        k<<<grid, WsGeom<DT, D>::NT, smem, st>>>(p);
        return cudaGetLastError();
      }
    }
    constexpr int NT = nt<D, NQV>();
    auto k = scan_gemv_kernel<DT, D, NQV, NT>;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
    if (e != cudaSuccess) return e;
    // grid = #SMs at one CTA per SM: every CTA is resident, so the fused merge's wait for the
    // other CTAs of the launch cannot deadlock (CTAs only wait on CTAs of the same launch).
    k<<<grid, NT, smem, st>>>(p);
    return cudaGetLastError();
  }
  template <int D>
  static cudaError_t by_nqv(int nqv, const ScanParams& p, int grid, size_t smem, cudaStream_t st) {
    switch (nqv) {
      case 1: return go<D, 1>(p, grid, smem, st);
      case 2: return go<D, 2>(p, grid, smem, st);
      case 4: return go<D, 4>(p, grid, smem, st);
      case 8: return go<D, 8>(p, grid, smem, st);
    }
    return cudaErrorInvalidValue;
  }
  static cudaError_t launch(int dim, int nqv, const ScanParams& p, int grid, size_t smem, cudaStream_t st) {
    switch (dim) {
      case 16: return by_nqv<16>(nqv, p, grid, smem, st);
      case 32: return by_nqv<32>(nqv, p, grid, smem, st);
      case 64: return by_nqv<64>(nqv, p, grid, smem, st);
      case 128: return by_nqv<128>(nqv, p, grid, smem, st);
      case 256: return by_nqv<256>(nqv, p, grid, smem, st);
      case 512: return by_nqv<512>(nqv, p, grid, smem, st);
      case 1024: return by_nqv<1024>(nqv, p, grid, smem, st);
    }
    return cudaErrorInvalidValue;
  }
  template <int D, int NQV>
  static ScanCfg cfg_dq() {
    using SG = ScanGeom<DT, D, NQV>;
    if constexpr (SG::kMma) {
      using W = WsGeom<DT, D>;
      static_assert(W::NT == nt<D, NQV>(), "both GEMV kernels run 512 threads");
      return ScanCfg{nt<D, NQV>(), SG::RPI, SG::RING, W::SLOT, W::FIXED, W::NCW * W::GR / 16};
    }
    return ScanCfg{nt<D, NQV>(), SG::RPI, SG::RING, 0, 0, 0};
  }
  template <int D>
  static ScanCfg cfg_d(int nqv) {
    switch (nqv) {
      case 1: return cfg_dq<D, 1>();
      case 2: return cfg_dq<D, 2>();
      case 4: return cfg_dq<D, 4>();
      case 8: return cfg_dq<D, 8>();
    }
    return ScanCfg{0, 0, 0};
  }
  static ScanCfg cfg(int dim, int nqv) {
    switch (dim) {
      case 16: return cfg_d<16>(nqv);
      case 32: return cfg_d<32>(nqv);
      case 64: return cfg_d<64>(nqv);
      case 128: return cfg_d<128>(nqv);
      case 256: return cfg_d<256>(nqv);
      case 512: return cfg_d<512>(nqv);
      case 1024: return cfg_d<1024>(nqv);
    }
    return ScanCfg{0, 0, 0};
  }
};

}  // namespace linr
