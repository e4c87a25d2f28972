// Host side of the C ABI declared in include/linr.h: validation, storage layout, launch planning.
// Every step of the search runs in this library's kernels (scan_gemv.cuh, merge.cu); PyTorch only
// supplies the device buffers and the stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace linr {
cudaError_t launch_scan_gemv_f32(int, int, const ScanParams&, int, size_t, cudaStream_t);
cudaError_t launch_scan_gemv_f16(int, int, const ScanParams&, int, size_t, cudaStream_t);
cudaError_t launch_scan_gemv_bf16(int, int, const ScanParams&, int, size_t, cudaStream_t);
cudaError_t launch_scan_gemv_i8(int, int, const ScanParams&, int, size_t, cudaStream_t);
ScanCfg scan_cfg_f32(int, int);
ScanCfg scan_cfg_f16(int, int);
ScanCfg scan_cfg_bf16(int, int);
ScanCfg scan_cfg_i8(int, int);

static unsigned long long* g_dbg_host_ptr = nullptr;
static bool g_dbg_on = false;
unsigned long long* debug_buffer() { return g_dbg_on ? g_dbg_host_ptr : nullptr; }

cudaError_t ensure_smem(const void* kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  size_t& have = granted[{kernel, dev}];
  if (smem <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) have = smem;
  return e;
}
// Tuning knobs: environment, read per search (each knob has a GPU parity test that sets it).
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
static thread_local std::string g_detail;   // launch-site detail appended to the next CUDA failure
void set_error_detail(const std::string& d) { g_detail = d; }

static int esize(int dt) { return dt == LINR_F32 ? 4 : (dt == LINR_I8 ? 1 : 2); }
static bool dim_ok(int d) { return d == 16 || d == 32 || d == 64 || d == 128 || d == 256 || d == 512 || d == 1024; }
static int64_t pad_rows(int64_t cap) { return (cap + kTileItems - 1) / kTileItems * kTileItems; }

cudaError_t launch_scan_gemv(int dtype, int dim, int nqv, const ScanParams& p, int grid, size_t smem,
                             cudaStream_t st) {
  switch (dtype) {
    case LINR_F32: return launch_scan_gemv_f32(dim, nqv, p, grid, smem, st);
    case LINR_F16: return launch_scan_gemv_f16(dim, nqv, p, grid, smem, st);
    case LINR_BF16: return launch_scan_gemv_bf16(dim, nqv, p, grid, smem, st);
    case LINR_I8: return launch_scan_gemv_i8(dim, nqv, p, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}
ScanCfg scan_gemv_cfg(int dtype, int dim, int nqv) {
  switch (dtype) {
    case LINR_F32: return scan_cfg_f32(dim, nqv);
    case LINR_F16: return scan_cfg_f16(dim, nqv);
    case LINR_BF16: return scan_cfg_bf16(dim, nqv);
    case LINR_I8: return scan_cfg_i8(dim, nqv);
  }
  return ScanCfg{0, 0, 0};
}
// query registers per lane = nqv * (chunks per lane) * (fp32 values or packed words per chunk);
// mirrors geom_lpr() in scan_gemv.cuh
bool scan_gemv_supported(int dtype, int dim, int nqv) {
  if (!dim_ok(dim)) return false;
  const int ch = dim * esize(dtype) / 16;
  const int per = dtype == LINR_I8 ? 4 : 16 / esize(dtype);
  int lpr = ch / 4 > 4 ? ch / 4 : 4;
  if (lpr > 32) lpr = 32;
  if (lpr > ch) lpr = ch;
  while (lpr < ch && lpr < 32 && nqv * (ch / lpr) * per > 32) lpr *= 2;
  return nqv * (ch / lpr) * per <= 64;
}

}  // namespace linr

using namespace linr;

constexpr int kPinSlots = 16;

struct ProfEvents {
  cudaEvent_t e0, e1, e2;   // before scan, after scan (= before merge), after merge
};

struct linr_index {
  linr_index_desc d;
  // batched tcgen05 path state
  CUtensorMap tmx;
  bool tmx_ok = false;
  // pinned staging ring for the batched path's clause tables: one slot per search in flight
  // (ABI: up to 16), reused round-robin; a slot is reused once its previous copy has executed
  struct PinSlot {
    void* p = nullptr;
    size_t bytes = 0;
    cudaEvent_t ev = nullptr;
  } pin[kPinSlots];
  int pin_next = 0;
  // Sign-OPORP 1-bit codes of the rows (linr_codes_attach): [cap_pad][code_k/64] u64 + params
  uint64_t* codes = nullptr;
  int code_k = 0, code_L = 0;
  int32_t* c_src = nullptr;
  int8_t* c_sign = nullptr;
  // ID-list attribute slots (linr_idlists_attach): ids [sumA][cap_pad] u64, counts [S][cap_pad] u8
  uint64_t* idl_ids = nullptr;
  uint8_t* idl_cnt = nullptr;
  int idl_S = 0;
  int idl_A[4] = {0, 0, 0, 0};
  int idl_off[4] = {0, 0, 0, 0};
  // learned scorer (linr_scorer_attach): weights + item features y [cap_pad][Fp]
  bool scorer = false;
  ScorerDev sw;
  float* sy = nullptr;
  void* comm = nullptr;         // NCCL communicator over the shards (linr_comm_init)
  int comm_rank = 0, comm_world = 1;
  bool prof = false;
  std::vector<ProfEvents> prof_used, prof_free;
  int64_t prof_launches = 0;
  uint64_t fuse_seq = 0;        // fused-merge ticket slot rotation
  bool force_gemv = false;
  int64_t cap_pad;
  int rowbytes;
  int num_sms;
  size_t smem_optin;
  void* emb;
  uint64_t* attr;
  uint32_t* live;
  DevHeader* hdr;
};

namespace {

struct DeviceGuard {
  int prev = -1, want;
  explicit DeviceGuard(int dev) : want(dev) {
    cudaGetDevice(&prev);
    if (prev != want) cudaSetDevice(want);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e) + (g_detail.empty() ? "" : " (" + g_detail + ")"));
  g_detail.clear();
  return LINR_ECUDA;
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ----------------------------------------------------------------- search planning
struct Plan {
  int nu_g = 0;       // users per scan launch
  int groups = 0;
  int nqv = 0;
  int nt = 0;
  int C = 0, bufcap = 0;
  int list_cap = 0;   // per-CTA output list capacity
  int ring = 0;       // > 0: warp-specialised scan with this many row-group slots
  size_t smem = 0;
  int grid = 0;
};

constexpr size_t kScanCtlBytes = 2048;   // >= sizeof(ScanCtl) (static_assert in scan_gemv.cuh)

bool make_plan(const linr_index* ix, int B, int V, int K, Plan* pl, std::string* why, bool one_user = false,
               int force_nu = 0) {
  const int dt = ix->d.dtype, dim = ix->d.dim;
  int nu = std::max(1, std::min(B, std::min(kMaxUsers, 8 / V)));
  if (one_user) nu = 1;   // per-user liveness bitmaps (ID-list clauses): one user per launch
  // The ring scan runs one user per launch: a user's key buffer then gets most of the shared
  // memory the ring leaves (measured at c2 HIGH, B = 4 / 8: one launch per user 0.31 / 0.62 ms,
  // users sharing a launch -- and its buffers, hence many compactions -- 0.81 / 2.48 ms).
  const bool ws_ok = !std::getenv("LINR_NO_WS") && !std::getenv("LINR_MAX_NU");
  const int nu_first = nu;
  if (ws_ok) nu = 1;
  if (const char* mn = std::getenv("LINR_MAX_NU")) nu = std::max(1, std::min(nu, std::atoi(mn)));
  if (force_nu > 0) nu = force_nu;   // union path: every user in one ring-scan launch, or no plan
  for (int pass = ws_ok ? 0 : 1; pass < 2; ++pass, nu = one_user ? 1 : nu_first) {
  for (; nu >= 1; --nu) {
    if (force_nu > 0 && (nu != force_nu || pass != 0)) return false;
    const int nqv = next_pow2(nu * V);
    if (nqv > 8 || !scan_gemv_supported(dt, dim, nqv)) continue;
    const ScanCfg cfg = scan_gemv_cfg(dt, dim, nqv);
    if (cfg.nt == 0) continue;
    const int nw = cfg.nt / 32;
    if (pass == 0 && cfg.ws_slot_bytes == 0) break;   // no ring kernel for this shape
    if (pass == 0) {
      // ring scan (scan_ws.cuh): R (a power of two) slots of 16 rows, ~128 KB of rows in flight
      // by default; the rest of shared memory for the per-user key buffers (>= K + 256 keys)
      const int head = cfg.ws_cons_warps * 16;
      const size_t rows_b = (size_t)cfg.ws_slot_bytes - 96;
      const char* rk = std::getenv("LINR_WS_RING_KB");   // tuning knob (KB of rows in the ring)
      const size_t ring_target = (rk ? (size_t)std::atoi(rk) : 128) * 1024;
      int R = 8;
      while (R < 64 && (size_t)(2 * R) * rows_b <= ring_target) R *= 2;
      long long C = 0;
      for (; R >= 8; R /= 2) {
        const size_t fixed = (size_t)cfg.ws_fixed_bytes + (size_t)R * cfg.ws_slot_bytes;
        if (ix->smem_optin <= fixed) continue;
        C = (long long)((ix->smem_optin - fixed) / (8 * (size_t)nu)) - head;
        // a smaller buffer raises the CTA's threshold earlier (compactions stall only the scoring
        // warps, the producers keep the ring busy) and leaves fewer keys for the tail to select
        const char* cm = std::getenv("LINR_WS_CMAX");
        C = std::min<long long>(C, std::max<long long>(cm ? std::atoll(cm) : 32768, K + 256));
        C &= ~255ll;
        if (C >= K + 256) break;
      }
      if (R >= 8) {
        pl->nu_g = nu;
        pl->groups = (B + nu - 1) / nu;
        pl->nqv = nqv;
        pl->nt = cfg.nt;
        pl->C = (int)C;
        pl->bufcap = (int)C + head;
        pl->ring = R;
        pl->smem = std::max((size_t)cfg.ws_fixed_bytes + (size_t)R * cfg.ws_slot_bytes + (size_t)nu * pl->bufcap * 8,
                            merge_smem());
        pl->grid = (pl->groups == 1 && ix->num_sms > 1) ? ix->num_sms - 1 : ix->num_sms;
        pl->list_cap = (B <= 8) ? pl->bufcap : std::min(pl->bufcap, std::max(2 * K, 2048));
        return true;
      }
      break;   // the ring kernel does not fit: per-warp kernel plans (pass 1)
    }
    const int head = nw * cfg.rows_per_iter;
    const size_t fixed = kScanCtlBytes + (size_t)nw * kTileItems * 2 + (size_t)nw * cfg.ring_bytes;
    if (ix->smem_optin <= fixed) continue;
    // the largest per-user buffer that fits: fewer compactions (each one drains the CTA)
    long long C = (long long)((ix->smem_optin - fixed) / (8 * (size_t)nu)) - head;
    C = std::min<long long>(C, 32768);
    C &= ~255ll;
    if (C < K + 256) continue;
    pl->nu_g = nu;
    pl->groups = (B + nu - 1) / nu;
    pl->nqv = nqv;
    pl->nt = cfg.nt;
    pl->C = (int)C;
    pl->bufcap = (int)C + head;
    pl->smem = std::max(fixed + (size_t)nu * pl->bufcap * 8, merge_smem());
    // one launch with a fused merge: leave one SM free so the merging CTA of this search and the
    // scan of a search issued on another stream overlap without a straggler CTA
    pl->grid = (pl->groups == 1 && ix->num_sms > 1) ? ix->num_sms - 1 : ix->num_sms;
    pl->list_cap = (B <= 8) ? pl->bufcap : std::min(pl->bufcap, std::max(2 * K, 2048));
    return true;
  }
  }
  *why = "no GEMV scan configuration fits (dtype " + std::to_string(dt) + ", dim " + std::to_string(dim) +
         ", V " + std::to_string(V) + ", K " + std::to_string(K) + ")";
  return false;
}

struct WsLayout {
  size_t samp = 0, list = 0, cnt = 0, pass = 0, end = 0;
};
WsLayout ws_layout(const Plan& pl, int B, int K) {
  (void)K;
  WsLayout w;
  const size_t parts = (size_t)B * pl.grid;
  w.samp = 0;
  w.list = align256(parts * kScanSample * 8);
  w.cnt = w.list + align256(parts * pl.list_cap * 8);
  w.pass = w.cnt + align256(parts * 4);
  w.end = w.pass + align256(parts * 8);
  return w;
}


// ----------------------------------------------------------------- batched tcgen05 path
struct TcWs {
  size_t sbuf, scnt, thr, mbuf, mcnt, flags, cl, ncl, fb, bar, end;
};
int max_clauses(const int32_t* off, int B) {
  int m = 0;
  for (int b = 0; b < B; ++b) m = std::max(m, (int)(off[b + 1] - off[b]));
  return m;
}
int max_word(const linr_clause* cl, const int32_t* off, int B) {   // attribute words the clauses read
  int w = 0;
  for (int i = 0; i < off[B]; ++i) w = std::max(w, (int)cl[i].word + 1);
  return w;
}
// Smallest B*V that takes the batched tensor-core path (tuning knob LINR_TC_MIN, default 9 from
// the measured crossover on c2 HIGH, profiles/r02z: B = 8 GEMV 0.63 ms vs tcgen05 0.73 ms, B = 12
// tcgen05 0.47 ms, GEMV ~0.08 ms per user; below it the GEMV ring scan runs one user per launch).
int tc_min_vectors() {
  static const int v = [] {
    const char* e = std::getenv("LINR_TC_MIN");
    return e ? std::max(1, std::atoi(e)) : 9;
  }();
  return v;
}
bool use_tc(const linr_index* ix, int B, int V, int maxc, int wmax) {
  return B * V >= tc_min_vectors() && tc_supported(ix->d.dtype, ix->d.dim, B * V, V) &&
         tc_smem_bytes(ix->d.dtype, ix->d.dim, tc_np(B * V), B, maxc, wmax) <= (size_t)ix->smem_optin;
}
// Without pass counts (the batched path computes them with an extra clause evaluation per
// (row, user)) the dense tcgen05 pass wins from B*V = 7: c2 HIGH B = 8 0.43 ms vs union 0.56 ms.
bool use_tc_nopass(const linr_index* ix, int B, int V, int maxc, int wmax) {
  return B * V >= std::min(tc_min_vectors(), 7) && tc_supported(ix->d.dtype, ix->d.dim, B * V, V) &&
         tc_smem_bytes(ix->d.dtype, ix->d.dim, tc_np(B * V), B, maxc, wmax) <= (size_t)ix->smem_optin;
}
bool tc_layout(const linr_index* ix, int B, int V, int K, TcWs* w, std::string* why) {
  (void)V;
  (void)why;
  const size_t nu = (size_t)B;
  w->sbuf = 0;
  const size_t G = (size_t)ix->num_sms;
  w->scnt = align256(w->sbuf + nu * G * kTcSampleCap * 8);
  w->thr = align256(w->scnt + nu * G * 4);
  w->mbuf = align256(w->thr + nu * 8);
  w->mcnt = align256(w->mbuf + nu * G * kTcMainCap * 8);
  w->flags = align256(w->mcnt + nu * G * 4);
  w->cl = align256(w->flags + nu * 4);
  w->ncl = w->cl + nu * 16 * sizeof(KClause);   // adjacent: one staging copy
  w->fb = align256(w->ncl + nu * 4);
  w->bar = align256(w->fb + fallback_ws_bytes(ix->num_sms, K));
  w->end = w->bar + 256;
  return true;
}

int search_impl(linr_index* ix, const void* q, int B, int V, const linr_clause* cl, const int32_t* off, int K,
                void* ws, size_t ws_bytes, int mode, int64_t* out_ids, float* out_scores, uint64_t* out_keys,
                int64_t* out_pass, cudaStream_t st, const uint32_t* live_ovr = nullptr, size_t live_ovr_words = 0);

// Clause table [B][16] KClause followed by counts [B] int, copied host -> pinned slot -> dst_dev on
// st (one copy). The pinned slot is reused kPinSlots calls later, once its copy has executed.
int stage_clause_table(linr_index* ix, const linr_clause* cl, const int32_t* off, int B, void* dst_dev,
                       cudaStream_t st) {
  const size_t clb = (size_t)B * 16 * sizeof(KClause), nclb = (size_t)B * 4;
  const size_t need = clb + nclb;
  linr_index::PinSlot& ps = ix->pin[ix->pin_next];
  ix->pin_next = (ix->pin_next + 1) % kPinSlots;
  if (!ps.ev && cudaEventCreateWithFlags(&ps.ev, cudaEventDisableTiming) != cudaSuccess)
    return fail(LINR_ECUDA, "staging event");
  cudaEventSynchronize(ps.ev);   // the copy out of this slot (kPinSlots searches ago) has executed
  if (ps.bytes < need) {
    if (ps.p) cudaFreeHost(ps.p);
    ps.p = nullptr;
    ps.bytes = 0;
    if (cudaHostAlloc(&ps.p, need, cudaHostAllocDefault) != cudaSuccess) return fail(LINR_ENOMEM, "pinned staging");
    ps.bytes = need;
  }
  KClause* hcl = (KClause*)ps.p;
  int* hncl = (int*)((char*)ps.p + clb);
  std::memset(hcl, 0, clb);
  for (int b = 0; b < B; ++b) {
    hncl[b] = off[b + 1] - off[b];
    for (int c = 0; c < hncl[b]; ++c) {
      const linr_clause& k = cl[off[b] + c];
      hcl[b * 16 + c].mask = k.mask;
      hcl[b * 16 + c].word = k.word;
      hcl[b * 16 + c].rev = k.reverse;
    }
  }
  cudaError_t e = cudaMemcpyAsync(dst_dev, ps.p, need, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaEventRecord(ps.ev, st);
  if (e != cudaSuccess) return cuda_fail(e, "clause staging");
  return LINR_OK;
}

int search_tc(linr_index* ix, const void* q, int B, int V, const linr_clause* cl, const int32_t* off, int K,
              void* ws, size_t ws_bytes, int mode, int64_t* out_ids, float* out_scores, uint64_t* out_keys,
              int64_t* out_pass, cudaStream_t st) {
  std::string why;
  TcWs w;
  if (!tc_layout(ix, B, V, K, &w, &why)) return fail(LINR_EUNSUPPORTED, why);
  if (!ws || ws_bytes < w.end) return fail(LINR_ENOMEM, "workspace too small");
  DeviceGuard dg(ix->d.device);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pending CUDA error");
  const int nvec = B * V, np = tc_np(nvec);
  char* W = (char*)ws;
  if (!ix->tmx_ok) {
    ix->tmx_ok = tc_encode_map(&ix->tmx, ix->emb, ix->cap_pad, ix->rowbytes, 128);
    if (!ix->tmx_ok) return fail(LINR_ECUDA, "cuTensorMapEncodeTiled failed for the item matrix");
  }
  TcParams p;
  std::memset(&p, 0, sizeof(p));
  p.tmx = ix->tmx;
  if (!tc_encode_map(&p.tmq, q, nvec, ix->rowbytes, np)) return fail(LINR_ECUDA, "cuTensorMapEncodeTiled failed for the queries");
  // clauses: host -> pinned staging slot -> device (clause lists are host memory per the ABI)
  {
    const int rc = stage_clause_table(ix, cl, off, B, W + w.cl, st);   // cl and ncl are adjacent in ws
    if (rc != LINR_OK) return rc;
  }

  ProfEvents pe{};
  if (ix->prof) {
    if (!ix->prof_free.empty()) {
      pe = ix->prof_free.back();
      ix->prof_free.pop_back();
    } else {
      cudaEventCreate(&pe.e0);
      cudaEventCreate(&pe.e1);
      cudaEventCreate(&pe.e2);
    }
    cudaEventRecord(pe.e0, st);
  }
  p.attr = ix->attr;
  p.cap_pad = ix->cap_pad;
  p.live = ix->live;
  p.hdr = ix->hdr;
  p.row0 = (uint32_t)ix->d.global_row0;
  p.nu = B;
  p.V = V;
  p.nvec = nvec;
  p.K = K;
  p.wmax = max_word(cl, off, B);
  p.cl = (const KClause*)(W + w.cl);
  p.ncl = (const int*)(W + w.ncl);
  p.maxc = max_clauses(off, B);
  p.dyn = env_int("LINR_TC_DYN", 0);   // measured slower (r02dyn: B=256 1.36 vs 1.30 ms)
  p.dbg = nullptr;
  // 1. sample pass (no threshold)
  p.thr = nullptr;
  p.buf = (uint64_t*)(W + w.sbuf);
  p.cap = kTcSampleCap;
  p.cnt = (int*)(W + w.scnt);
  p.sample_tiles = kTcSampleTiles;
  e = launch_tc_scan(ix->d.dtype, ix->d.dim, np, p, ix->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "tc sample launch");
  // 2. thresholds
  e = launch_tc_threshold((const uint64_t*)(W + w.sbuf), (const int*)(W + w.scnt), kTcSampleCap, ix->num_sms, B, K,
                          ix->num_sms * kTcSampleTiles * 128, ix->hdr, (uint64_t*)(W + w.thr), st);
  if (e != cudaSuccess) return cuda_fail(e, "tc threshold launch");
  {
    // 2b. large shards: the first sample covers too few rows (lambda = K * sampled / rows < 8: a
    // threshold several times looser than the K-th key, hence several times more hot pairs in the
    // main pass). A second, main-style pass over more spread tiles collects only keys >= T1 (few,
    // so the regions do not truncate) and refines the thresholds (never below T1). Rows are taken
    // from the capacity (the host does not read the high-water mark).
    const double rows = (double)std::max<int64_t>(1, ix->d.capacity_rows);
    const double lam1 = (double)K * std::min(1.0, (double)ix->num_sms * kTcSampleTiles * 128 / rows);
    const int s2 = (int)std::min(256.0, std::ceil(12.0 * rows / ((double)K * ix->num_sms * 128)));
    if (lam1 < 8.0 && s2 > kTcSampleTiles && env_int("LINR_TC_REFINE", 1)) {
      TcParams p2 = p;
      p2.thr = (const uint64_t*)(W + w.thr);
      p2.buf = (uint64_t*)(W + w.sbuf);
      p2.cap = kTcSampleCap;
      p2.cnt = (int*)(W + w.scnt);
      p2.sample_tiles = s2;
      p2.sample_thr = 1;
      e = launch_tc_scan(ix->d.dtype, ix->d.dim, np, p2, ix->num_sms, st);
      if (e != cudaSuccess) return cuda_fail(e, "tc refine launch");
      e = launch_tc_threshold((const uint64_t*)(W + w.sbuf), (const int*)(W + w.scnt), kTcSampleCap, ix->num_sms, B,
                              K, ix->num_sms * s2 * 128, ix->hdr, (uint64_t*)(W + w.thr), st,
                              (const uint64_t*)(W + w.thr));
      if (e != cudaSuccess) return cuda_fail(e, "tc refine threshold launch");
      if (ix->prof) ix->prof_launches += 2;
    }
  }
  // 3. main pass
  p.thr = (const uint64_t*)(W + w.thr);
  p.buf = (uint64_t*)(W + w.mbuf);
  p.cap = kTcMainCap;
  if (const char* mc = std::getenv("LINR_TC_MAIN_CAP"))   // test knob: small regions force the fallback
    p.cap = std::max(1, std::min(kTcMainCap, std::atoi(mc)));
  p.cnt = (int*)(W + w.mcnt);
  p.sample_tiles = 0;
  p.dbg = debug_buffer();
  e = launch_tc_scan(ix->d.dtype, ix->d.dim, np, p, ix->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "tc main launch");
  if (ix->prof) cudaEventRecord(pe.e1, st);
  // 4. finalize
  e = launch_tc_finalize((const uint64_t*)(W + w.mbuf), (const int*)(W + w.mcnt), p.cap, ix->num_sms,
                         (const uint64_t*)(W + w.thr), B, K, mode == 0 ? out_ids : nullptr,
                         mode == 0 ? out_scores : nullptr, mode == 1 ? out_keys : nullptr, (int*)(W + w.flags),
                         (unsigned int*)(W + w.bar), st);
  if (e != cudaSuccess) return cuda_fail(e, "tc finalize launch");
  // 5. certification on the device: flagged users are recomputed exactly (fallback.cu); when no
  //    user is flagged the launch reads the flags and exits. No host synchronisation.
  FbParams fp;
  std::memset(&fp, 0, sizeof(fp));
  fp.emb = ix->emb;
  fp.attr = ix->attr;
  fp.cap_pad = ix->cap_pad;
  fp.live = ix->live;
  fp.hdr = ix->hdr;
  fp.row0 = (uint32_t)ix->d.global_row0;
  fp.dim = ix->d.dim;
  fp.V = V;
  fp.K = K;
  fp.nu = B;
  fp.q = q;
  fp.cl = p.cl;
  fp.ncl = p.ncl;
  fp.flags = (const int*)(W + w.flags);
  fp.lists = (uint64_t*)(W + w.fb);
  fp.bar = (unsigned int*)(W + w.bar);
  fp.out_ids = mode == 0 ? out_ids : nullptr;
  fp.out_scores = mode == 0 ? out_scores : nullptr;
  fp.out_keys = mode == 1 ? out_keys : nullptr;
  e = launch_fallback(ix->d.dtype, fp, ix->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "tc fallback launch");
  if (out_pass) {
    e = cudaMemsetAsync(out_pass, 0, (size_t)B * 8, st);
    if (e == cudaSuccess)
      e = launch_tc_count(ix->attr, ix->cap_pad, ix->live, ix->hdr, p.cl, p.ncl, B, (unsigned long long*)out_pass,
                          ix->num_sms * 4, st);
    if (e != cudaSuccess) return cuda_fail(e, "tc pass-count launch");
  }
  if (ix->prof) {
    cudaEventRecord(pe.e2, st);
    ix->prof_used.push_back(pe);
    ix->prof_launches += 5 + (out_pass ? 1 : 0);
  }
  return LINR_OK;
}

int validate_query(const linr_index* ix, const void* q, int B, int V, const linr_clause* cl, const int32_t* off,
                   int K, std::string* why) {
  if (!ix) { *why = "null index"; return LINR_EINVAL; }
  if (!q) { *why = "null queries"; return LINR_EINVAL; }
  if (B < 1) { *why = "B must be >= 1"; return LINR_EINVAL; }
  if (V < 1 || V > 8) { *why = "V must be in [1, 8]"; return LINR_EINVAL; }
  if (K < 1 || K > LINR_MAX_K) { *why = "K must be in [1, 2048]"; return LINR_EINVAL; }
  if (!off) { *why = "null clause offsets"; return LINR_EINVAL; }
  if (off[0] != 0) { *why = "clause_off[0] must be 0"; return LINR_EINVAL; }
  for (int b = 0; b < B; ++b) {
    const int n = off[b + 1] - off[b];
    if (n < 0) { *why = "clause offsets must be non-decreasing"; return LINR_EINVAL; }
    if (n > LINR_MAX_CLAUSES) { *why = "more than 16 clauses in one query"; return LINR_EINVAL; }
    if (n > 0 && !cl) { *why = "null clauses"; return LINR_EINVAL; }
    for (int c = off[b]; c < off[b + 1]; ++c) {
      if (cl[c].mask == 0) { *why = "empty clause mask (omit the clause instead)"; return LINR_EINVAL; }
      if (cl[c].word >= ix->d.attr_words) { *why = "clause word >= attr_words"; return LINR_EINVAL; }
      if (cl[c].reverse > 1) { *why = "clause reverse must be 0 or 1"; return LINR_EINVAL; }
    }
  }
  return LINR_OK;
}

// ----------------------------------------------------------------- union path (2 <= B*V <= 8)
// Small batches share one pass over the index: the tcgen05 sample pass + threshold kernel give
// each user a starting threshold T_u (the batched path's, reading R23), then ONE ring-scan launch
// evaluates every user's clauses per tile and gathers the union of their passing rows once
// (instead of one attribute pass + one row gather per user), keeping only keys >= T_u, so the
// per-user CTA buffers stay small; the merge flags users with fewer than K keys >= T_u and the
// fallback kernel recomputes them exactly (no host synchronisation). LINR_UNION=0 disables it.
bool union_ok(const linr_index* ix, int B, int V, int maxc, int wmax) {
  // measured (profiles/r02w): B = 8 HIGH 0.56 vs 0.62 ms per-user, ALL 0.58 vs 3.9 ms, LOW 0.20 vs
  // 0.38 ms; B = 4 equal at HIGH; B = 2 and V > 1 (the consumers' V-max path) slower -> per user
  // B in [9, 16] (two ring-scan launches of <= 8 users) only behind the device-side gate, i.e.
  // without pass counts (search_impl)
  if (V != 1 || B < 3 || B > 16 || env_int("LINR_UNION", 1) == 0) return false;
  if (std::getenv("LINR_NO_WS") || std::getenv("LINR_MAX_NU")) return false;   // kernel-variant knobs
  return tc_supported(ix->d.dtype, ix->d.dim, B * V, V) &&
         tc_smem_bytes(ix->d.dtype, ix->d.dim, tc_np(B * V), B, maxc, wmax) <= (size_t)ix->smem_optin;
}
size_t union_ws_bytes(const linr_index* ix, int B, int V, int K, Plan* pl) {
  std::string why;
  TcWs w;
  if (!tc_layout(ix, B, V, K, &w, &why)) return 0;
  if (!make_plan(ix, B, V, K, pl, &why, false, std::min(B, kMaxUsers))) return 0;
  return align256(w.end) + ws_layout(*pl, B, K).end;
}

int search_union(linr_index* ix, const void* q, int B, int V, const linr_clause* cl, const int32_t* off, int K,
                 void* ws, size_t ws_bytes, int mode, int64_t* out_ids, float* out_scores, uint64_t* out_keys,
                 int64_t* out_pass, cudaStream_t st) {
  std::string why;
  Plan pl;
  const size_t need = union_ws_bytes(ix, B, V, K, &pl);
  if (need == 0) return fail(LINR_EUNSUPPORTED, "no union-path plan");
  if (!ws || ws_bytes < need) return fail(LINR_ENOMEM, "workspace too small");
  TcWs w;
  tc_layout(ix, B, V, K, &w, &why);
  DeviceGuard dg(ix->d.device);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pending CUDA error");
  char* W = (char*)ws;
  const int nvec = B * V, np = tc_np(nvec);
  if (!ix->tmx_ok) {
    ix->tmx_ok = tc_encode_map(&ix->tmx, ix->emb, ix->cap_pad, ix->rowbytes, 128);
    if (!ix->tmx_ok) return fail(LINR_ECUDA, "cuTensorMapEncodeTiled failed for the item matrix");
  }
  TcParams p;
  std::memset(&p, 0, sizeof(p));
  p.tmx = ix->tmx;
  if (!tc_encode_map(&p.tmq, q, nvec, ix->rowbytes, np)) return fail(LINR_ECUDA, "cuTensorMapEncodeTiled failed for the queries");
  {
    const int rc = stage_clause_table(ix, cl, off, B, W + w.cl, st);
    if (rc != LINR_OK) return rc;
  }
  ProfEvents pe{};
  if (ix->prof) {
    if (!ix->prof_free.empty()) {
      pe = ix->prof_free.back();
      ix->prof_free.pop_back();
    } else {
      cudaEventCreate(&pe.e0);
      cudaEventCreate(&pe.e1);
      cudaEventCreate(&pe.e2);
    }
    cudaEventRecord(pe.e0, st);
  }
  // 1. sample pass + thresholds (the batched path's kernels)
  p.attr = ix->attr;
  p.cap_pad = ix->cap_pad;
  p.live = ix->live;
  p.hdr = ix->hdr;
  p.row0 = (uint32_t)ix->d.global_row0;
  p.nu = B;
  p.V = V;
  p.nvec = nvec;
  p.K = K;
  p.wmax = max_word(cl, off, B);
  p.cl = (const KClause*)(W + w.cl);
  p.ncl = (const int*)(W + w.ncl);
  p.maxc = max_clauses(off, B);
  p.dyn = env_int("LINR_TC_DYN", 0);   // measured slower (r02dyn: B=256 1.36 vs 1.30 ms)
  p.thr = nullptr;
  p.buf = (uint64_t*)(W + w.sbuf);
  p.cap = kTcSampleCap;
  p.cnt = (int*)(W + w.scnt);
  p.sample_tiles = kTcSampleTiles;
  e = launch_tc_scan(ix->d.dtype, ix->d.dim, np, p, ix->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "union sample launch");
  uint64_t* thr = (uint64_t*)(W + w.thr);
  e = launch_tc_threshold((const uint64_t*)(W + w.sbuf), (const int*)(W + w.scnt), kTcSampleCap, ix->num_sms, B, K,
                          ix->num_sms * kTcSampleTiles * 128, ix->hdr, thr, st);
  if (e != cudaSuccess) return cuda_fail(e, "union threshold launch");
  if (env_int("LINR_UNION_FORCE_FB", 0))   // test knob: thresholds above every key -> every user recomputed
    e = cudaMemsetAsync(thr, 0xFF, (size_t)B * 8, st);
  if (e != cudaSuccess) return cuda_fail(e, "union threshold override");
  // 2a. B*V >= 7 without pass counts: at high/medium pass rates the dense tcgen05 pass beats the
  //     union scan (B = 8: 0.44 vs 0.56 ms); at low pass rates it does not (1.38 vs 0.20 ms). The thresholds live on the device, so the
  //     choice is made there: a one-CTA kernel writes a gate, both paths are launched and the one
  //     not chosen exits at once (profiles/r02gate).
  int* gate = nullptr;
  if (out_pass == nullptr && B * V >= 7 && env_int("LINR_UNION_TC", 1) &&
      use_tc_nopass(ix, B, V, max_clauses(off, B), max_word(cl, off, B))) {
    gate = (int*)(W + w.bar + 128);
    e = launch_tc_decide(thr, (const int*)(W + w.scnt), ix->num_sms, (int64_t)ix->num_sms * kTcSampleTiles * 128,
                         ix->hdr, B, gate, st);
    if (e != cudaSuccess) return cuda_fail(e, "union decide launch");
    TcParams pm = p;
    pm.thr = thr;
    pm.buf = (uint64_t*)(W + w.mbuf);
    pm.cap = kTcMainCap;
    pm.cnt = (int*)(W + w.mcnt);
    pm.sample_tiles = 0;
    pm.gate = gate;
    pm.gate_want = 1;
    e = launch_tc_scan(ix->d.dtype, ix->d.dim, np, pm, ix->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "union tc main launch");
    e = launch_tc_finalize((const uint64_t*)(W + w.mbuf), (const int*)(W + w.mcnt), kTcMainCap, ix->num_sms, thr, B,
                           K, mode == 0 ? out_ids : nullptr, mode == 0 ? out_scores : nullptr,
                           mode == 1 ? out_keys : nullptr, (int*)(W + w.flags), (unsigned int*)(W + w.bar), st, gate);
    if (e != cudaSuccess) return cuda_fail(e, "union tc finalize launch");
    if (ix->prof) ix->prof_launches += 3;
  }
  // 2. one ring-scan launch for every user, starting from the thresholds
  const size_t uoff = align256(w.end);
  const WsLayout wl = ws_layout(pl, B, K);
  uint64_t* samp = (uint64_t*)(W + uoff + wl.samp);
  uint64_t* lists = (uint64_t*)(W + uoff + wl.list);
  int* cnts = (int*)(W + uoff + wl.cnt);
  int64_t* pass = (int64_t*)(W + uoff + wl.pass);
  MergeParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.samp = samp;
  mp.samp_sl = kScanSample;
  mp.samp_su = (int64_t)pl.grid * kScanSample;
  mp.ms = kScanSample;
  mp.list = lists;
  mp.list_sl = pl.list_cap;
  mp.list_su = (int64_t)pl.grid * pl.list_cap;
  mp.cnt = cnts;
  mp.cnt_sl = 1;
  mp.cnt_su = pl.grid;
  mp.list_len = pl.list_cap;
  mp.pass = pass;
  mp.pstride_l = 1;
  mp.pstride_u = pl.grid;
  mp.L = pl.grid;
  mp.K = K;
  mp.out_ids = out_ids;
  mp.out_scores = out_scores;
  mp.out_keys = out_keys;
  mp.out_pass = out_pass;
  mp.mode = mode;
  mp.thr = thr;
  mp.flags = (int*)(W + w.flags);
  mp.dbg = debug_buffer();
  mp.gate = gate;
  mp.gate_want = 0;
  // one ring-scan launch per group of <= kMaxUsers users (one launch for B <= 8)
  for (int u0 = 0; u0 < B; u0 += pl.nu_g) {
    const int nu = std::min(pl.nu_g, B - u0);
    ScanParams sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.emb = ix->emb;
    sp.attr = ix->attr;
    sp.live = ix->live;
    sp.hdr = ix->hdr;
    sp.cap_pad = ix->cap_pad;
    sp.row0 = (uint32_t)ix->d.global_row0;
    sp.nu = nu;
    sp.V = V;
    sp.K = K;
    sp.C = pl.C;
    sp.bufcap = pl.bufcap;
    sp.list_cap = pl.list_cap;
    sp.dbg = debug_buffer();
    sp.q = (const char*)q + (size_t)u0 * V * ix->rowbytes;
    const size_t part0 = (size_t)u0 * pl.grid;
    sp.out_samp = samp + part0 * kScanSample;
    sp.out_list = lists + part0 * pl.list_cap;
    sp.out_cnt = cnts + part0;
    sp.out_pass = pass + part0;
    uint32_t wmask = 0;
    for (int u = 0; u < nu; ++u) {
      const int b = u0 + u;
      sp.ncl[u] = off[b + 1] - off[b];
      for (int c = 0; c < sp.ncl[u]; ++c) {
        const linr_clause& k = cl[off[b] + c];
        sp.cl[u][c].mask = k.mask;
        sp.cl[u][c].word = k.word;
        sp.cl[u][c].rev = k.reverse;
        wmask |= 1u << k.word;
      }
    }
    sp.wmask = wmask;
    sp.ring = pl.ring;
    sp.init_thr = thr + u0;
    sp.gate = gate;
    sp.gate_want = 0;
    sp.mp = mp;
    e = launch_scan_gemv(ix->d.dtype, ix->d.dim, pl.nqv, sp, pl.grid, pl.smem, st);
    if (e != cudaSuccess) return cuda_fail(e, "union scan launch");
    if (ix->prof && u0 > 0) ix->prof_launches += 1;
  }
  if (ix->prof) cudaEventRecord(pe.e1, st);
  // 3. merge (flags users with fewer than K keys >= T_u), 4. exact recomputation of flagged users
  e = launch_merge(mp, B, st, false);
  if (e != cudaSuccess) return cuda_fail(e, "union merge launch");
  e = cudaMemsetAsync(W + w.bar, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return cuda_fail(e, "union barrier reset");
  FbParams fp;
  std::memset(&fp, 0, sizeof(fp));
  fp.emb = ix->emb;
  fp.attr = ix->attr;
  fp.cap_pad = ix->cap_pad;
  fp.live = ix->live;
  fp.hdr = ix->hdr;
  fp.row0 = (uint32_t)ix->d.global_row0;
  fp.dim = ix->d.dim;
  fp.V = V;
  fp.K = K;
  fp.nu = B;
  fp.q = q;
  fp.cl = p.cl;
  fp.ncl = p.ncl;
  fp.flags = (const int*)(W + w.flags);
  fp.lists = (uint64_t*)(W + w.fb);
  fp.bar = (unsigned int*)(W + w.bar);
  fp.out_ids = mode == 0 ? out_ids : nullptr;
  fp.out_scores = mode == 0 ? out_scores : nullptr;
  fp.out_keys = mode == 1 ? out_keys : nullptr;
  e = launch_fallback(ix->d.dtype, fp, ix->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "union fallback launch");
  if (ix->prof) {
    cudaEventRecord(pe.e2, st);
    ix->prof_used.push_back(pe);
    ix->prof_launches += 5;
  }
  return LINR_OK;
}

// scan (+ per-CTA lists) then merge into either ids/scores (mode 0) or keys (mode 1)
// live_ovr: per-user liveness bitmaps [B][live_ovr_words] replacing the index's (ID-list clauses
// already applied, see linr_search_idc); forces the GEMV path with one user per launch.
int search_impl(linr_index* ix, const void* q, int B, int V, const linr_clause* cl, const int32_t* off, int K,
                void* ws, size_t ws_bytes, int mode, int64_t* out_ids, float* out_scores, uint64_t* out_keys,
                int64_t* out_pass, cudaStream_t st, const uint32_t* live_ovr, size_t live_ovr_words) {
  std::string why;
  int rc = validate_query(ix, q, B, V, cl, off, K, &why);
  if (rc != LINR_OK) return fail(rc, why);
  if (mode == 0 && (!out_ids || !out_scores)) return fail(LINR_EINVAL, "null outputs");
  if (mode == 1 && !out_keys) return fail(LINR_EINVAL, "null out_keys");
  // (without pass counts the dense tcgen05 pass would win from B*V = 7 at HIGH/ALL -- B = 8 0.43 ms
  // vs 0.56 ms on the union path -- but at LOW every user's sample threshold is 0 and it takes
  // 1.36 ms vs 0.20 ms; the host cannot tell the two apart, so B*V <= 8 stays on the union path
  // unless LINR_TC_NOPASS=1; profiles/r02np)
  if (!live_ovr && !ix->force_gemv && out_pass == nullptr && B * V >= 9 &&
      union_ok(ix, B, V, max_clauses(off, B), max_word(cl, off, B))) {
    // 9 <= B <= 16 without pass counts: the union path with its device-side gate runs the dense
    // tcgen05 pass at high pass rates and the union scans (two launches) at low ones
    Plan up;
    if (union_ws_bytes(ix, B, V, K, &up) > 0)
      return search_union(ix, q, B, V, cl, off, K, ws, ws_bytes, mode, out_ids, out_scores, out_keys, out_pass, st);
  }
  if (!live_ovr && !ix->force_gemv &&
      (use_tc(ix, B, V, max_clauses(off, B), max_word(cl, off, B)) ||
       (out_pass == nullptr && env_int("LINR_TC_NOPASS", 0) &&
        use_tc_nopass(ix, B, V, max_clauses(off, B), max_word(cl, off, B)))))
    return search_tc(ix, q, B, V, cl, off, K, ws, ws_bytes, mode, out_ids, out_scores, out_keys, out_pass, st);
  if (!live_ovr && !ix->force_gemv && B <= 8 && union_ok(ix, B, V, max_clauses(off, B), max_word(cl, off, B))) {
    Plan up;
    if (union_ws_bytes(ix, B, V, K, &up) > 0)
      return search_union(ix, q, B, V, cl, off, K, ws, ws_bytes, mode, out_ids, out_scores, out_keys, out_pass, st);
  }
  Plan pl;
  if (!make_plan(ix, B, V, K, &pl, &why, live_ovr != nullptr)) return fail(LINR_EUNSUPPORTED, why);
  const WsLayout wl = ws_layout(pl, B, K);
  if (!ws || ws_bytes < wl.end) return fail(LINR_ENOMEM, "workspace too small");
  DeviceGuard dg(ix->d.device);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pending CUDA error");

  uint64_t* samp = (uint64_t*)((char*)ws + wl.samp);
  uint64_t* lists = (uint64_t*)((char*)ws + wl.list);
  int* cnts = (int*)((char*)ws + wl.cnt);
  int64_t* pass = (int64_t*)((char*)ws + wl.pass);
  ProfEvents pe{};
  if (ix->prof) {
    if (!ix->prof_free.empty()) {
      pe = ix->prof_free.back();
      ix->prof_free.pop_back();
    } else {
      cudaEventCreate(&pe.e0);
      cudaEventCreate(&pe.e1);
      cudaEventCreate(&pe.e2);
    }
    cudaEventRecord(pe.e0, st);
  }
  MergeParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.samp = samp;
  mp.samp_sl = kScanSample;
  mp.samp_su = (int64_t)pl.grid * kScanSample;
  mp.ms = kScanSample;
  mp.list = lists;
  mp.list_sl = pl.list_cap;
  mp.list_su = (int64_t)pl.grid * pl.list_cap;
  mp.cnt = cnts;
  mp.cnt_sl = 1;
  mp.cnt_su = pl.grid;
  mp.list_len = pl.list_cap;
  mp.pass = pass;
  mp.pstride_l = 1;
  mp.pstride_u = pl.grid;
  mp.L = pl.grid;
  mp.K = K;
  mp.out_ids = out_ids;
  mp.out_scores = out_scores;
  mp.out_keys = out_keys;
  mp.out_pass = out_pass;
  mp.mode = mode;
  mp.dbg = debug_buffer();
  // one scan launch: its last CTAs run the merge (saves a launch); several: a merge kernel
  // LINR_FUSE_MERGE=1: the last CTAs of a single scan launch run the merge (saves a launch, but the
  // scan kernel then also carries the merge's latency); default: a separate merge kernel, which
  // overlaps the next search's scan when searches are pipelined on two streams
  const char* fe = std::getenv("LINR_FUSE_MERGE");
  const bool fuse_env = fe && std::atoi(fe) != 0;
  const bool fused = pl.groups == 1 && fuse_env;
  for (int g = 0; g < pl.groups; ++g) {
    const int u0 = g * pl.nu_g;
    const int nu = std::min(pl.nu_g, B - u0);
    ScanParams p;
    std::memset(&p, 0, sizeof(p));
    p.emb = ix->emb;
    p.attr = ix->attr;
    p.live = live_ovr ? live_ovr + (size_t)u0 * live_ovr_words : ix->live;
    p.hdr = ix->hdr;
    p.cap_pad = ix->cap_pad;
    p.row0 = (uint32_t)ix->d.global_row0;
    p.nu = nu;
    p.V = V;
    p.K = K;
    p.C = pl.C;
    p.bufcap = pl.bufcap;
    p.list_cap = pl.list_cap;
    p.dbg = debug_buffer();
    p.q = (const char*)q + (size_t)u0 * V * ix->rowbytes;
    const size_t part0 = (size_t)u0 * pl.grid;
    p.out_samp = samp + part0 * kScanSample;
    p.out_list = lists + part0 * pl.list_cap;
    p.out_cnt = cnts + part0;
    p.out_pass = pass + part0;
    uint32_t wmask = 0;
    for (int u = 0; u < nu; ++u) {
      const int b = u0 + u;
      p.ncl[u] = off[b + 1] - off[b];
      for (int c = 0; c < p.ncl[u]; ++c) {
        const linr_clause& k = cl[off[b] + c];
        p.cl[u][c].mask = k.mask;
        p.cl[u][c].word = k.word;
        p.cl[u][c].rev = k.reverse;
        wmask |= 1u << k.word;
      }
    }
    p.wmask = wmask;
    p.fuse_merge = fused ? 1 : 0;
    p.ring = pl.ring;
    p.fuse_slot = fused ? (int)(ix->fuse_seq++ % kFuseSlots) : 0;
    p.mp = mp;
    e = launch_scan_gemv(ix->d.dtype, ix->d.dim, pl.nqv, p, pl.grid, pl.smem, st);
    if (e != cudaSuccess) return cuda_fail(e, "scan launch");
  }
  if (ix->prof) cudaEventRecord(pe.e1, st);
  if (!fused) {
    // LINR_PDL=1: programmatic dependent launch of the merge (saves ~1.3 us of launch gap per serial
    // search, but the early-resident merge CTA costs ~4 % of pipelined throughput: off by default)
    e = launch_merge(mp, B, st, env_int("LINR_PDL", 0) != 0);
    if (e != cudaSuccess) return cuda_fail(e, "merge launch");
  }
  if (ix->prof) {
    cudaEventRecord(pe.e2, st);
    ix->prof_used.push_back(pe);
    ix->prof_launches += pl.groups + (fused ? 0 : 1);
  }
  return LINR_OK;
}

bool desc_ok(const linr_index_desc* d, std::string* why) {
  if (!d) { *why = "null desc"; return false; }
  if (d->capacity_rows < 1) { *why = "capacity_rows must be >= 1"; return false; }
  if (d->global_row0 < 0 || d->global_row0 + d->capacity_rows > 0xFFFFFFFFll) {
    *why = "global ids must be < 2^32-1";
    return false;
  }
  if (d->dtype < LINR_F32 || d->dtype > LINR_I8) { *why = "bad dtype"; return false; }
  if (d->dim < 16 || d->dim % 16) { *why = "dim must be a positive multiple of 16"; return false; }
  if (d->attr_words < 1 || d->attr_words > LINR_MAX_ATTR_WORDS) { *why = "attr_words must be in [1,4]"; return false; }
  return true;
}

}  // namespace

extern "C" {

int linr_version(void) { return 2; }

int linr_debug_timers(int enable) {
  unsigned long long* p = nullptr;
  if (enable) {
    if (!g_dbg_host_ptr && cudaMalloc(&g_dbg_host_ptr, 8192 * 8) != cudaSuccess) return fail(LINR_ECUDA, "dbg alloc");
    cudaMemset(g_dbg_host_ptr, 0, 8192 * 8);
    p = g_dbg_host_ptr;
  }
  g_dbg_on = p != nullptr;
  return LINR_OK;
}

int linr_debug_read(uint64_t* host, int32_t n) {
  if (!g_dbg_host_ptr || !host || n < 0 || n > 8192) return fail(LINR_EINVAL, "debug timers not enabled");
  cudaError_t e = cudaMemcpy(host, g_dbg_host_ptr, (size_t)n * 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "dbg read");
  cudaMemset(g_dbg_host_ptr, 0, 8192 * 8);
  return LINR_OK;
}
const char* linr_last_error(void) { return g_err.c_str(); }

size_t linr_storage_bytes(const linr_index_desc* d, int which) {
  std::string why;
  if (!desc_ok(d, &why)) return 0;
  const int64_t cp = pad_rows(d->capacity_rows);
  switch (which) {
    case 0: return (size_t)cp * d->dim * esize(d->dtype);
    case 1: return (size_t)cp * d->attr_words * 8;
    case 2: return kHdrBytes + (size_t)cp / 32 * 4;
  }
  return 0;
}

int linr_index_create(const linr_index_desc* d, linr_index** out) {
  std::string why;
  if (!out) return fail(LINR_EINVAL, "null out");
  *out = nullptr;
  if (!desc_ok(d, &why)) return fail(LINR_EINVAL, why);
  if (!dim_ok(d->dim)) return fail(LINR_EUNSUPPORTED, "dim must be a power of two in [16, 1024]");
  if (!d->emb_storage || !d->attr_storage || !d->live_storage) return fail(LINR_EINVAL, "null storage");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (d->device < 0 || d->device >= ndev) return fail(LINR_EINVAL, "bad device");
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d->device);
  linr_index* ix = new (std::nothrow) linr_index;
  if (!ix) return fail(LINR_ENOMEM, "host allocation");
  ix->d = *d;
  ix->cap_pad = pad_rows(d->capacity_rows);
  ix->rowbytes = d->dim * esize(d->dtype);
  ix->num_sms = sms;
  ix->smem_optin = (size_t)optin;
  ix->emb = d->emb_storage;
  ix->attr = (uint64_t*)d->attr_storage;
  ix->hdr = (DevHeader*)d->live_storage;
  ix->live = (uint32_t*)((char*)d->live_storage + kHdrBytes);
  if (const char* gf = std::getenv("LINR_L2_FETCH")) {
    // tuning knob: the L2's maximum DRAM fetch granularity (bytes; a device-wide hint). The row
    // gather touches isolated short rows (64 B int8 d = 64), so a coarse fetch wastes traffic.
    DeviceGuard g(d->device);
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)std::atoi(gf));
  }
  *out = ix;
  return LINR_OK;
}

void linr_index_destroy(linr_index* ix) {
  if (!ix) return;
  if (ix->comm) comm_destroy(ix->comm);
  for (auto& ps : ix->pin) {
    if (ps.ev) {
      cudaEventSynchronize(ps.ev);
      cudaEventDestroy(ps.ev);
    }
    if (ps.p) cudaFreeHost(ps.p);
  }
  for (auto* v : {&ix->prof_used, &ix->prof_free})
    for (auto& pe : *v) {
      cudaEventDestroy(pe.e0);
      cudaEventDestroy(pe.e1);
      cudaEventDestroy(pe.e2);
    }
  delete ix;
}

int linr_index_profile(linr_index* ix, int enable) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  ix->prof = enable != 0;
  return LINR_OK;
}

int linr_index_profile_read(linr_index* ix, double* scan_ms, double* merge_ms, int64_t* searches,
                            int64_t* launches) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  DeviceGuard dg(ix->d.device);
  double s = 0.0, m = 0.0;
  for (auto& pe : ix->prof_used) {
    cudaError_t e = cudaEventSynchronize(pe.e2);
    if (e != cudaSuccess) return cuda_fail(e, "profile events");
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, pe.e0, pe.e1);
    cudaEventElapsedTime(&b, pe.e1, pe.e2);
    s += a;
    m += b;
  }
  if (scan_ms) *scan_ms = s;
  if (merge_ms) *merge_ms = m;
  if (searches) *searches = (int64_t)ix->prof_used.size();
  if (launches) *launches = ix->prof_launches;
  for (auto& pe : ix->prof_used) ix->prof_free.push_back(pe);
  ix->prof_used.clear();
  ix->prof_launches = 0;
  return LINR_OK;
}

int linr_index_load(linr_index* ix, int64_t row0, int64_t n, const void* emb, const uint64_t* attrs, void* stream) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (n < 0) return fail(LINR_EINVAL, "n < 0");
  if (n == 0) return LINR_OK;
  if (!emb || !attrs) return fail(LINR_EINVAL, "null input");
  const int64_t r0 = row0 - ix->d.global_row0;
  if (r0 < 0 || r0 + n > ix->d.capacity_rows) return fail(LINR_ERANGE, "rows outside this shard");
  DeviceGuard dg(ix->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync((char*)ix->emb + r0 * ix->rowbytes, emb, (size_t)n * ix->rowbytes,
                                  cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "load emb copy");
  e = launch_attr_soa(attrs, n, ix->d.attr_words, ix->attr, ix->cap_pad, r0, st);
  if (e != cudaSuccess) return cuda_fail(e, "load attrs");
  e = launch_set_live_range(ix->live, ix->hdr, r0, n, st);
  if (e != cudaSuccess) return cuda_fail(e, "load live");
  if (ix->codes) {   // keep the 1-bit codes in step with the rows (quantised embedding per item)
    e = launch_oporp_encode(ix->d.dtype, ix->emb, ix->d.dim, n, r0, nullptr, 0, ix->d.capacity_rows, ix->code_k,
                            ix->code_L, ix->c_src, ix->c_sign, ix->codes, st);
    if (e != cudaSuccess) return cuda_fail(e, "load encode");
  }
  if (ix->scorer) {   // learned-scorer item features follow the rows
    e = launch_features(ix->d.dtype, ix->emb, ix->d.dim, n, r0, nullptr, 0, ix->d.capacity_rows, ix->sw.M, ix->sw.Mb,
                        ix->sw.Fm, ix->sw.Fp, ix->sy, st);
    if (e != cudaSuccess) return cuda_fail(e, "load features");
  }
  return LINR_OK;
}

int linr_index_update_rows(linr_index* ix, const int64_t* rows, int64_t n, const void* emb, const uint64_t* attrs,
                           void* stream) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (n < 0) return fail(LINR_EINVAL, "n < 0");
  if (n == 0) return LINR_OK;
  if (!rows || !emb || !attrs) return fail(LINR_EINVAL, "null input");
  DeviceGuard dg(ix->d.device);
  cudaError_t e = launch_update_rows(rows, n, ix->d.global_row0, ix->d.capacity_rows, ix->rowbytes, emb, attrs,
                                     ix->d.attr_words, ix->emb, ix->attr, ix->cap_pad, ix->live, ix->hdr,
                                     (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "update launch");
  if (ix->codes) {   // re-encode the overwritten rows (after the update on the same stream)
    e = launch_oporp_encode(ix->d.dtype, ix->emb, ix->d.dim, n, 0, rows, ix->d.global_row0, ix->d.capacity_rows,
                            ix->code_k, ix->code_L, ix->c_src, ix->c_sign, ix->codes, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "update encode");
  }
  if (ix->scorer) {
    e = launch_features(ix->d.dtype, ix->emb, ix->d.dim, n, 0, rows, ix->d.global_row0, ix->d.capacity_rows, ix->sw.M,
                        ix->sw.Mb, ix->sw.Fm, ix->sw.Fp, ix->sy, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "update features");
  }
  return LINR_OK;
}

int linr_index_delete_rows(linr_index* ix, const int64_t* rows, int64_t n, void* stream) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (n < 0) return fail(LINR_EINVAL, "n < 0");
  if (n == 0) return LINR_OK;
  if (!rows) return fail(LINR_EINVAL, "null rows");
  DeviceGuard dg(ix->d.device);
  cudaError_t e = launch_delete_rows(rows, n, ix->d.global_row0, ix->d.capacity_rows, ix->live, ix->hdr,
                                     (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "delete launch");
  return LINR_OK;
}

int linr_index_stats(linr_index* ix, int64_t* hwm, int64_t* skipped, int64_t* overflow, void* stream) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  DeviceGuard dg(ix->d.device);
  DevHeader h;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(&h, ix->hdr, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "stats");
  if (hwm) *hwm = (int64_t)h.hwm;
  if (skipped) *skipped = (int64_t)h.skipped;
  if (overflow) *overflow = (int64_t)h.overflow;
  return LINR_OK;
}

int linr_index_counters(linr_index* ix, linr_counters* out, void* stream) {
  if (!ix || !out) return fail(LINR_EINVAL, "null argument");
  DeviceGuard dg(ix->d.device);
  DevHeader h;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(&h, ix->hdr, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "counters");
  out->hwm = (int64_t)h.hwm;
  out->skipped = (int64_t)h.skipped;
  out->scan_overflow = (int64_t)h.overflow;
  out->tc_fallbacks = (int64_t)h.tc_fallbacks;
  return LINR_OK;
}

static size_t local_ws_bytes(const linr_index* ix, int32_t B, int32_t V, int32_t K);

// exchange buffers of a sharded search: send [B*(K+1)] u64, receive [world][B*(K+1)] u64
static size_t comm_ws_bytes(const linr_index* ix, int32_t B, int32_t K) {
  if (!ix->comm) return 0;
  const size_t per = (size_t)B * (K + 1) * 8;
  return align256(per) + align256(per * ix->comm_world);
}

size_t linr_search_workspace_bytes(const linr_index* ix, int32_t B, int32_t V, int32_t K) {
  const size_t n = local_ws_bytes(ix, B, V, K);
  if (n == 0) return 0;
  return ix->comm ? align256(n) + comm_ws_bytes(ix, B, K) : n;
}

static size_t local_ws_bytes(const linr_index* ix, int32_t B, int32_t V, int32_t K) {
  if (!ix || B < 1 || V < 1 || V > 8 || K < 1 || K > LINR_MAX_K) return 0;
  Plan pl;
  std::string why;
  size_t n = 0;
  if (use_tc(ix, B, V, 0, 1) || use_tc_nopass(ix, B, V, 0, 1)) {   // clause-light bound: the batched path may be taken
    TcWs w;
    if (tc_layout(ix, B, V, K, &w, &why)) n = w.end;
  }
  if (make_plan(ix, B, V, K, &pl, &why)) n = std::max(n, ws_layout(pl, B, K).end);
  if (union_ok(ix, B, V, 0, 1)) {   // clause-light bound, as for the batched path
    Plan up;
    n = std::max(n, union_ws_bytes(ix, B, V, K, &up));
  }
  return n;
}

// With a communicator attached: shard-local keys + pass counts packed into one send buffer, one
// ncclAllGather, one merge (every rank receives the global result). Without: the local search.
static int search_global(linr_index* ix, const void* q, int32_t B, int32_t V, const linr_clause* cl,
                         const int32_t* off, int32_t K, void* ws, size_t ws_bytes, int64_t* out_ids,
                         float* out_scores, int64_t* out_pass, cudaStream_t st) {
  if (!ix || !ix->comm)
    return search_impl(ix, q, B, V, cl, off, K, ws, ws_bytes, 0, out_ids, out_scores, nullptr, out_pass, st);
  if (!out_ids || !out_scores) return fail(LINR_EINVAL, "null outputs");
  const size_t local = local_ws_bytes(ix, B, V, K);
  if (local == 0) return fail(LINR_EINVAL, "bad B/V/K");
  if (!ws || ws_bytes < align256(local) + comm_ws_bytes(ix, B, K)) return fail(LINR_ENOMEM, "workspace too small");
  const size_t per = (size_t)B * (K + 1);
  uint64_t* send = (uint64_t*)((char*)ws + align256(local));
  uint64_t* recv = (uint64_t*)((char*)send + align256(per * 8));
  int rc = search_impl(ix, q, B, V, cl, off, K, ws, local, 1, nullptr, nullptr, send, (int64_t*)(send + (size_t)B * K),
                       st);
  if (rc != LINR_OK) return rc;
  DeviceGuard dg(ix->d.device);
  rc = comm_allgather_u64(ix->comm, send, recv, per, st);
  if (rc != LINR_OK) return rc;
  MergeParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.samp = recv;            // each rank's list is sorted: its first min(K, 32) keys are its sample
  mp.samp_sl = (int64_t)per;
  mp.samp_su = K;
  mp.ms = std::min(K, kScanSample);
  mp.list = recv;
  mp.list_sl = (int64_t)per;
  mp.list_su = K;
  mp.list_len = K;
  mp.pass = (const int64_t*)(recv + (size_t)B * K);
  mp.pstride_l = (int64_t)per;
  mp.pstride_u = 1;
  mp.L = ix->comm_world;
  mp.K = K;
  mp.out_ids = out_ids;
  mp.out_scores = out_scores;
  mp.out_pass = out_pass;
  mp.mode = 0;
  mp.dbg = debug_buffer();
  cudaError_t e = launch_merge(mp, B, st);
  if (e != cudaSuccess) return cuda_fail(e, "shard merge launch");
  return LINR_OK;
}

int linr_search(linr_index* ix, const void* q, int32_t B, int32_t V, const linr_clause* cl, const int32_t* off,
                int32_t K, void* ws, size_t ws_bytes, int64_t* out_ids, float* out_scores, int64_t* out_pass,
                void* stream) {
  return search_global(ix, q, B, V, cl, off, K, ws, ws_bytes, out_ids, out_scores, out_pass, (cudaStream_t)stream);
}

int linr_comm_init(linr_index* ix, const uint8_t* id, int32_t rank, int32_t world) {
  if (!ix || !id) return fail(LINR_EINVAL, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(LINR_EINVAL, "bad rank/world");
  if (ix->comm) return fail(LINR_EINVAL, "a communicator is already attached");
  void* c = nullptr;
  const int rc = comm_create(ix->d.device, id, rank, world, &c);
  if (rc != LINR_OK) return rc;
  ix->comm = c;
  ix->comm_rank = rank;
  ix->comm_world = world;
  return LINR_OK;
}

int linr_search_keys(linr_index* ix, const void* q, int32_t B, int32_t V, const linr_clause* cl,
                     const int32_t* off, int32_t K, void* ws, size_t ws_bytes, uint64_t* out_keys,
                     int64_t* out_pass, void* stream) {
  return search_impl(ix, q, B, V, cl, off, K, ws, ws_bytes, 1, nullptr, nullptr, out_keys, out_pass,
                     (cudaStream_t)stream);
}

size_t linr_merge_workspace_bytes(int32_t L, int32_t B, int32_t K) {
  if (L < 1 || B < 1 || K < 1 || K > LINR_MAX_K) return 0;
  return 0;   // the merge kernel works entirely in shared memory
}

int linr_merge_keys(const uint64_t* keys, const int64_t* pass, int32_t L, int32_t B, int32_t K, void* ws,
                    size_t ws_bytes, int64_t* out_ids, float* out_scores, int64_t* out_pass, void* stream) {
  (void)ws;
  (void)ws_bytes;
  if (!keys || !pass || !out_ids || !out_scores) return fail(LINR_EINVAL, "null pointer");
  if (L < 1 || B < 1 || K < 1 || K > LINR_MAX_K) return fail(LINR_EINVAL, "bad L/B/K");
  if ((int64_t)L * K > 0x7FFFFFFF) return fail(LINR_EINVAL, "L*K too large");
  // shard lists are fully sorted: sample = their first min(32, K) keys, list = the whole list
  MergeParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.samp = keys;
  mp.samp_sl = (int64_t)B * K;
  mp.samp_su = K;
  mp.ms = std::min(K, kScanSample);
  mp.list = keys;
  mp.list_sl = (int64_t)B * K;
  mp.list_su = K;
  mp.cnt = nullptr;
  mp.list_len = K;
  mp.pass = pass;
  mp.pstride_l = B;
  mp.pstride_u = 1;
  mp.L = L;
  mp.K = K;
  mp.out_ids = out_ids;
  mp.out_scores = out_scores;
  mp.out_pass = out_pass;
  mp.mode = 0;
  mp.dbg = debug_buffer();
  cudaError_t e = launch_merge(mp, B, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "merge launch");
  return LINR_OK;
}

size_t linr_search_host_extra_bytes(const linr_index* ix, int32_t B, int32_t V, int32_t K) {
  if (!ix || B < 1 || V < 1 || K < 1) return 0;
  return align256((size_t)B * V * ix->rowbytes) + align256((size_t)B * K * 8) + align256((size_t)B * K * 4) +
         align256((size_t)B * 8);
}

static int search_host_impl(linr_index* ix, const void* q_host, int32_t B, int32_t V, const linr_clause* cl,
                            const int32_t* off, int32_t K, void* ws, size_t ws_bytes, int64_t* ids_host,
                            float* scores_host, int64_t* pass_host, void* stream, bool sync);

int linr_search_host(linr_index* ix, const void* q_host, int32_t B, int32_t V, const linr_clause* cl,
                     const int32_t* off, int32_t K, void* ws, size_t ws_bytes, int64_t* ids_host,
                     float* scores_host, int64_t* pass_host, void* stream) {
  return search_host_impl(ix, q_host, B, V, cl, off, K, ws, ws_bytes, ids_host, scores_host, pass_host, stream,
                          true);
}

int linr_search_host_async(linr_index* ix, const void* q_host, int32_t B, int32_t V, const linr_clause* cl,
                           const int32_t* off, int32_t K, void* ws, size_t ws_bytes, int64_t* ids_host,
                           float* scores_host, int64_t* pass_host, void* stream) {
  return search_host_impl(ix, q_host, B, V, cl, off, K, ws, ws_bytes, ids_host, scores_host, pass_host, stream,
                          false);
}

static int search_host_impl(linr_index* ix, const void* q_host, int32_t B, int32_t V, const linr_clause* cl,
                            const int32_t* off, int32_t K, void* ws, size_t ws_bytes, int64_t* ids_host,
                            float* scores_host, int64_t* pass_host, void* stream, bool sync) {
  if (!ix || !q_host || !ids_host || !scores_host) return fail(LINR_EINVAL, "null pointer");
  const size_t need = linr_search_workspace_bytes(ix, B, V, K);
  const size_t extra = linr_search_host_extra_bytes(ix, B, V, K);
  if (need == 0 || extra == 0) return fail(LINR_EINVAL, "bad B/V/K");
  if (!ws || ws_bytes < need + extra) return fail(LINR_ENOMEM, "workspace too small");
  DeviceGuard dg(ix->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  char* x = (char*)ws + align256(need);
  void* qd = x;
  x += align256((size_t)B * V * ix->rowbytes);
  int64_t* idd = (int64_t*)x;
  x += align256((size_t)B * K * 8);
  float* scd = (float*)x;
  x += align256((size_t)B * K * 4);
  int64_t* psd = (int64_t*)x;
  if (ws_bytes < align256(need) + extra) return fail(LINR_ENOMEM, "workspace too small");
  cudaError_t e = cudaMemcpyAsync(qd, q_host, (size_t)B * V * ix->rowbytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "query H2D");
  // pass counts only when the caller asks (on the batched path they cost a clause evaluation per
  // (row, user): 7 ms at B = 256 over 10M rows)
  int rc = search_global(ix, qd, B, V, cl, off, K, ws, need, idd, scd, pass_host ? psd : nullptr, st);
  if (rc != LINR_OK) return rc;
  e = cudaMemcpyAsync(ids_host, idd, (size_t)B * K * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(scores_host, scd, (size_t)B * K * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && pass_host) e = cudaMemcpyAsync(pass_host, psd, (size_t)B * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && sync) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "search_host copies");
  return LINR_OK;
}

int linr_index_generate(linr_index* ix, uint64_t seed, int32_t mode, int64_t row_begin, int64_t n, void* stream) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (mode != 0 && mode != 1) return fail(LINR_EINVAL, "mode must be 0 or 1");
  if (n < 0 || row_begin < 0 || row_begin + n > ix->d.capacity_rows) return fail(LINR_ERANGE, "rows outside shard");
  if (n == 0) return LINR_OK;
  DeviceGuard dg(ix->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  // counters are GLOBAL row ids, so every shard of a sharded index generates consistent rows
  cudaError_t e = launch_generate(ix->d.dtype, ix->d.dim, ix->d.attr_words, seed, mode,
                                  ix->d.global_row0 + row_begin, n, (char*)ix->emb, row_begin, ix->attr,
                                  ix->cap_pad, true, st);
  if (e != cudaSuccess) return cuda_fail(e, "generate");
  e = launch_set_live_range(ix->live, ix->hdr, row_begin, n, st);
  if (e != cudaSuccess) return cuda_fail(e, "generate live");
  if (ix->codes) {
    e = launch_oporp_encode(ix->d.dtype, ix->emb, ix->d.dim, n, row_begin, nullptr, 0, ix->d.capacity_rows,
                            ix->code_k, ix->code_L, ix->c_src, ix->c_sign, ix->codes, st);
    if (e != cudaSuccess) return cuda_fail(e, "generate encode");
  }
  if (ix->scorer) {
    e = launch_features(ix->d.dtype, ix->emb, ix->d.dim, n, row_begin, nullptr, 0, ix->d.capacity_rows, ix->sw.M,
                        ix->sw.Mb, ix->sw.Fm, ix->sw.Fp, ix->sy, st);
    if (e != cudaSuccess) return cuda_fail(e, "generate features");
  }
  return LINR_OK;
}

int linr_generate_rows(int32_t dtype, int32_t dim, int32_t W, uint64_t seed, int32_t mode, int64_t row_begin,
                       int64_t n, void* emb, uint64_t* attrs, void* stream) {
  if (dtype < 0 || dtype > 3 || dim < 1 || W < 1 || W > 4 || n < 0 || (mode != 0 && mode != 1))
    return fail(LINR_EINVAL, "bad generator arguments");
  if (n == 0) return LINR_OK;
  cudaError_t e = launch_generate(dtype, dim, W, seed, mode, row_begin, n, emb, 0, attrs, 0, false,
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "generate");
  return LINR_OK;
}


// ------------------------------------------------------------------ quantised path (codes.cu)
static bool oporp_ok(const linr_index* ix, const linr_oporp_params* pr, std::string* why) {
  if (!ix || !pr) { *why = "null argument"; return false; }
  if (pr->bits < 64 || pr->bits > 1024 || pr->bits % 64 || ((pr->bits / 64) & (pr->bits / 64 - 1))) {
    *why = "bits must be 64, 128, 256, 512 or 1024";
    return false;
  }
  if (pr->L < pr->bits || pr->L % pr->bits || !pr->src_host || !pr->sign_host) { *why = "L must be a multiple of bits"; return false; }
  for (int p = 0; p < pr->L; ++p) {
    if (pr->src_host[p] < -1 || pr->src_host[p] >= ix->d.dim) { *why = "src entry outside [-1, dim)"; return false; }
    if (pr->sign_host[p] != 1 && pr->sign_host[p] != -1) { *why = "sign entry not +-1"; return false; }
  }
  return true;
}

size_t linr_codes_storage_bytes(const linr_index* ix, const linr_oporp_params* pr) {
  std::string why;
  if (!oporp_ok(ix, pr, &why)) return 0;
  return align256((size_t)ix->cap_pad * (pr->bits / 64) * 8) + align256((size_t)pr->L * 4) + align256((size_t)pr->L);
}

int linr_codes_attach(linr_index* ix, const linr_oporp_params* pr, void* storage, void* stream) {
  std::string why;
  if (!oporp_ok(ix, pr, &why)) return fail(LINR_EINVAL, why);
  if (!storage) return fail(LINR_EINVAL, "null storage");
  if (ix->codes) return fail(LINR_EINVAL, "codes already attached");
  DeviceGuard dg(ix->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  char* b = (char*)storage;
  uint64_t* codes = (uint64_t*)b;
  int32_t* src = (int32_t*)(b + align256((size_t)ix->cap_pad * (pr->bits / 64) * 8));
  int8_t* sign = (int8_t*)((char*)src + align256((size_t)pr->L * 4));
  DevHeader h;
  cudaError_t e = cudaStreamSynchronize(st);   // setup call: the rows to encode are those below the hwm now
  if (e == cudaSuccess) e = cudaMemcpy(&h, ix->hdr, sizeof(h), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(src, pr->src_host, (size_t)pr->L * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(sign, pr->sign_host, (size_t)pr->L, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "codes attach");
  ix->codes = codes;
  ix->code_k = pr->bits;
  ix->code_L = pr->L;
  ix->c_src = src;
  ix->c_sign = sign;
  e = launch_oporp_encode(ix->d.dtype, ix->emb, ix->d.dim, (int64_t)h.hwm, 0, nullptr, 0, ix->d.capacity_rows, ix->code_k,
                          ix->code_L, src, sign, codes, st);
  if (e != cudaSuccess) return cuda_fail(e, "codes encode");
  return LINR_OK;
}

int linr_oporp_encode(const linr_index* ix, const void* x, int64_t n, uint64_t* out, void* stream) {
  if (!ix || !x || !out || n < 0) return fail(LINR_EINVAL, "bad argument");
  if (!ix->codes) return fail(LINR_EINVAL, "no codes attached");
  if (n == 0) return LINR_OK;
  DeviceGuard dg(ix->d.device);
  cudaError_t e = launch_oporp_encode(ix->d.dtype, x, ix->d.dim, n, 0, nullptr, 0, n, ix->code_k, ix->code_L, ix->c_src,
                                      ix->c_sign, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "encode");
  return LINR_OK;
}

namespace {
constexpr int kCodeWarps = 16;   // warps per code-scan CTA (codes.cu kCodeNW)

struct CodeWs {
  size_t q, cl, kept, pass, mstar, T, H, off, marr, tmax, cand, lists, above, end;
  int g;   // users per launch group
};

int code_group(const linr_index* ix, int B, int V) {
  const int K1 = ix->code_k + 1;
  int g = std::min(B, kCodeMaxUsers);
  while (g > 1 && (code_hist_smem(g, V, ix->code_k) > ix->smem_optin ||
                   (size_t)kCodeWarps * 3072 + (size_t)kCodeWarps * g * K1 * 4 > ix->smem_optin))
    --g;
  return g;
}

CodeWs code_layout(const linr_index* ix, int B, int V, int64_t K, bool v3) {
  CodeWs w;
  const int g = code_group(ix, B, V);
  const size_t GW = (size_t)ix->num_sms * kCodeWarps, K1 = (size_t)ix->code_k + 1, words = ix->code_k / 64;
  const size_t msz = ix->code_k <= 192 ? 1 : 2;
  w.g = g;
  w.q = 0;
  w.cl = align256((size_t)B * V * words * 8);
  w.kept = w.cl + align256((size_t)B * 16 * sizeof(KClause) + (size_t)B * 4);
  w.pass = w.kept + align256((size_t)B * 8);
  w.mstar = w.pass + align256((size_t)B * 8);
  w.T = w.mstar + align256((size_t)g * 4);          // T [g][K1] u64 followed by the ticket (one memset)
  w.above = w.T + align256((size_t)g * K1 * 8 + 8);
  w.H = w.above + align256((size_t)g * (K1 + 1) * 8);
  w.off = w.H + align256((size_t)g * GW * K1 * 4);
  w.marr = w.off + align256((size_t)g * GW * K1 * 4);
  w.tmax = w.marr + align256((size_t)g * ix->cap_pad * msz);
  w.cand = w.tmax + align256((size_t)g * (ix->cap_pad / 256) * 2);
  w.lists = w.cand + (v3 ? align256((size_t)g * ix->cap_pad * 4) : 0);
  w.end = w.lists + (v3 ? align256((size_t)ix->num_sms * g * K * 8) : 0);
  return w;
}

// the shared pipeline: query codes + clause table staged once; per user group: pass 1, offsets,
// pass 2 (ids/m for the code search, kept rows for V3), and for V3 the rerank + merge.
int code_pipeline(linr_index* ix, const void* q, int B, int V, const linr_clause* cl, const int32_t* off, int64_t K,
                  double keep, void* ws, size_t ws_bytes, int64_t* out_ids, int32_t* out_m, float* out_scores,
                  int64_t* out_pass, int64_t* out_kept, cudaStream_t st) {
  std::string why;
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (!ix->codes) return fail(LINR_EINVAL, "no codes attached (linr_codes_attach)");
  int rc = validate_query(ix, q, B, V, cl, off, 1, &why);
  if (rc != LINR_OK) return fail(rc, why);
  const bool v3 = keep > 0.0;
  if (K < 1 || (v3 && K > LINR_MAX_K)) return fail(LINR_EINVAL, v3 ? "K must be in [1, 2048]" : "K must be >= 1");
  if (v3 && !(keep <= 1.0)) return fail(LINR_EINVAL, "keep must be in (0, 1]");
  if (!out_ids || (!v3 && !out_m) || (v3 && !out_scores)) return fail(LINR_EINVAL, "null outputs");
  const CodeWs w = code_layout(ix, B, V, K, v3);
  if (!ws || ws_bytes < w.end) return fail(LINR_ENOMEM, "workspace too small");
  DeviceGuard dg(ix->d.device);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pending CUDA error");
  char* W = (char*)ws;
  const int words = ix->code_k / 64, K1 = ix->code_k + 1, GW = ix->num_sms * kCodeWarps;
  const size_t msz = ix->code_k <= 192 ? 1 : 2;
  uint64_t* qc = (uint64_t*)(W + w.q);
  e = launch_oporp_encode(ix->d.dtype, q, ix->d.dim, (int64_t)B * V, 0, nullptr, 0, (int64_t)B * V, ix->code_k,
                          ix->code_L, ix->c_src, ix->c_sign, qc, st);
  if (e != cudaSuccess) return cuda_fail(e, "query encode");
  rc = stage_clause_table(ix, cl, off, B, W + w.cl, st);
  if (rc != LINR_OK) return rc;
  const KClause* dcl = (const KClause*)(W + w.cl);
  const int* dncl = (const int*)(W + w.cl + (size_t)B * 16 * sizeof(KClause));
  int64_t* kept = (int64_t*)(W + w.kept);
  int64_t* pass = out_pass ? out_pass : (int64_t*)(W + w.pass);
  for (int u0 = 0; u0 < B; u0 += w.g) {
    const int g = std::min(w.g, B - u0);
    uint32_t wmask = 0;
    for (int b = u0; b < u0 + g; ++b)
      for (int c = off[b]; c < off[b + 1]; ++c) wmask |= 1u << cl[c].word;
    e = cudaMemsetAsync(W + w.T, 0, (size_t)g * K1 * 8 + 8, st);
    if (e != cudaSuccess) return cuda_fail(e, "code totals reset");
    CodeScanParams sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.codes = ix->codes;
    sp.attr = ix->attr;
    sp.cap_pad = ix->cap_pad;
    sp.live = ix->live;
    sp.hdr = ix->hdr;
    sp.nu = g;
    sp.V = V;
    sp.qcodes = qc + (size_t)u0 * V * words;
    sp.cl = dcl + (size_t)u0 * 16;
    sp.ncl = dncl + u0;
    sp.wmask = wmask;
    sp.marr = W + w.marr;
    sp.tmax = (uint16_t*)(W + w.tmax);
    sp.tmax_stride = ix->cap_pad / 256;
    sp.H = (uint32_t*)(W + w.H);
    sp.T = (unsigned long long*)(W + w.T);
    sp.ticket = (unsigned int*)(W + w.T + (size_t)g * K1 * 8);
    sp.K = K;
    sp.keep = keep;
    sp.mstar = (int*)(W + w.mstar);
    sp.kept = kept + u0;
    sp.pass = pass + u0;
    sp.above = (unsigned long long*)(W + w.above);
    ProfEvents pe{};
    if (ix->prof) {   // stage timing: pass 1 (the dominant kernel) vs the rest of the pipeline
      if (!ix->prof_free.empty()) {
        pe = ix->prof_free.back();
        ix->prof_free.pop_back();
      } else {
        cudaEventCreate(&pe.e0);
        cudaEventCreate(&pe.e1);
        cudaEventCreate(&pe.e2);
      }
      cudaEventRecord(pe.e0, st);
    }
    e = launch_code_hist(ix->code_k, sp, ix->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "code pass 1 launch");
    if (ix->prof) cudaEventRecord(pe.e1, st);
    CodeOffsetParams op;
    op.H = sp.H;
    op.above = sp.above;
    op.mstar = sp.mstar;
    op.GW = GW;
    op.k = ix->code_k;
    op.off = (uint32_t*)(W + w.off);
    e = launch_code_offsets(op, g, st);
    if (e != cudaSuccess) return cuda_fail(e, "code offsets launch");
    CodeEmitParams ep;
    std::memset(&ep, 0, sizeof(ep));
    ep.marr = W + w.marr;
    ep.tmax = sp.tmax;
    ep.tmax_stride = sp.tmax_stride;
    ep.hdr = ix->hdr;
    ep.cap_pad = ix->cap_pad;
    ep.row0 = (uint32_t)ix->d.global_row0;
    ep.nu = g;
    ep.off = op.off;
    ep.mstar = sp.mstar;
    ep.kept = sp.kept;
    if (v3) {
      ep.out_stride = ix->cap_pad;
      ep.cand = (uint32_t*)(W + w.cand);
    } else {
      ep.out_stride = K;
      ep.out_ids = out_ids + (size_t)u0 * K;
      ep.out_m = out_m + (size_t)u0 * K;
    }
    e = launch_code_emit(ix->code_k, ep, ix->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "code pass 2 launch");
    if (!v3) {
      e = launch_code_pad(sp.kept, g, K, ep.out_ids, ep.out_m, ix->num_sms * 4, st);
      if (e != cudaSuccess) return cuda_fail(e, "code pad launch");
      if (ix->prof) {
        cudaEventRecord(pe.e2, st);
        ix->prof_used.push_back(pe);
        ix->prof_launches += 4;   // pass 1, offsets, pass 2, pad
      }
      continue;
    }
    RerankParams rp;
    std::memset(&rp, 0, sizeof(rp));
    rp.emb = ix->emb;
    rp.row0 = (uint32_t)ix->d.global_row0;
    rp.dim = ix->d.dim;
    rp.V = V;
    rp.K = (int)K;
    rp.nu = g;
    rp.q = (const char*)q + (size_t)u0 * V * ix->rowbytes;
    rp.cand = ep.cand;
    rp.cand_stride = ix->cap_pad;
    rp.kept = sp.kept;
    rp.lists = (uint64_t*)(W + w.lists);
    e = launch_rerank(ix->d.dtype, rp, ix->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "rerank launch");
    MergeParams mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.samp = rp.lists;                 // [cta][u][K], each list sorted: its first keys are its sample
    mp.samp_sl = (int64_t)g * K;
    mp.samp_su = K;
    mp.ms = (int)std::min<int64_t>(K, kScanSample);
    mp.list = rp.lists;
    mp.list_sl = (int64_t)g * K;
    mp.list_su = K;
    mp.list_len = (int)K;
    mp.L = ix->num_sms;
    mp.K = (int)K;
    mp.out_ids = out_ids + (size_t)u0 * K;
    mp.out_scores = out_scores + (size_t)u0 * K;
    mp.mode = 0;
    mp.dbg = debug_buffer();
    e = launch_merge(mp, g, st);
    if (e != cudaSuccess) return cuda_fail(e, "rerank merge launch");
    if (ix->prof) {
      cudaEventRecord(pe.e2, st);
      ix->prof_used.push_back(pe);
      ix->prof_launches += 5;   // pass 1, offsets, pass 2, rerank, merge
    }
  }
  if (ix->prof) ix->prof_launches += 1;   // the query encoding
  if (out_kept) {
    e = cudaMemcpyAsync(out_kept, kept, (size_t)B * 8, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "kept copy");
  }
  (void)msz;
  return LINR_OK;
}
}  // namespace

size_t linr_code_search_workspace_bytes(const linr_index* ix, int32_t B, int32_t V, int64_t K, int32_t v3) {
  if (!ix || !ix->codes || B < 1 || V < 1 || V > LINR_MAX_V || K < 1) return 0;
  if (v3 && K > LINR_MAX_K) return 0;
  return code_layout(ix, B, V, K, v3 != 0).end;
}

int linr_code_search(linr_index* ix, const void* q, int32_t B, int32_t V, const linr_clause* cl, const int32_t* off,
                     int64_t K, void* ws, size_t ws_bytes, int64_t* out_ids, int32_t* out_matched, int64_t* out_pass,
                     void* stream) {
  return code_pipeline(ix, q, B, V, cl, off, K, 0.0, ws, ws_bytes, out_ids, out_matched, nullptr, out_pass, nullptr,
                       (cudaStream_t)stream);
}

int linr_search_v3(linr_index* ix, const void* q, int32_t B, int32_t V, const linr_clause* cl, const int32_t* off,
                   int32_t K, double keep, void* ws, size_t ws_bytes, int64_t* out_ids, float* out_scores,
                   int64_t* out_pass, int64_t* out_kept, void* stream) {
  if (!(keep > 0.0)) return fail(LINR_EINVAL, "keep must be in (0, 1]");
  return code_pipeline(ix, q, B, V, cl, off, K, keep, ws, ws_bytes, out_ids, nullptr, out_scores, out_pass, out_kept,
                       (cudaStream_t)stream);
}


// ------------------------------------------------------------------ ID-list clauses (idlist.cu)
static bool idl_desc_ok(int32_t slots, const int32_t* widths, std::string* why) {
  if (slots < 1 || slots > LINR_MAX_ID_SLOTS || !widths) { *why = "slots must be in [1, 4]"; return false; }
  for (int s = 0; s < slots; ++s)
    if (widths[s] < 1 || widths[s] > LINR_MAX_IDS_PER_ITEM) { *why = "width must be in [1, 16]"; return false; }
  return true;
}

size_t linr_idlists_storage_bytes(const linr_index* ix, int32_t slots, const int32_t* widths) {
  std::string why;
  if (!ix || !idl_desc_ok(slots, widths, &why)) return 0;
  size_t A = 0;
  for (int s = 0; s < slots; ++s) A += widths[s];
  return align256(A * ix->cap_pad * 8) + align256((size_t)slots * ix->cap_pad);
}

int linr_idlists_attach(linr_index* ix, int32_t slots, const int32_t* widths, void* storage) {
  std::string why;
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (!idl_desc_ok(slots, widths, &why)) return fail(LINR_EINVAL, why);
  if (!storage) return fail(LINR_EINVAL, "null storage");
  if (ix->idl_ids) return fail(LINR_EINVAL, "ID lists already attached");
  DeviceGuard dg(ix->d.device);
  size_t A = 0;
  for (int s = 0; s < slots; ++s) {
    ix->idl_A[s] = widths[s];
    ix->idl_off[s] = (int)A;
    A += widths[s];
  }
  ix->idl_S = slots;
  ix->idl_ids = (uint64_t*)storage;
  ix->idl_cnt = (uint8_t*)((char*)storage + align256(A * ix->cap_pad * 8));
  cudaError_t e = cudaMemset(ix->idl_cnt, 0, (size_t)slots * ix->cap_pad);   // setup: no row has ids yet
  if (e != cudaSuccess) return cuda_fail(e, "ID-list init");
  return LINR_OK;
}

int linr_idlists_set_rows(linr_index* ix, int32_t slot, const int64_t* rows, int64_t row0, int64_t n,
                          const uint64_t* ids, const uint8_t* counts, void* stream) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (!ix->idl_ids) return fail(LINR_EINVAL, "no ID lists attached");
  if (slot < 0 || slot >= ix->idl_S) return fail(LINR_EINVAL, "bad slot");
  if (n < 0) return fail(LINR_EINVAL, "n < 0");
  if (n == 0) return LINR_OK;
  if (!ids || !counts) return fail(LINR_EINVAL, "null input");
  const int64_t r0 = row0 - ix->d.global_row0;
  if (!rows && (r0 < 0 || r0 + n > ix->d.capacity_rows)) return fail(LINR_ERANGE, "rows outside this shard");
  DeviceGuard dg(ix->d.device);
  cudaError_t e = launch_idl_set_rows(rows, r0, ix->d.global_row0, ix->d.capacity_rows, n, ix->idl_A[slot], ids, counts,
                                      ix->idl_ids + (size_t)ix->idl_off[slot] * ix->cap_pad,
                                      ix->idl_cnt + (size_t)slot * ix->cap_pad, ix->cap_pad, ix->hdr,
                                      (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "ID-list set rows");
  return LINR_OK;
}

namespace {
struct IdcWs {
  size_t bitmaps, qcl, qncl, qids, local, end;
};
IdcWs idc_layout(const linr_index* ix, int B, int V, int K) {
  IdcWs w;
  w.bitmaps = 0;
  w.qcl = align256((size_t)B * (ix->cap_pad / 8));
  w.qncl = w.qcl + align256((size_t)B * 16 * 16);
  w.qids = w.qncl + align256((size_t)B * 4);
  w.local = w.qids + align256((size_t)B * kIdlMaxQueryIds * 8);
  Plan pl;
  std::string why;
  size_t loc = 0;
  if (make_plan(ix, B, V, K, &pl, &why, true)) loc = ws_layout(pl, B, K).end;
  w.end = loc ? w.local + loc : 0;
  return w;
}
}  // namespace

size_t linr_search_idc_workspace_bytes(const linr_index* ix, int32_t B, int32_t V, int32_t K) {
  if (!ix || B < 1 || V < 1 || V > LINR_MAX_V || K < 1 || K > LINR_MAX_K) return 0;
  return idc_layout(ix, B, V, K).end;
}

int linr_search_idc(linr_index* ix, const void* q, int32_t B, int32_t V, const linr_clause* cl, const int32_t* off,
                    const linr_id_clause* icl, const int32_t* ioff, int32_t K, void* ws, size_t ws_bytes,
                    int64_t* out_ids, float* out_scores, int64_t* out_pass, void* stream) {
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (!ioff) return fail(LINR_EINVAL, "null ID clause offsets");
  if (!ix->idl_ids) return fail(LINR_EINVAL, "no ID lists attached (linr_idlists_attach)");
  if (B < 1 || V < 1 || V > LINR_MAX_V || K < 1 || K > LINR_MAX_K) return fail(LINR_EINVAL, "bad B/V/K");
  if (ioff[0] != 0) return fail(LINR_EINVAL, "id_clause_off[0] must be 0");
  // host validation + staging: per query its ID clauses (slot, reverse, first id, count) and the
  // sorted, de-duplicated id lists (the filter kernel binary-searches them)
  std::vector<int32_t> hcl((size_t)B * 16 * 4, 0), hncl(B, 0);
  std::vector<uint64_t> hids;
  for (int b = 0; b < B; ++b) {
    const int n = ioff[b + 1] - ioff[b];
    if (n < 0) return fail(LINR_EINVAL, "ID clause offsets must be non-decreasing");
    if (n > LINR_MAX_CLAUSES) return fail(LINR_EINVAL, "more than 16 ID clauses in one query");
    if (n > 0 && !icl) return fail(LINR_EINVAL, "null ID clauses");
    size_t qtot = 0;
    for (int c = 0; c < n; ++c) {
      const linr_id_clause& k = icl[ioff[b] + c];
      if (k.slot >= ix->idl_S) return fail(LINR_EINVAL, "ID clause slot >= attached slots");
      if (k.n < 1 || !k.ids_host) return fail(LINR_EINVAL, "empty ID clause (omit the clause instead)");
      if (k.reverse > 1) return fail(LINR_EINVAL, "ID clause reverse must be 0 or 1");
      std::vector<uint64_t> v(k.ids_host, k.ids_host + k.n);
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      qtot += v.size();
      if (qtot > (size_t)kIdlMaxQueryIds) return fail(LINR_EINVAL, "more than 1024 query ids in one query");
      int32_t* r = &hcl[((size_t)b * 16 + c) * 4];
      r[0] = k.slot;
      r[1] = k.reverse;
      r[2] = (int32_t)hids.size();
      r[3] = (int32_t)v.size();
      hids.insert(hids.end(), v.begin(), v.end());
    }
    hncl[b] = n;
  }
  const IdcWs w = idc_layout(ix, B, V, K);
  if (w.end == 0) return fail(LINR_EUNSUPPORTED, "no scan configuration for this shape");
  if (!ws || ws_bytes < w.end) return fail(LINR_ENOMEM, "workspace too small");
  DeviceGuard dg(ix->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  char* W = (char*)ws;
  // the staging copies go through a pinned slot (the caller's host arrays may be freed on return)
  linr_index::PinSlot& ps = ix->pin[ix->pin_next];
  ix->pin_next = (ix->pin_next + 1) % kPinSlots;
  if (!ps.ev && cudaEventCreateWithFlags(&ps.ev, cudaEventDisableTiming) != cudaSuccess)
    return fail(LINR_ECUDA, "staging event");
  cudaEventSynchronize(ps.ev);
  const size_t b1 = hcl.size() * 4, b2 = hncl.size() * 4, b3 = std::max<size_t>(8, hids.size() * 8);
  const size_t need = align256(b1) + align256(b2) + align256(b3);
  if (ps.bytes < need) {
    if (ps.p) cudaFreeHost(ps.p);
    ps.p = nullptr;
    ps.bytes = 0;
    if (cudaHostAlloc(&ps.p, need, cudaHostAllocDefault) != cudaSuccess) return fail(LINR_ENOMEM, "pinned staging");
    ps.bytes = need;
  }
  char* h = (char*)ps.p;
  std::memcpy(h, hcl.data(), b1);
  std::memcpy(h + align256(b1), hncl.data(), b2);
  if (!hids.empty()) std::memcpy(h + align256(b1) + align256(b2), hids.data(), hids.size() * 8);
  cudaError_t e = cudaMemcpyAsync(W + w.qcl, h, b1, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(W + w.qncl, h + align256(b1), b2, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !hids.empty())
    e = cudaMemcpyAsync(W + w.qids, h + align256(b1) + align256(b2), hids.size() * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaEventRecord(ps.ev, st);
  if (e != cudaSuccess) return cuda_fail(e, "ID clause staging");
  const int64_t words = ix->cap_pad / 32;
  const int grid_x = (int)std::min<int64_t>(ix->cap_pad / 256, (int64_t)ix->num_sms * 8);
  e = launch_idl_filter(ix->idl_ids, ix->idl_cnt, ix->cap_pad, ix->live, ix->hdr, ix->idl_off, (const int*)(W + w.qncl),
                        W + w.qcl, (const uint64_t*)(W + w.qids), B, (uint32_t*)(W + w.bitmaps), grid_x, st);
  if (e != cudaSuccess) return cuda_fail(e, "ID-list filter launch");
  if (ix->prof) ix->prof_launches += 1;
  return search_impl(ix, q, B, V, cl, off, K, W + w.local, ws_bytes - w.local, 0, out_ids, out_scores, nullptr,
                     out_pass, st, (const uint32_t*)(W + w.bitmaps), (size_t)words);
}


// ------------------------------------------------------------------ learned scorers (scorers.cu)
namespace {
struct ScLay {
  size_t Wm, bm, W1, b1, w2, b2, Fk, Wgu, bg, Wo, bo, M, Mb, y, end;
  int Fp, Fm;
};
bool scorer_ok(const linr_index* ix, const linr_scorer* w, std::string* why) {
  if (!ix || !w) { *why = "null argument"; return false; }
  if (w->kind == LINR_SCORER_HADAMARD) {
    if (w->F < 1 || w->F > 256 || w->H < 1 || w->H > 64) { *why = "Hadamard widths: F in [1,256], H in [1,64]"; return false; }
    if (!w->Wm || !w->bm || !w->Wi || !w->bi || !w->W1 || !w->b1 || !w->w2 || !w->b2) { *why = "null Hadamard weight"; return false; }
    return true;
  }
  if (w->kind == LINR_SCORER_MOL) {
    if (w->K < 1 || w->K > 8 || w->dc < 4 || w->dc % 4 || w->K * w->dc > 512 || w->G < 1 || w->G > 64) {
      *why = "MoL widths: K in [1,8], dc a multiple of 4 (K*dc <= 512), G in [1,64]";
      return false;
    }
    if (!w->Fk || !w->Gk || !w->Wgu || !w->Wgx || !w->bg || !w->Wo || !w->bo) { *why = "null MoL weight"; return false; }
    return true;
  }
  *why = "unknown scorer kind";
  return false;
}
ScLay sc_layout(const linr_index* ix, const linr_scorer* w) {
  ScLay l;
  std::memset(&l, 0, sizeof(l));
  const size_t d = ix->d.dim;
  size_t o = 0;
  auto take = [&](size_t floats) { const size_t at = o; o = align256(o + floats * 4); return at; };
  if (w->kind == LINR_SCORER_HADAMARD) {
    l.Fm = w->F;
    l.Wm = take((size_t)w->F * d); l.bm = take(w->F); l.W1 = take((size_t)w->H * w->F); l.b1 = take(w->H);
    l.w2 = take(w->H); l.b2 = take(1);
    l.M = take((size_t)w->F * d); l.Mb = take(w->F);
  } else {
    l.Fm = w->K * w->dc + w->G;
    l.Fk = take((size_t)w->K * w->dc * d); l.Wgu = take((size_t)w->G * d); l.bg = take(w->G);
    l.Wo = take((size_t)w->K * w->G); l.bo = take(w->K);
    l.M = take((size_t)l.Fm * d);   // [Gk; Wgx]
  }
  l.Fp = (l.Fm + 3) & ~3;
  l.y = o;
  l.end = o + (size_t)ix->cap_pad * l.Fp * 4;
  return l;
}
}  // namespace

size_t linr_scorer_storage_bytes(const linr_index* ix, const linr_scorer* w) {
  std::string why;
  if (!scorer_ok(ix, w, &why)) return 0;
  return sc_layout(ix, w).end;
}

int linr_scorer_attach(linr_index* ix, const linr_scorer* w, void* storage, void* stream) {
  std::string why;
  if (!scorer_ok(ix, w, &why)) return fail(LINR_EINVAL, why);
  if (!storage) return fail(LINR_EINVAL, "null storage");
  if (ix->scorer) return fail(LINR_EINVAL, "a scorer is already attached");
  DeviceGuard dg(ix->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  const ScLay l = sc_layout(ix, w);
  char* S = (char*)storage;
  const size_t d = ix->d.dim;
  cudaError_t e = cudaStreamSynchronize(st);   // setup call (like linr_codes_attach)
  auto put = [&](size_t off, const float* src, size_t floats) {
    if (e == cudaSuccess) e = cudaMemcpy(S + off, src, floats * 4, cudaMemcpyHostToDevice);
  };
  ScorerDev sd;
  std::memset(&sd, 0, sizeof(sd));
  sd.kind = w->kind;
  sd.Fp = l.Fp;
  sd.Fm = l.Fm;
  if (w->kind == LINR_SCORER_HADAMARD) {
    sd.F = w->F;
    sd.H = w->H;
    put(l.Wm, w->Wm, (size_t)w->F * d); put(l.bm, w->bm, w->F); put(l.W1, w->W1, (size_t)w->H * w->F);
    put(l.b1, w->b1, w->H); put(l.w2, w->w2, w->H); put(l.b2, w->b2, 1);
    put(l.M, w->Wi, (size_t)w->F * d); put(l.Mb, w->bi, w->F);
    sd.Wm = (const float*)(S + l.Wm); sd.bm = (const float*)(S + l.bm); sd.W1 = (const float*)(S + l.W1);
    sd.b1 = (const float*)(S + l.b1); sd.w2 = (const float*)(S + l.w2); sd.b2 = (const float*)(S + l.b2);
    sd.Mb = (const float*)(S + l.Mb);
  } else {
    sd.K = w->K;
    sd.dc = w->dc;
    sd.G = w->G;
    put(l.Fk, w->Fk, (size_t)w->K * w->dc * d); put(l.Wgu, w->Wgu, (size_t)w->G * d); put(l.bg, w->bg, w->G);
    put(l.Wo, w->Wo, (size_t)w->K * w->G); put(l.bo, w->bo, w->K);
    put(l.M, w->Gk, (size_t)w->K * w->dc * d);
    put(l.M + (size_t)w->K * w->dc * d * 4, w->Wgx, (size_t)w->G * d);
    sd.Fk = (const float*)(S + l.Fk); sd.Wgu = (const float*)(S + l.Wgu); sd.bg = (const float*)(S + l.bg);
    sd.Wo = (const float*)(S + l.Wo); sd.bo = (const float*)(S + l.bo);
    sd.Mb = nullptr;
  }
  sd.M = (const float*)(S + l.M);
  DevHeader h;
  if (e == cudaSuccess) e = cudaMemcpy(&h, ix->hdr, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "scorer attach");
  ix->sw = sd;
  ix->sy = (float*)(S + l.y);
  ix->scorer = true;
  e = launch_features(ix->d.dtype, ix->emb, ix->d.dim, (int64_t)h.hwm, 0, nullptr, 0, ix->d.capacity_rows, sd.M, sd.Mb,
                      sd.Fm, sd.Fp, ix->sy, st);
  if (e != cudaSuccess) return cuda_fail(e, "scorer features");
  return LINR_OK;
}

namespace {
struct ScWs {
  size_t params, cl, lists, pass, end;
  int stride;
};
ScWs scws_layout(const linr_index* ix, int B, int K) {
  ScWs w;
  w.stride = (sc_param_floats(ix->sw) + 3) & ~3;
  w.params = 0;
  w.cl = align256((size_t)B * w.stride * 4);
  w.lists = w.cl + align256((size_t)B * 16 * sizeof(KClause) + (size_t)B * 4);
  w.pass = w.lists + align256((size_t)ix->num_sms * B * K * 8);
  w.end = w.pass + align256((size_t)ix->num_sms * B * 8);
  return w;
}
}  // namespace

size_t linr_search_scored_workspace_bytes(const linr_index* ix, int32_t B, int32_t K) {
  if (!ix || !ix->scorer || B < 1 || K < 1 || K > LINR_MAX_K) return 0;
  return scws_layout(ix, B, K).end;
}

int linr_search_scored(linr_index* ix, const void* q, int32_t B, const linr_clause* cl, const int32_t* off, int32_t K,
                       void* ws, size_t ws_bytes, int64_t* out_ids, float* out_scores, int64_t* out_pass, void* stream) {
  std::string why;
  if (!ix) return fail(LINR_EINVAL, "null index");
  if (!ix->scorer) return fail(LINR_EINVAL, "no scorer attached (linr_scorer_attach)");
  int rc = validate_query(ix, q, B, 1, cl, off, K, &why);
  if (rc != LINR_OK) return fail(rc, why);
  if (!out_ids || !out_scores) return fail(LINR_EINVAL, "null outputs");
  const ScWs w = scws_layout(ix, B, K);
  if (!ws || ws_bytes < w.end) return fail(LINR_ENOMEM, "workspace too small");
  DeviceGuard dg(ix->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  char* W = (char*)ws;
  cudaError_t e = launch_query_prep(ix->d.dtype, ix->sw, q, ix->d.dim, B, (float*)(W + w.params), w.stride, st);
  if (e != cudaSuccess) return cuda_fail(e, "scorer query launch");
  rc = stage_clause_table(ix, cl, off, B, W + w.cl, st);
  if (rc != LINR_OK) return rc;
  ScorerScanParams p;
  std::memset(&p, 0, sizeof(p));
  p.w = ix->sw;
  p.y = ix->sy;
  p.attr = ix->attr;
  p.cap_pad = ix->cap_pad;
  p.live = ix->live;
  p.hdr = ix->hdr;
  p.row0 = (uint32_t)ix->d.global_row0;
  p.nu = B;
  p.K = K;
  p.params = (const float*)(W + w.params);
  p.param_stride = w.stride;
  p.cl = (const KClause*)(W + w.cl);
  p.ncl = (const int*)(W + w.cl + (size_t)B * 16 * sizeof(KClause));
  p.lists = (uint64_t*)(W + w.lists);
  p.pass = (int64_t*)(W + w.pass);
  if (scorer_scan_smem(w.stride) > ix->smem_optin) return fail(LINR_EUNSUPPORTED, "scorer parameters exceed shared memory");
  e = launch_scorer_scan(p, ix->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "scorer scan launch");
  MergeParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.samp = p.lists;
  mp.samp_sl = (int64_t)B * K;
  mp.samp_su = K;
  mp.ms = std::min(K, kScanSample);
  mp.list = p.lists;
  mp.list_sl = (int64_t)B * K;
  mp.list_su = K;
  mp.list_len = K;
  mp.pass = p.pass;
  mp.pstride_l = B;
  mp.pstride_u = 1;
  mp.L = ix->num_sms;
  mp.K = K;
  mp.out_ids = out_ids;
  mp.out_scores = out_scores;
  mp.out_pass = out_pass;
  mp.mode = 0;
  mp.dbg = debug_buffer();
  e = launch_merge(mp, B, st);
  if (e != cudaSuccess) return cuda_fail(e, "scorer merge launch");
  if (ix->prof) ix->prof_launches += 3;
  return LINR_OK;
}

}  // extern "C"
