// Internal declarations shared by the library's translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/linr.h"

namespace linr {

constexpr int kHdrBytes = 256;   // device header at the start of live_storage
constexpr int kFuseSlots = 16;   // searches of one index that may be in flight at once (any streams)
struct DevHeader {               // lives in device memory
  unsigned long long hwm;        // local rows [0, hwm) may be live
  unsigned long long skipped;    // out-of-shard ids seen by update/delete
  unsigned long long overflow;   // scan buffer overflows (must stay 0; checked by tests)
  // fused-merge tickets, one slot per in-flight search (searches may overlap across streams):
  unsigned int done_ctas[kFuseSlots];   // scan CTAs finished (self-resetting)
  unsigned int merged[kFuseSlots];      // users merged by the fused tail (self-resetting)
  unsigned long long tc_fallbacks;      // batched-path users recomputed exactly (fallback.cu)
};
static_assert(sizeof(DevHeader) <= kHdrBytes, "device header too large");

struct KClause {                 // clause as the kernels see it (16 B)
  unsigned long long mask;
  uint32_t word;
  uint32_t rev;
};

// Merge L partition results per user into the final top-K. Partition l of user u provides a
// sorted descending sample samp[l][u][0..ms) (its top-ms keys, 0-padded) and a list of all its
// candidate keys list[l][u][0..cnt) in any order (the sample keys included).
struct MergeParams {
  const uint64_t* samp;
  int64_t samp_sl, samp_su;      // strides (keys) per partition / per user
  int ms;                        // sample length (<= 64)
  const uint64_t* list;
  int64_t list_sl, list_su;
  const int* cnt;                // cnt[l*cnt_sl + u*cnt_su]; null: every list has list_len keys (0-padded)
  int64_t cnt_sl, cnt_su;
  int list_len;                  // max keys per list
  const int64_t* pass;           // pass[l*pstride_l + u*pstride_u]
  int64_t pstride_l, pstride_u;
  int L, K;
  int64_t* out_ids;              // [B][K] (mode 0)
  float* out_scores;             // [B][K] (mode 0)
  uint64_t* out_keys;            // [B][K] (mode 1)
  int64_t* out_pass;             // [B] (may be null)
  int mode;                      // 0: decode ids/scores, 1: sorted keys
  int bucket_sort;               // 1: skip the sorted-prefix merge (bucket sort; A/B knob LINR_MERGE_BUCKET)
  const uint64_t* thr;           // [B] thresholds the scan started from (union path), or null
  int* flags;                    // [B] set to 1 when fewer than K keys >= thr[u] were found (recompute)
  const int* gate;               // merge_kernel: run only if *gate == gate_want (null: always)
  int gate_want;
  unsigned long long* dbg;       // diagnostics timers
};

// Parameters of one GEMV scan launch (passed by value; <= 4 KB).
struct ScanParams {
  const void* emb;               // [cap_pad][dim]
  const uint64_t* attr;          // SoA [W][cap_pad]
  const uint32_t* live;          // bitmap [cap_pad/32]
  DevHeader* hdr;
  int64_t cap_pad;
  uint32_t row0;                 // global id of local row 0
  int nu;                        // users in this launch
  int V;                         // vectors per user
  int K;
  int C;                         // soft capacity of the per-user CTA buffer
  int bufcap;                    // hard capacity (C + headroom)
  int list_cap;                  // capacity of each per-CTA output list (keys)
  uint32_t wmask;                // attribute words referenced by any clause
  const void* q;                 // [nu][V][dim] queries of this launch's users
  uint64_t* out_samp;            // [nu][gridDim.x][32] sorted top-32 of each CTA
  uint64_t* out_list;            // [nu][gridDim.x][list_cap] every key the CTA kept (unsorted)
  int* out_cnt;                  // [nu][gridDim.x] keys in out_list
  int64_t* out_pass;             // [nu][gridDim.x]
  unsigned long long* dbg;        // diagnostics timers (null unless linr_debug_timers(1))
  int fuse_slot;          // DevHeader ticket slot of this search
  int fuse_merge;                // 1: the last nu CTAs run the merge (mp) for this launch's users
  int ring;                      // > 0: warp-specialised scan with this many row-group slots
  const uint64_t* init_thr;      // [nu] starting CTA thresholds (union path: sample-derived), or null
  const int* gate;               // non-null: run only if *gate == gate_want (device-side path choice)
  int gate_want;
  MergeParams mp;                // merge of this launch's users (user index relative to the launch)
  int ncl[8];
  KClause cl[8][16];
};

struct ScanCfg {                 // launch geometry chosen for one (dtype, dim, nqv)
  int nt;                        // threads per CTA
  int rows_per_iter;             // rows a warp scores per inner iteration (append burst bound)
  int ring_bytes;                // per-warp cp.async row ring (stages x rows_per_iter x row bytes)
  int ws_slot_bytes;             // > 0: warp-specialised kernel available; bytes per row-group slot
  int ws_fixed_bytes;            // its shared memory besides the slots and the key buffers
  int ws_cons_warps;             // its warps that append keys (buffer headroom: 16 keys each)
};
constexpr int kScanSample = 32;  // sorted per-CTA sample length

// Launch the fused filter + score + CTA top-K scan. nqv = padded vectors per launch (1,2,4,8).
cudaError_t launch_scan_gemv(int dtype, int dim, int nqv, const ScanParams& p, int grid,
                             size_t smem, cudaStream_t st);
bool scan_gemv_supported(int dtype, int dim, int nqv);
ScanCfg scan_gemv_cfg(int dtype, int dim, int nqv);

cudaError_t launch_merge(const MergeParams& p, int B, cudaStream_t st, bool pdl = false);
size_t merge_smem();

// index maintenance kernels
cudaError_t launch_attr_soa(const uint64_t* src, int64_t n, int W, uint64_t* dst_soa, int64_t cap_pad,
                            int64_t r0, cudaStream_t st);
cudaError_t launch_set_live_range(uint32_t* live, DevHeader* hdr, int64_t r0, int64_t n, cudaStream_t st);
cudaError_t launch_update_rows(const int64_t* rows, int64_t n, int64_t grow0, int64_t cap, int rowbytes,
                               const void* emb_src, const uint64_t* attr_src, int W, void* emb,
                               uint64_t* attr, int64_t cap_pad, uint32_t* live, DevHeader* hdr,
                               cudaStream_t st);
cudaError_t launch_delete_rows(const int64_t* rows, int64_t n, int64_t grow0, int64_t cap, uint32_t* live,
                               DevHeader* hdr, cudaStream_t st);
cudaError_t launch_generate(int dtype, int dim, int W, uint64_t seed, int mode, int64_t row_begin, int64_t n,
                            void* emb, int64_t emb_row_offset, uint64_t* attrs, int64_t attr_stride_rows,
                            bool attrs_soa, cudaStream_t st);

// batched tcgen05 path (scan_tc.cu)
struct TcParams {
  CUtensorMap tmx;   // items: [cap_pad][ROWB] bytes, box {SW, 128}
  CUtensorMap tmq;   // queries: [nvec][ROWB] bytes, box {SW, NP}
  const uint64_t* attr;
  int64_t cap_pad;
  const uint32_t* live;
  const DevHeader* hdr;
  uint32_t row0;
  int nu, V, nvec, K;
  int wmax;              // attribute words staged per tile (1 + highest word any clause reads; 0 = none)
  const KClause* cl;     // [nu][16]
  const int* ncl;        // [nu]
  int maxc;              // clause slots per user in the shared-memory table (max clauses of any user)
  const uint64_t* thr;   // [nu] (main pass) ; null in the sample pass (T = 0)
  uint64_t* buf;         // [nu][grid][cap] per-(user, CTA) regions
  int cap;
  int* cnt;              // [nu][grid] keys each CTA produced for each user (may exceed cap)
  int sample_tiles;      // sample pass: tiles per CTA (0 = main pass, all tiles)
  int dyn;               // 1: epilogue warps of a TMEM lane quarter take chunks dynamically
  int sample_thr;        // 1: tiles spread like the sample pass, main-pass epilogue (keys >= thr)
  const int* gate;       // non-null: run only if *gate == gate_want (device-side path choice)
  int gate_want;
  unsigned long long* dbg;   // diagnostics: per-tile role timestamps of CTA 0 (null = off)
};

bool tc_supported(int dtype, int dim, int nvec, int V);
int tc_np(int nvec);
size_t tc_smem_bytes(int dtype, int dim, int np, int nu, int maxc, int wmax);
bool tc_encode_map(CUtensorMap* m, const void* base, int64_t rows, int rowbytes, int box_rows);
cudaError_t launch_tc_scan(int dtype, int dim, int np, const TcParams& p, int grid, cudaStream_t st);
cudaError_t launch_tc_threshold(const uint64_t* sbuf, const int* scnt, int scap, int grid, int nu, int K,
                                int sample_items, const DevHeader* hdr, uint64_t* thr, cudaStream_t st, const uint64_t* floor = nullptr);
cudaError_t launch_tc_decide(const uint64_t* thr, const int* scnt, int grid, int64_t sample_rows, const DevHeader* hdr,
                             int nu, int* gate, cudaStream_t st);
cudaError_t launch_tc_finalize(const uint64_t* buf, const int* cnt, int cap, int grid, const uint64_t* thr, int nu,
                               int K, int64_t* out_ids, float* out_scores, uint64_t* out_keys, int* flags,
                               unsigned int* fb_bar, cudaStream_t st, const int* gate = nullptr);
cudaError_t launch_tc_count(const uint64_t* attr, int64_t cap_pad, const uint32_t* live, const DevHeader* hdr,
                            const KClause* cl, const int* ncl, int nu, unsigned long long* counts, int grid,
                            cudaStream_t st);
constexpr int kTcSampleTiles = 8;
constexpr int kTcSampleCap = 256;   // per (user, CTA) region of the sample: first passers in row order
constexpr int kTcMainCap = 256;                      // per (user, CTA) region of the main pass


// exact device-side recomputation of the batched path's uncertified users (fallback.cu)
struct FbParams {
  const void* emb;
  const uint64_t* attr;
  int64_t cap_pad;
  const uint32_t* live;
  DevHeader* hdr;
  uint32_t row0;
  int dim, V, K, nu;
  const void* q;            // [nu][V][dim] index dtype
  const KClause* cl;        // [nu][16]
  const int* ncl;           // [nu]
  const int* flags;         // [nu] 1 = recompute
  uint64_t* lists;          // [2][grid][K] per-CTA top-K lists
  unsigned int* bar;        // grid barrier counter, zeroed before the launch (tc_finalize_kernel)
  int64_t* out_ids;         // [nu][K] (mode 0)
  float* out_scores;
  uint64_t* out_keys;       // [nu][K] (mode 1)
};
cudaError_t launch_fallback(int dtype, const FbParams& p, int grid, cudaStream_t st);
size_t fallback_ws_bytes(int grid, int K);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is
// per device, so the cache is keyed by the current device ordinal.
cudaError_t ensure_smem(const void* kernel, size_t smem);

// ---------------------------------------------------------------- quantised path (codes.cu)
constexpr int kCodeMaxUsers = 8;   // users per code-scan launch
struct CodeScanParams {            // pass 1: filter + matched bits + histograms
  const uint64_t* codes;           // [cap_pad][k/64]
  const uint64_t* attr;
  int64_t cap_pad;
  const uint32_t* live;
  const DevHeader* hdr;
  int nu, V;
  const uint64_t* qcodes;          // [nu][V][k/64] query codes (NOT applied in the kernel)
  const KClause* cl;               // [nu][16]
  const int* ncl;                  // [nu]
  uint32_t wmask;                  // attribute words any clause reads
  void* marr;                      // [nu][cap_pad] u8 (k <= 192) / u16 matched bits, none = 0xFF / 0xFFFF
  uint16_t* tmax;                  // [nu][tmax_stride] per-tile max m (0xFFFF: no passing item)
  int64_t tmax_stride;
  uint32_t* H;                     // [nu][k+1][GW] per-warp histograms
  unsigned long long* T;           // [nu][k+1] totals (zeroed before the launch)
  unsigned int* ticket;            // CTA completion counter (zeroed before; reset by the last CTA)
  int64_t K;                       // results wanted (code search) / the K floor of V3
  double keep;                     // > 0: V3 keep fraction
  int* mstar;                      // [nu] out: the lowest m emitted (k+1: nothing)
  int64_t* kept;                   // [nu] out: positions to produce
  int64_t* pass;                   // [nu] out: passing items (may be null)
  unsigned long long* above;       // [nu][k+2] out: #items with a larger m
};
struct CodeOffsetParams {
  const uint32_t* H;               // [nu][k+1][GW]
  const unsigned long long* above; // [nu][k+2]
  const int* mstar;                // [nu]
  int GW, k;
  uint32_t* off;                   // [nu][GW][k+1] first output position (valid for m >= m*)
};
struct CodeEmitParams {
  const void* marr;
  const uint16_t* tmax;
  int64_t tmax_stride;
  const DevHeader* hdr;
  int64_t cap_pad;
  uint32_t row0;
  int nu;
  const uint32_t* off;
  const int* mstar;
  const int64_t* kept;
  int64_t out_stride;              // per-user stride of the outputs below
  int64_t* out_ids;                // code search: ids, matched bits
  int32_t* out_m;
  uint32_t* cand;                  // V3: kept local rows
};
struct RerankParams {
  const void* emb;
  uint32_t row0;
  int dim, V, K, nu;
  const void* q;                   // [nu][V][dim]
  const uint32_t* cand;            // [nu][cand_stride] local rows
  int64_t cand_stride;
  const int64_t* kept;             // [nu]
  uint64_t* lists;                 // [grid][nu][K] sorted per-CTA top-K
};
cudaError_t launch_oporp_encode(int dtype, const void* x, int dim, int64_t n, int64_t row_begin, const int64_t* rows,
                                int64_t grow0, int64_t cap, int k, int L, const int32_t* src, const int8_t* sign,
                                uint64_t* codes, cudaStream_t st);
size_t code_hist_smem(int nu, int V, int k);
size_t rerank_smem(int V, int dim);
cudaError_t launch_code_hist(int k, const CodeScanParams& p, int grid, cudaStream_t st);
cudaError_t launch_code_offsets(const CodeOffsetParams& p, int nu, cudaStream_t st);
cudaError_t launch_code_emit(int k, const CodeEmitParams& p, int grid, cudaStream_t st);
cudaError_t launch_code_pad(const int64_t* kept, int nu, int64_t K, int64_t* out_ids, int32_t* out_m, int grid,
                            cudaStream_t st);
cudaError_t launch_rerank(int dtype, const RerankParams& p, int grid, cudaStream_t st);

// ---------------------------------------------------------------- ID-list clauses (idlist.cu)
constexpr int kIdlMaxQueryIds = 1024;   // query ids over all ID clauses of one query
cudaError_t launch_idl_filter(const uint64_t* ids, const uint8_t* counts, int64_t cap_pad, const uint32_t* live,
                              const DevHeader* hdr, const int* slot_off, const int* q_ncl, const void* q_cl,
                              const uint64_t* q_ids, int B, uint32_t* out, int grid_x, cudaStream_t st);
cudaError_t launch_idl_set_rows(const int64_t* rows, int64_t r0, int64_t grow0, int64_t cap, int64_t n, int A,
                                const uint64_t* src_ids, const uint8_t* src_cnt, uint64_t* dst_ids, uint8_t* dst_cnt,
                                int64_t cap_pad, DevHeader* hdr, cudaStream_t st);

// ---------------------------------------------------------------- learned scorers (scorers.cu)
struct ScorerDev {                 // device pointers into the caller's scorer storage
  int kind, F, H, Fp, K, dc, G;
  const float *Wm, *bm, *W1, *b1, *w2, *b2;   // Hadamard query side
  const float *Fk, *Wgu, *bg, *Wo, *bo;       // MoL query side
  const float *M, *Mb;                        // item side: y = M x (+ Mb), [Fm][dim]
  int Fm;                                     // rows of M (F, or K*dc + G)
};
struct ScorerScanParams {
  ScorerDev w;
  const float* y;                  // [cap_pad][Fp] item features
  const uint64_t* attr;
  int64_t cap_pad;
  const uint32_t* live;
  const DevHeader* hdr;
  uint32_t row0;
  int nu, K;
  const float* params;             // [nu][param_stride] query-side parameters
  int param_stride;
  const KClause* cl;               // [nu][16]
  const int* ncl;
  uint64_t* lists;                 // [grid][nu][K]
  int64_t* pass;                   // [grid][nu]
};
cudaError_t launch_features(int dtype, const void* emb, int dim, int64_t n, int64_t r_begin, const int64_t* rows,
                            int64_t grow0, int64_t cap, const float* M, const float* bias, int F, int Fp, float* y,
                            cudaStream_t st);
int sc_param_floats(const ScorerDev& w);
cudaError_t launch_query_prep(int dtype, const ScorerDev& w, const void* q, int dim, int B, float* out, int stride,
                              cudaStream_t st);
size_t scorer_scan_smem(int param_floats);
cudaError_t launch_scorer_scan(const ScorerScanParams& p, int grid, cudaStream_t st);

// NCCL communicator of a row-sharded index (comm.cu; NCCL loaded at run time)
int comm_create(int device, const uint8_t id[128], int rank, int world, void** out);
void comm_destroy(void* comm);
int comm_allgather_u64(void* comm, const uint64_t* send, uint64_t* recv, size_t count, cudaStream_t st);

void set_error(const std::string& msg);
void set_error_detail(const std::string& detail);
int env_int(const char* name, int dflt);
unsigned long long* debug_buffer();

}  // namespace linr
