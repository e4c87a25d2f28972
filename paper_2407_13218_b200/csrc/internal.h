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

cudaError_t launch_merge(const MergeParams& p, int B, cudaStream_t st);
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
  unsigned long long* dbg;   // diagnostics: per-tile role timestamps of CTA 0 (null = off)
};

bool tc_supported(int dtype, int dim, int nvec, int V);
int tc_np(int nvec);
size_t tc_smem_bytes(int dtype, int dim, int np, int nu, int maxc, int wmax);
bool tc_encode_map(CUtensorMap* m, const void* base, int64_t rows, int rowbytes, int box_rows);
cudaError_t launch_tc_scan(int dtype, int dim, int np, const TcParams& p, int grid, cudaStream_t st);
cudaError_t launch_tc_threshold(const uint64_t* sbuf, const int* scnt, int scap, int grid, int nu, int K,
                                int sample_items, const DevHeader* hdr, uint64_t* thr, cudaStream_t st);
cudaError_t launch_tc_finalize(const uint64_t* buf, const int* cnt, int cap, int grid, const uint64_t* thr, int nu,
                               int K, int64_t* out_ids, float* out_scores, uint64_t* out_keys, int* flags,
                               cudaStream_t st);
cudaError_t launch_tc_count(const uint64_t* attr, int64_t cap_pad, const uint32_t* live, const DevHeader* hdr,
                            const KClause* cl, const int* ncl, int nu, unsigned long long* counts, int grid,
                            cudaStream_t st);
constexpr int kTcSampleTiles = 8;
constexpr int kTcSampleCap = 256;   // per (user, CTA) region of the sample: first passers in row order
constexpr int kTcMainCap = 256;                      // per (user, CTA) region of the main pass


void set_error(const std::string& msg);
unsigned long long* debug_buffer();

}  // namespace linr
