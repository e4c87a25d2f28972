/*
 * linr.h — C ABI of the B200-native LiNR pre-filtered exhaustive top-K scan.
 *
 * The operation (arXiv 2407.13218, §3.1 "Exhaustive Search with Attribute-Based
 * Matching"): for each query, evaluate its boolean attribute clauses against every
 * item's attribute bitmask ("Feasible items should satisfy all clauses, requiring at least one of
 * the attribute in each clauses is matched. Reverse clauses are also supported"), score
 * every surviving item by dot product with the query embedding ("KNN uses dot-product
 * similarity"), and return the best K (score, item-id) pairs ("Top-1 selection",
 * top-2k in §5.3). Filtered items are excluded, never scored as zero (DESIGN.md reading
 * R1). Live updates overwrite rows in place in pre-allocated storage under a high-water mark
 * (§4.3 "Model Live Update").
 *
 * Conventions shared by every entry point
 *  - Every call returns a linr_status (0 = OK). No C++ exception crosses the ABI. On failure
 *    linr_last_error() returns a thread-local message. Validation happens before anything is
 *    enqueued; asynchronous CUDA errors are sticky and surface as LINR_ECUDA on a later call.
 *  - "_dev" pointers are CUDA device pointers on the index's device; "_host" pointers are host
 *    memory (pinned or pageable). All data buffers are caller-owned (PyTorch allocates them);
 *    the library never frees them and they must outlive every call that uses them.
 *  - `stream` is a cudaStream_t passed as void*. All device work is enqueued on it; calls
 *    return before the work finishes, except linr_search_host, linr_index_stats and
 *    linr_index_counters, which
 *    synchronise `stream`. A search observes exactly the updates enqueued before it on the same
 *    stream (snapshot consistency by stream order; reading R16). Searches (only searches) of one
 *    index may run concurrently on different streams, up to 16 in flight, each with its own
 *    workspace (pipelined serving); any other unordered concurrent use of one index from two
 *    streams (an update racing a search) is undefined.
 *  - Item ids are global row ids: local row r of a shard has id global_row0 + r (int64 in the
 *    ABI, < 2^32-1 internally). Results are ordered by score descending, then id ascending
 *    (reading R5); slots past min(K, pass_count) hold id -1 and score -inf (reading R6).
 *  - Scores are returned as fp32: float dtypes accumulate in fp32 (reading R8); int8 scores are
 *    exact integer dot products, exactly representable in fp32 for dim <= 1024 (reading R10).
 */
#ifndef LINR_H_
#define LINR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct linr_index linr_index; /* opaque: library-owned metadata only */

typedef enum {
  LINR_OK = 0,
  LINR_EINVAL = -1,       /* bad argument (null pointer, shape, clause, dtype …)        */
  LINR_ERANGE = -2,       /* row range outside [global_row0, global_row0 + capacity)     */
  LINR_ENOMEM = -3,       /* workspace too small / host allocation failed                */
  LINR_ECUDA = -4,        /* CUDA launch / runtime error (sticky asynchronous errors too) */
  LINR_ENCCL = -5,        /* NCCL failure (communicator creation / collective)           */
  LINR_EUNSUPPORTED = -6  /* valid but not built (e.g. a dim with no compiled kernel)     */
} linr_status;

typedef enum { LINR_F32 = 0, LINR_F16 = 1, LINR_BF16 = 2, LINR_I8 = 3 } linr_dtype;

/* One clause of a query (16 bytes, host memory).
 * passes(item) = ((attrs[item][word] & mask) != 0) XOR reverse
 * mask: the clause's attribute set as bits of attribute word `word` (reading R2: a clause lists
 *       attribute values; OR within the clause = any bit overlaps). mask == 0 is rejected
 *       (EINVAL; reading R3 — omit the clause to disable it).
 * word: attribute word index, < attr_words.  reverse: 0 = Match, 1 = Reverse. */
typedef struct {
  uint64_t mask;
  uint8_t word;
  uint8_t reverse;
  uint8_t pad[6];
} linr_clause;

#define LINR_MAX_K 2048          /* K range 1..2048 (paper uses K=2000; reading R14) */
#define LINR_MAX_V 8             /* query vectors per user (multi-embedding, reading R12)     */
#define LINR_MAX_CLAUSES 16      /* clauses per query                                         */
#define LINR_MAX_ATTR_WORDS 4    /* u64 attribute words per item                              */

typedef struct {
  int64_t capacity_rows; /* rows pre-allocated on this shard ("pre-allocating larger tensors") */
  int64_t global_row0;   /* global id of local row 0 (row sharding)                                 */
  int32_t dim;           /* d: power of two in [16, 1024]                                           */
  int32_t dtype;         /* linr_dtype of items AND queries                                         */
  int32_t attr_words;    /* W in [1, 4]                                                             */
  int32_t device;        /* CUDA device ordinal the storage lives on                                */
  void* emb_storage;     /* device, linr_storage_bytes(desc, 0) bytes, caller-owned                 */
  void* attr_storage;    /* device, linr_storage_bytes(desc, 1) bytes                               */
  void* live_storage;    /* device, linr_storage_bytes(desc, 2) bytes; MUST be zero-filled at create */
} linr_index_desc;

/* Bytes the caller must allocate for storage `which` (0 emb, 1 attrs, 2 live bitmap + device
 * header incl. the high-water mark). Capacity is padded internally to a multiple of 256 rows.
 * Returns 0 for an invalid desc/which. Layout is private to the library. */
size_t linr_storage_bytes(const linr_index_desc* desc, int which);

/* Validate desc and create a handle over the caller's storage. live_storage must be zeroed
 * (no row live, high-water mark 0: "empty index; high_water_mark = 0"). */
int linr_index_create(const linr_index_desc* desc, linr_index** out);
void linr_index_destroy(linr_index* index);

/* Bulk load rows [row0, row0+n) (global ids) from device buffers:
 *   emb_dev   [n][dim] row-major in the index dtype;  attrs_dev [n][attr_words] u64 row-major.
 * Marks the rows live and raises the high-water mark ("using a high-water mark").
 * ERANGE if the range leaves the shard. n == 0 is a no-op. */
int linr_index_load(linr_index* index, int64_t row0, int64_t n, const void* emb_dev,
                    const uint64_t* attrs_dev, void* stream);

/* Live upsert (§4.3, "expose Upsert and Delete APIs"): overwrite rows
 * rows_dev[0..n) (global ids, device int64) in place with emb_dev [n][dim], attrs_dev [n][W];
 * mark them live; raise the high-water mark. Ids outside this shard are skipped on the device
 * and counted (linr_index_stats). If an id repeats within one call, its LAST occurrence wins
 * (the earlier copies are not written). A search on the same stream sees each row wholly old or
 * wholly new. Cost: one warp per entry, plus a scan of the later entries for duplicates. */
int linr_index_update_rows(linr_index* index, const int64_t* rows_dev, int64_t n,
                           const void* emb_dev, const uint64_t* attrs_dev, void* stream);

/* Live delete: clear the liveness bit of rows_dev[0..n) (tombstone; reading R7). The
 * high-water mark never decreases. Out-of-shard ids are skipped and counted. */
int linr_index_delete_rows(linr_index* index, const int64_t* rows_dev, int64_t n, void* stream);

/* Synchronising read of the device header: high-water mark (local rows), the number of
 * out-of-shard ids skipped by update/delete so far, and the number of scan-buffer overflows (an
 * internal invariant that must stay 0; tests assert it). Any output may be NULL. */
int linr_index_stats(linr_index* index, int64_t* hwm_host, int64_t* skipped_host,
                     int64_t* scan_overflow_host, void* stream);

/* Synchronising read of all device-side counters (a superset of linr_index_stats):
 *   hwm            high-water mark (local rows)
 *   skipped        out-of-shard ids skipped by update/delete
 *   scan_overflow  scan-buffer overflows (internal invariant, must stay 0)
 *   tc_fallbacks   batched-path users whose pruned result could not be certified and were
 *                  recomputed exactly on the device (reading R23; statistics only, results are
 *                  exact either way) */
typedef struct {
  int64_t hwm, skipped, scan_overflow, tc_fallbacks;
} linr_counters;
int linr_index_counters(linr_index* index, linr_counters* out_host, void* stream);

/* Workspace bytes needed by linr_search / linr_search_keys for (B, V, K). 0 if invalid. */
size_t linr_search_workspace_bytes(const linr_index* index, int32_t B, int32_t V, int32_t K);

/* The hot path: filtered exhaustive top-K over this shard.
 *   queries_dev  [B][V][dim] in the index dtype (V <= LINR_MAX_V query vectors per user; score =
 *                max over the user's V dot products, reading R12)
 *   clauses_host  all clauses, CSR by clause_off_host[B+1] (host int32, non-decreasing,
 *                 clause_off_host[0] == 0, at most LINR_MAX_CLAUSES per query)
 *   ws_dev        device workspace of >= linr_search_workspace_bytes(index, B, V, K) bytes
 *   out_ids_dev [B][K] int64, out_scores_dev [B][K] fp32, out_pass_dev [B] int64 (may be NULL:
 *                 number of live items passing each query's clauses)
 * EINVAL on: null pointers, B < 1, V < 1 or > LINR_MAX_V, K < 1 or > LINR_MAX_K, bad offsets,
 * clause word >= W, clause mask == 0, too many clauses.
 * The library picks the kernel path by batch shape: one fused ring-scan launch per
 * user (B = 1, B = 2, or V > 1); the union path (V = 1, 3 <= B <= 8: one launch over the union of
 * the users' passing rows from sample-derived thresholds); the tcgen05 batched path (B*V >= 9;
 * bf16/f16/int8, dim 64/128). Every path returns the exact result: the two thresholded paths
 * certify each user on the device and recompute uncertified users exactly (readings R23, R33). */
int linr_search(linr_index* index, const void* queries_dev, int32_t B, int32_t V,
                const linr_clause* clauses_host, const int32_t* clause_off_host, int32_t K,
                void* ws_dev, size_t ws_bytes, int64_t* out_ids_dev, float* out_scores_dev,
                int64_t* out_pass_dev, void* stream);

/* Row sharding over GPUs (BASELINE.json north_star: "sharded row-wise across the 8 GPUs of one
 * B200 box, each shard produces its local top-K, and an NCCL allgather of K (score, item-id)
 * pairs over NVLink feeds a final merge"). One process per GPU, one index handle per shard
 * (global_row0 = first global row of the shard).
 *   linr_nccl_unique_id: out[128] = a fresh NCCL unique id (call on one rank, broadcast the bytes).
 *   linr_comm_init: attach a communicator of `world` ranks (this handle is rank `rank`) to the
 *     index; collective over the ranks (blocks until all have joined). Once attached, linr_search
 *     and linr_search_host return the GLOBAL result on every rank: the shard's sorted keys and
 *     pass counts are packed into one buffer of B*(K+1) u64, one ncclAllGather exchanges them and
 *     the merge kernel reduces the world lists (exact, reading R13); out_pass is the global count.
 *     linr_search_workspace_bytes includes the exchange buffers. The communicator is destroyed
 *     with the index. NCCL is loaded at run time (libnccl.so.2); LINR_ENCCL if it is missing or
 *     a collective fails. Ranks must call linr_search in the same order with the same B, V, K. */
int linr_nccl_unique_id(uint8_t* out);
int linr_comm_init(linr_index* index, const uint8_t* id, int32_t rank, int32_t world);

/* Shard-local variant for row-sharded indexes: same inputs as linr_search, output is this
 * shard's top-K as packed keys out_keys_dev [B][K] u64 (sorted descending, 0-padded) plus
 * out_pass_dev [B] int64. key = (ordered_u32(score) << 32) | (0xFFFFFFFF - global_id), where
 * ordered_u32 maps fp32 order to unsigned order (-0.0 as +0.0); larger key = better result. The
 * keys of all shards are exchanged (all-gather over torch.distributed/NCCL) and merged by
 * linr_merge_keys. */
int linr_search_keys(linr_index* index, const void* queries_dev, int32_t B, int32_t V,
                     const linr_clause* clauses_host, const int32_t* clause_off_host, int32_t K,
                     void* ws_dev, size_t ws_bytes, uint64_t* out_keys_dev, int64_t* out_pass_dev,
                     void* stream);

/* Workspace for linr_merge_keys. */
size_t linr_merge_workspace_bytes(int32_t L, int32_t B, int32_t K);

/* Merge L shard results (BASELINE.json north_star: "allgather of K (score, item-id) pairs ...
 * feeds a final merge"; reading R13: union then top-K under the same total order):
 *   keys_dev [L][B][K] u64 (each list sorted descending, 0-padded), pass_dev [L][B] int64
 * -> out_ids_dev [B][K] int64, out_scores_dev [B][K] fp32, out_pass_dev [B] (sum; may be NULL). */
int linr_merge_keys(const uint64_t* keys_dev, const int64_t* pass_dev, int32_t L, int32_t B,
                    int32_t K, void* ws_dev, size_t ws_bytes, int64_t* out_ids_dev,
                    float* out_scores_dev, int64_t* out_pass_dev, void* stream);

/* End-to-end convenience call with HOST buffers (the e2e path the benchmark times): copies
 * queries_host [B][V][dim] to the device, runs linr_search, copies ids/scores/pass back to
 * out_ids_host [B][K], out_scores_host [B][K], out_pass_host [B] (may be NULL) and synchronises
 * `stream`. ws_dev must hold linr_search_workspace_bytes(...) + linr_search_host_extra_bytes(...). */
size_t linr_search_host_extra_bytes(const linr_index* index, int32_t B, int32_t V, int32_t K);
int linr_search_host(linr_index* index, const void* queries_host, int32_t B, int32_t V,
                     const linr_clause* clauses_host, const int32_t* clause_off_host, int32_t K,
                     void* ws_dev, size_t ws_bytes, int64_t* out_ids_host, float* out_scores_host,
                     int64_t* out_pass_host, void* stream);

/* linr_search_host without the final synchronisation (pipelined serving: several searches in
 * flight on different streams, each with its own ws_dev and host buffers). The query copy and the
 * result copies are enqueued on `stream`; queries_host and the out_*_host buffers must be pinned
 * and stay valid until `stream` has completed them (the caller synchronises the stream before it
 * reads the results or reuses the buffers). Errors: as linr_search_host (copy errors may surface
 * at the caller's synchronisation). */
int linr_search_host_async(linr_index* index, const void* queries_host, int32_t B, int32_t V,
                           const linr_clause* clauses_host, const int32_t* clause_off_host, int32_t K,
                           void* ws_dev, size_t ws_bytes, int64_t* out_ids_host, float* out_scores_host,
                           int64_t* out_pass_host, void* stream);

/* ---------------------------------------------------------------- quantised KNN (§3.2)
 * Sign-OPORP 1-bit codes ("Sign One Permutation One Random Projection ... compress
 * embeddings to 1-bit and approximate dot-products via bitwise matching"). The projection is ONE
 * permutation and ONE random sign vector of length L = bits * b, given as
 *   src_host[L]  : the input coordinate at permuted position p, in [0, dim), or -1 (zero padding)
 *   sign_host[L] : +1 / -1
 * Bit j of a vector's code = [ sum_{p in [j*b, (j+1)*b)} sign[p] * x[src[p]] >= 0 ] (sum in fp64 in
 * position order, so codes are deterministic; sign(0) = +); codes are bits/64 u64 words, LSB
 * first. How src/sign are drawn (padding for bits <= dim, replication for bits > dim) is the
 * caller's choice (reading R25; datagen.oporp_params). */
typedef struct {
  int32_t bits;              /* k: 64, 128, 256, 512 or 1024                          */
  int32_t L;                 /* parameter length, a multiple of bits                  */
  const int32_t* src_host;   /* [L]                                                   */
  const int8_t* sign_host;   /* [L]                                                   */
} linr_oporp_params;

/* Bytes of the caller-owned device storage for the codes of every row + the parameters; 0 if the
 * parameters are invalid. */
size_t linr_codes_storage_bytes(const linr_index* index, const linr_oporp_params* params);

/* Attach 1-bit codes to the index: copies the parameters, encodes every row below the high-water
 * mark (setup call: synchronises `stream`, then enqueues the encoding on it). From then on load,
 * update_rows and generate re-encode the rows they write, on the same stream (live updates keep
 * the codes exact). EINVAL on bad parameters (src outside [-1, dim), sign not +-1, L % bits). */
int linr_codes_attach(linr_index* index, const linr_oporp_params* params, void* code_storage_dev,
                      void* stream);

/* Encode n vectors x_dev [n][dim] (index dtype) with the attached parameters -> codes_dev
 * [n][bits/64] u64 (the same arithmetic the index and the searches use). */
int linr_oporp_encode(const linr_index* index, const void* x_dev, int64_t n, uint64_t* codes_dev,
                      void* stream);

/* Workspace for linr_code_search (v3 = 0) / linr_search_v3 (v3 = 1). 0 if invalid or no codes. */
size_t linr_code_search_workspace_bytes(const linr_index* index, int32_t B, int32_t V, int64_t K,
                                        int32_t v3);

/* Filtered search ranked by matched bits only (Fig. 3 caption P:4310: "The quantized KNN module
 * can be used without full precision matrix multiplication when K is large in top-K selection";
 * top-50M of 1B). Per query: the clause filter (as linr_search), m(item) = max over the
 * user's V query codes of popcount(NOT(q) XOR code(item)) = matched bits, results ordered by
 * (m desc, id asc). K is UNBOUNDED (any K >= 1, up to the index size: exact selection by a
 * counting sort over m in two passes). out_ids_dev [B][K] int64, out_matched_dev [B][K] int32;
 * slots past min(K, pass) hold id -1 and m -1. out_pass_dev [B] may be NULL. */
int linr_code_search(linr_index* index, const void* queries_dev, int32_t B, int32_t V,
                     const linr_clause* clauses_host, const int32_t* clause_off_host, int64_t K,
                     void* ws_dev, size_t ws_bytes, int64_t* out_ids_dev, int32_t* out_matched_dev,
                     int64_t* out_pass_dev, void* stream);

/* V3 two-stage search ("leverage the approximated similarity as an extra pre-filtering
 * step to reduce the computation of the full-precision matrix multiplication", Fig. 3; SPEC
 * S:346-354): clause filter; keep the K' = min(pass, max(K, ceil(keep * pass))) best items by
 * matched bits (m desc, id asc); re-score the kept items by the full-precision dot product (max
 * over V, fp32 accumulation as linr_search) and return their top-K (score desc, id asc).
 * keep in (0, 1]; keep = 1 is the exact search. K in [1, 2048]. out_kept_dev [B] (may be NULL) =
 * K' per query. */
int linr_search_v3(linr_index* index, const void* queries_dev, int32_t B, int32_t V,
                   const linr_clause* clauses_host, const int32_t* clause_off_host, int32_t K,
                   double keep, void* ws_dev, size_t ws_bytes, int64_t* out_ids_dev,
                   float* out_scores_dev, int64_t* out_pass_dev, int64_t* out_kept_dev, void* stream);

/* ---------------------------------------------------------------- ID-list clauses
 * "Each query clause could contain multiple attributes. Feasible items should satisfy all
 * clauses, requiring at least one of the attribute in each clauses is matched. Reverse clauses
 * are also supported ... we store all clause attributes in a single matrix ... and have an extra
 * counting matrix to record the number of attributes for each item in each clause";
 * attributes are "converted to 64-bit integers before GPU comparison". This is the
 * high-cardinality companion of the bitmask clauses (geo, company, title as 64-bit ids).
 * An index may carry up to LINR_MAX_ID_SLOTS slots; slot s holds up to widths[s] ids per item. */
#define LINR_MAX_ID_SLOTS 4
#define LINR_MAX_IDS_PER_ITEM 16

/* Query-side clause on an ID-list slot: passes iff (item ids INTERSECT ids_host[0..n)) != {}
 * XOR reverse. ids_host needs no order (the library sorts and de-duplicates a copy); n >= 1
 * (an empty list is rejected: omit the clause, reading R3); <= 1024 ids over one query's ID
 * clauses. */
typedef struct {
  const uint64_t* ids_host;
  int32_t n;
  uint8_t slot;
  uint8_t reverse;
  uint8_t pad[2];
} linr_id_clause;

/* Caller-owned device storage for `slots` ID-list slots of widths[s] ids per item (all rows). */
size_t linr_idlists_storage_bytes(const linr_index* index, int32_t slots, const int32_t* widths_host);

/* Attach ID-list slots (setup call: zero-fills the counts synchronously; no row has ids yet). */
int linr_idlists_attach(linr_index* index, int32_t slots, const int32_t* widths_host, void* storage_dev);

/* Write the ID lists of slot `slot` for n rows: rows_dev = global ids (live upsert; out-of-shard
 * ids skipped and counted), or NULL for the contiguous rows [row0, row0+n) (bulk load).
 * ids_dev [n][widths[slot]] u64 (entries past the row's count are ignored), counts_dev [n] u8
 * (<= width). Stream-ordered like linr_index_update_rows. */
int linr_idlists_set_rows(linr_index* index, int32_t slot, const int64_t* rows_dev, int64_t row0, int64_t n,
                          const uint64_t* ids_dev, const uint8_t* counts_dev, void* stream);

/* linr_search with ID-list clauses in addition to the bitmask clauses (CSR by
 * id_clause_off_host[B+1]). The ID clauses of each query are evaluated by a filter kernel into a
 * per-query liveness bitmap (live AND every ID clause); the fused scan then runs one user per
 * launch on that bitmap with the bitmask clauses. Same outputs as linr_search. Workspace:
 * linr_search_idc_workspace_bytes. */
size_t linr_search_idc_workspace_bytes(const linr_index* index, int32_t B, int32_t V, int32_t K);
int linr_search_idc(linr_index* index, const void* queries_dev, int32_t B, int32_t V,
                    const linr_clause* clauses_host, const int32_t* clause_off_host,
                    const linr_id_clause* id_clauses_host, const int32_t* id_clause_off_host, int32_t K,
                    void* ws_dev, size_t ws_bytes, int64_t* out_ids_dev, float* out_scores_dev,
                    int64_t* out_pass_dev, void* stream);

/* ---------------------------------------------------------------- learned scorers (§3.3)
 * The filtered exhaustive search with a learned similarity in place of the dot product, weights
 * supplied by the caller (float32 host arrays, row-major; training is out of scope):
 *  Hadamard MLP (Table 1 "Member & Item MLP [50]+[10, 1]"):
 *     s(q, x) = w2 . ReLU(W1 ((Wm q + bm) (.) (Wi x + bi)) + b1) + b2
 *     Wm, Wi [F][dim]; bm, bi [F]; W1 [H][F]; b1, w2 [H]; b2 [1]
 *  Mixture-of-Logits ("phi_MoL(x, u) = sum_k pi_k(x, u) delta_k(x, u)"):
 *     delta_k = <Fk_k u, Gk_k x> (component k = rows [k*dc, (k+1)*dc) of Fk, Gk [K*dc][dim]),
 *     pi = softmax(Wo ReLU(Wgu u + Wgx x + bg) + bo); Wgu, Wgx [G][dim]; bg [G]; Wo [K][G]; bo [K]
 * The query-independent item side (Wi x + bi; or [Gk x, Wgx x]) is computed once per row at
 * attach time and again whenever rows are loaded, upserted or generated (same stream), so a
 * search evaluates only the per-query remainder on the passing rows. fp32 arithmetic. */
#define LINR_SCORER_HADAMARD 1
#define LINR_SCORER_MOL 2
typedef struct {
  int32_t kind;              /* LINR_SCORER_HADAMARD or LINR_SCORER_MOL                */
  int32_t F, H;              /* Hadamard: member/item width (<= 256), head hidden (<= 64) */
  int32_t K, dc, G;          /* MoL: components (<= 8), component width (multiple of 4), gate hidden (<= 64) */
  const float *Wm, *bm, *Wi, *bi, *W1, *b1, *w2, *b2;
  const float *Fk, *Gk, *Wgu, *Wgx, *bg, *Wo, *bo;
} linr_scorer;

/* Caller-owned device storage for the scorer weights + the item features of every row. */
size_t linr_scorer_storage_bytes(const linr_index* index, const linr_scorer* scorer);
/* Attach a learned scorer (setup call: synchronises `stream`, copies the weights, enqueues the
 * item features of the rows below the high-water mark). EINVAL on bad widths / null weights. */
int linr_scorer_attach(linr_index* index, const linr_scorer* scorer, void* storage_dev, void* stream);
/* Filtered top-K under the attached scorer: queries_dev [B][dim] (one vector per query), clauses
 * as linr_search, K in [1, 2048]; outputs as linr_search (scores fp32, order score desc / id asc). */
size_t linr_search_scored_workspace_bytes(const linr_index* index, int32_t B, int32_t K);
int linr_search_scored(linr_index* index, const void* queries_dev, int32_t B, const linr_clause* clauses_host,
                       const int32_t* clause_off_host, int32_t K, void* ws_dev, size_t ws_bytes,
                       int64_t* out_ids_dev, float* out_scores_dev, int64_t* out_pass_dev, void* stream);

/* Device-side synthetic data generator (benchmark plumbing, not part of the method): fills local
 * rows [row_begin, row_begin+n) of the index with the counter-based recipe of DESIGN.md
 * "Input recipe" (identical bytes to datagen/ in Python), marks them live and raises the
 * high-water mark. Lets 1B-row shards be built in place. mode: 0 integer grid, 1 dense. */
int linr_index_generate(linr_index* index, uint64_t seed, int32_t mode, int64_t row_begin,
                        int64_t n, void* stream);

/* Generate rows [row_begin, row_begin+n) into plain device buffers (no index): emb_dev
 * [n][dim] dtype, attrs_dev [n][W] (either may be NULL). Used by the generator cross-check. */
int linr_generate_rows(int32_t dtype, int32_t dim, int32_t attr_words, uint64_t seed, int32_t mode,
                       int64_t row_begin, int64_t n, void* emb_dev, uint64_t* attrs_dev,
                       void* stream);

/* Stage timing for benchmarks (measured on the search stream with CUDA events, no extra sync
 * on the hot path): while enabled, every linr_search / linr_search_keys / linr_search_host on
 * this index records events around its scan launches and its merge launch.
 * linr_index_profile_read synchronises the recorded events, returns the summed scan and merge
 * milliseconds, the number of searches and the number of this library's kernel launches since
 * the last read, and resets the counters. */
int linr_index_profile(linr_index* index, int enable);
int linr_index_profile_read(linr_index* index, double* scan_ms, double* merge_ms, int64_t* searches,
                            int64_t* kernel_launches);

/* Diagnostics (development only; not needed by users): enable device-side phase timers
 * (%globaltimer ns per CTA phase of the scan and merge kernels) and read them back. */
int linr_debug_timers(int enable);
int linr_debug_read(uint64_t* host, int32_t n);

/* Thread-local message for the last non-OK return on this thread ("" if none). */
const char* linr_last_error(void);

/* ABI version (incremented on any signature change). */
int linr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LINR_H_ */
