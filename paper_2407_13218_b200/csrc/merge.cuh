// Merge of L partition results into the final top-K of one user (CTA-wide device function).
//
// Used twice on the hot path: (a) at the end of the scan, L = number of scan CTAs (partition =
// one CTA's item range; run by the last CTAs of the scan kernel itself, or by merge_kernel);
// (b) after the cross-GPU all-gather, L = number of shards (BASELINE.json north_star: "an NCCL
// allgather of K (score, id) pairs ... feeds a final merge"). Exact by reading R13: the union of
// the partitions' top-Ks contains the global top-K under the total key order (score desc, id asc).
//
// Each partition provides a sorted sample (its top ms keys) and a list of all its candidate keys.
// LB = K-th largest key of the union of the samples is a lower bound of the answer's K-th key
// (those K keys exist), so the answer is {samples >= LB} plus, only for partitions whose whole
// sample is >= LB ("saturated"), their list keys in [LB, sample[ms-1]). For item ranges of
// similar statistics saturation is rare and the merge touches only the samples. If the samples
// hold fewer than K keys, every list key is gathered (exact fallback, in global memory if large).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace linr {

constexpr int kMergeCap = 16384;    // keys staged in shared memory (128 KB)
constexpr int kMergeOut = 4096;     // survivor / sort buffer (32 KB)
constexpr int kMergeRegs = 16;      // sample keys held per thread on the fast path

struct MergeCtl {
  SelScratch sel;
  BucketScratch bs;
  int cnt;
  int nnz;
  long long pass;
};

constexpr size_t merge_smem_bytes() {
  return ((sizeof(MergeCtl) + 15) & ~size_t(15)) + (size_t)(kMergeCap + kMergeOut) * 8;
}

// Append the nonzero keys >= lb among n_items keys get(i) to dst (warp-aggregated); returns the count.
template <int NT, typename Get>
__device__ int merge_gather(uint64_t* dst, int cap, MergeCtl* ctl, int n_items, Get get, uint64_t lb) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) ctl->cnt = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n_items; i0 += NT) {   // uniform trip count: full-warp ballots
    const int i = i0 + tid;
    uint64_t v = 0ull;
    if (i < n_items) v = get(i);
    const bool keep = v != 0ull && v >= lb;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (bal) {
      const int leader = __ffs(bal) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(&ctl->cnt, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, leader);
      const int pos = base + __popc(bal & lanemask_lt());
      if (keep && pos < cap) dst[pos] = v;
    }
  }
  __syncthreads();
  return ctl->cnt;
}

// Warp-aggregated append of v (if keep) at ctl->cnt.
LINR_DEV void merge_append(uint64_t* dst, int cap, MergeCtl* ctl, bool keep, uint64_t v) {
  const int lane = threadIdx.x & 31;
  const uint32_t bal = __ballot_sync(0xffffffffu, keep);
  if (bal) {
    const int leader = __ffs(bal) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&ctl->cnt, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, leader);
    const int pos = base + __popc(bal & lanemask_lt());
    if (keep && pos < cap) dst[pos] = v;
  }
}

// Fast path of step 3+4 when no partition is saturated: the answer is exactly the union of each
// partition's sample prefix >= lb, and each prefix is already sorted (descending). Merge the L
// sorted runs pairwise (ceil(log2 L) rounds); in a round every key finds its merged position as
// (its index in its run) + (keys of the partner run greater than it: a binary search), so a
// round is one parallel scatter. Keys are distinct (ids are part of the key). Writes the n sorted keys
// to the returned buffer (one of b0 / b1). Scratch: b0, b1 >= n keys; rid0, rid1 >= n bytes;
// off0, off1 >= L + 1 ints.
template <int NT>
__device__ uint64_t* merge_sorted_prefixes(const uint64_t* samp, int L, int ms, uint64_t lb, int n, uint64_t* b0,
                                           uint64_t* b1, uint8_t* rid0, uint8_t* rid1, int* off0, int* off1,
                                           int* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  // run lengths (prefix of keys >= lb) and their exclusive scan (L <= NT)
  int c = 0;
  if (tid < L) {
    const uint64_t* r = samp + tid * ms;
    while (c < ms && r[c] != 0ull && r[c] >= lb) ++c;
  }
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  if (tid < L) off0[tid] = base + incl - c;
  if (tid == 0) off0[L] = n;
  __syncthreads();
  for (int i = tid; i < L * ms; i += NT) {   // copy the prefixes, run id = partition index
    const int l = i / ms, j = i - l * ms;
    const int o = off0[l];
    if (o + j < off0[l + 1]) {
      b0[o + j] = samp[i];
      rid0[o + j] = (uint8_t)l;
    }
  }
  __syncthreads();
  // pairwise rounds (ceil(log2 L)); every thread places two keys per iteration, their branchless
  // binary searches (fixed step count) interleaved so the dependent shared-memory loads overlap
  int R = L, maxlen = ms;
  (void)NW;
  while (R > 1) {
    int steps = 0;
    while ((1 << steps) <= maxlen) ++steps;
    for (int i0 = tid; i0 < n; i0 += 2 * NT) {
      const int i1 = i0 + NT;
      const bool h1 = i1 < n;
      const uint64_t x0 = b0[i0], x1 = h1 ? b0[i1] : 0ull;
      const int r0 = rid0[i0], r1 = h1 ? rid0[i1] : r0;
      const int p0 = r0 ^ 1, p1 = r1 ^ 1;
      const int lo0 = p0 < R ? off0[p0] : 0, len0 = p0 < R ? off0[p0 + 1] - lo0 : 0;
      const int lo1 = p1 < R ? off0[p1] : 0, len1 = p1 < R ? off0[p1 + 1] - lo1 : 0;
      int c0 = 0, c1 = 0;   // partner keys greater than x: a prefix (runs are descending)
      for (int b = steps - 1; b >= 0; --b) {
        const int t0 = c0 + (1 << b), t1 = c1 + (1 << b);
        const bool g0 = t0 <= len0 && b0[lo0 + t0 - 1] > x0;
        const bool g1 = t1 <= len1 && b0[lo1 + t1 - 1] > x1;
        c0 = g0 ? t0 : c0;
        c1 = g1 ? t1 : c1;
      }
      const int q0 = off0[r0 & ~1] + (i0 - off0[r0]) + c0;
      b1[q0] = x0;
      rid1[q0] = (uint8_t)(r0 >> 1);
      if (h1) {
        const int q1 = off0[r1 & ~1] + (i1 - off0[r1]) + c1;
        b1[q1] = x1;
        rid1[q1] = (uint8_t)(r1 >> 1);
      }
    }
    const int R2 = (R + 1) >> 1;
    for (int k = tid; k <= R2; k += NT) off1[k] = k < R2 ? off0[2 * k] : n;
    __syncthreads();
    uint64_t* tb = b0; b0 = b1; b1 = tb;
    uint8_t* tr = rid0; rid0 = rid1; rid1 = tr;
    int* to = off0; off0 = off1; off1 = to;
    R = R2;
    maxlen = maxlen * 2 < n ? maxlen * 2 : n;
  }
  return b0;
}

// Decode the n sorted keys of user u into the outputs (padding past n), and the pass count.
template <int NT>
__device__ void merge_write(const MergeParams& p, int u, const uint64_t* sorted, int n, long long pass) {
  const int tid = threadIdx.x, K = p.K;
  if (p.mode == 0) {
    for (int j = tid; j < K; j += NT) {
      const int64_t at = (int64_t)u * K + j;
      if (j < n) {
        p.out_ids[at] = key_id(sorted[j]);
        p.out_scores[at] = key_score(sorted[j]);
      } else {
        p.out_ids[at] = -1;
        p.out_scores[at] = -INFINITY;
      }
    }
  } else {
    for (int j = tid; j < K; j += NT) p.out_keys[(int64_t)u * K + j] = (j < n) ? sorted[j] : 0ull;
  }
  if (tid == 0 && p.out_pass) p.out_pass[u] = pass;
  // union path: the scan kept only keys >= thr[u]; fewer than K of them (while the user has K
  // passers above 0) means the result is not provably the top-K -> recomputed exactly
  if (tid == 0 && p.flags) p.flags[u] = (p.thr != nullptr && p.thr[u] != 0ull && n < K) ? 1 : 0;
}

template <int NT>
__device__ void merge_user(const MergeParams& p, int u, unsigned char* smem) {
  MergeCtl* ctl = reinterpret_cast<MergeCtl*>(smem);
  uint64_t* s = reinterpret_cast<uint64_t*>(smem + ((sizeof(MergeCtl) + 15) & ~size_t(15)));
  uint64_t* s2 = s + kMergeCap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int L = p.L, K = p.K, ms = p.ms;
  const uint64_t* samp = p.samp + (int64_t)u * p.samp_su;
  const uint64_t* list = p.list + (int64_t)u * p.list_su;
  const int64_t ssl = p.samp_sl, lsl = p.list_sl, csl = p.cnt_sl;
  const int* cntp = p.cnt ? p.cnt + (int64_t)u * p.cnt_su : nullptr;
  const int len = p.list_len;
  const int DB = 4096 + u * 8;
  dbg_mark(p.dbg, DB + 0);

  if (tid == 0) { ctl->nnz = 0; ctl->cnt = 0; ctl->pass = 0; }
  __syncthreads();
  {   // pass counts: all loads in flight at once
    long long acc = 0;
    if (p.pass)
      for (int l = tid; l < L; l += NT) acc += p.pass[(int64_t)l * p.pstride_l + (int64_t)u * p.pstride_u];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd((unsigned long long*)&ctl->pass, (unsigned long long)acc);
  }
  auto lcount = [cntp, csl, len](int l) -> int { return cntp ? cntp[(int64_t)l * csl] : len; };
  __syncthreads();

  int n = -1;
  const int ns = L * ms;
  if (ns <= kMergeRegs * NT && ns <= kMergeCap) {
    // 1. samples: batched loads into registers (all in flight at once), copy to shared memory
    uint64_t r[kMergeRegs];
#pragma unroll
    for (int e = 0; e < kMergeRegs; ++e) {
      const int i = tid + e * NT;
      r[e] = 0ull;
      if (i < ns) {
        const int l = i / ms;
        r[e] = samp[(int64_t)l * ssl + (i - l * ms)];
      }
    }
    int nz = 0;
#pragma unroll
    for (int e = 0; e < kMergeRegs; ++e) {
      const int i = tid + e * NT;
      if (i < ns) {
        s[i] = r[e];
        nz += r[e] != 0ull;
      }
    }
    for (int o = 16; o; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    if (lane == 0 && nz) atomicAdd(&ctl->nnz, nz);
    __syncthreads();
    dbg_mark(p.dbg, DB + 1);
    if (ctl->nnz >= K) {
      // 2. LB = K-th largest sample key (zero padding sorts below it)
      const uint64_t lb = block_select_ge<NT>([s](int i) { return s[i]; }, ns, K, &ctl->sel);
      dbg_mark(p.dbg, DB + 2);
      // no saturated partition (every sample holds a key < lb): the answer is the K sample keys
      // >= lb, already sorted within each partition -> merge the sorted prefixes
      if (tid == 0) ctl->cnt = 0;
      __syncthreads();
      bool sat = false;
      for (int l = tid; l < L; l += NT) sat = sat || s[l * ms + ms - 1] >= lb;
      if (__syncthreads_or(sat) == 0 && !p.bucket_sort && L <= NT && L <= 256 && K <= 4096) {
        dbg_mark(p.dbg, DB + 3);
        dbg_mark(p.dbg, DB + 4);
        uint64_t* b1 = s + 8192;
        uint8_t* rid = reinterpret_cast<uint8_t*>(s + 12288);
        int* offs = reinterpret_cast<int*>(s + 14336);
        const uint64_t* sorted = merge_sorted_prefixes<NT>(s, L, ms, lb, K, s2, b1, rid, rid + 4096, offs, offs + 512,
                                                           offs + 1024);
        dbg_mark(p.dbg, DB + 5);
        merge_write<NT>(p, u, sorted, K, ctl->pass);
        dbg_mark(p.dbg, DB + 6);
        if (p.dbg != nullptr && tid == 0) p.dbg[DB + 7] = (unsigned long long)K;
        __syncthreads();
        return;
      }
      // 3. survivors: sample keys >= lb (exactly K) + saturated partitions' keys in [lb, last)
#pragma unroll
      for (int e = 0; e < kMergeRegs; ++e) merge_append(s2, kMergeOut, ctl, r[e] != 0ull && r[e] >= lb, r[e]);
      for (int l = warp; l < L; l += NW) {
        const uint64_t last = s[l * ms + ms - 1];   // the sample is staged in shared memory
        if (last < lb) continue;   // warp-uniform
        const int c = lcount(l);
        const uint64_t* lp = list + (int64_t)l * lsl;
        for (int j0 = 0; j0 < c; j0 += 32) {
          const int j = j0 + lane;
          const uint64_t v = j < c ? lp[j] : 0ull;
          merge_append(s2, kMergeOut, ctl, v != 0ull && v >= lb && v < last, v);
        }
      }
      __syncthreads();
      n = ctl->cnt;
      if (n > kMergeOut) n = -1;
    }
  }
  dbg_mark(p.dbg, DB + 3);
  if (n < 0) {
    // exact fallback: every list key (a partition's list includes its sample keys)
    const int items = L * len;
    auto get = [list, lsl, len, lcount](int i) -> uint64_t {
      const int l = i / len, j = i - l * len;
      return j < lcount(l) ? list[(int64_t)l * lsl + j] : 0ull;
    };
    int n1 = merge_gather<NT>(s, kMergeCap, ctl, items, get, 1ull);
    if (n1 > kMergeCap) {
      // zeros sort below every real key and K <= n1, so they are never selected
      const uint64_t T = block_select_ge<NT>(get, items, K, &ctl->sel);
      n1 = merge_gather<NT>(s, kMergeCap, ctl, items, get, T);
    }
    if (n1 > K) {
      const uint64_t T = block_select_ge<NT>([s](int i) { return s[i]; }, n1, K, &ctl->sel);
      n1 = block_compact_ge<NT>(s, n1, T, &ctl->sel);
    }
    for (int i = tid; i < n1; i += NT) s2[i] = s[i];
    __syncthreads();
    n = n1;
  } else if (n > K) {
    const uint64_t T = block_select_ge<NT>([s2](int i) { return s2[i]; }, n, K, &ctl->sel);
    n = block_compact_ge<NT>(s2, n, T, &ctl->sel);
  }
  dbg_mark(p.dbg, DB + 4);
  // 4. sort the <= K survivors: bucket sort, general bitonic if a bucket is too full
  const uint64_t* sorted = s;
  const bool bucket_ok = block_bucket_sort_desc<NT>(s2, n, s, &ctl->bs);
  if (p.dbg != nullptr && tid == 0) p.dbg[6144 + u * 4 + 0] = (unsigned long long)ctl->bs.maxb | ((unsigned long long)bucket_ok << 32);
  if (!bucket_ok) {
    const int P2 = next_pow2(n > 1 ? n : 1);
    for (int i = n + tid; i < P2; i += NT) s2[i] = 0ull;
    __syncthreads();
    block_sort_desc<NT>(s2, P2);
    sorted = s2;
  }
  dbg_mark(p.dbg, DB + 5);

  merge_write<NT>(p, u, sorted, n, ctl->pass);
  dbg_mark(p.dbg, DB + 6);
  if (p.dbg != nullptr && tid == 0) p.dbg[DB + 7] = (unsigned long long)n;
  __syncthreads();
}

}  // namespace linr
