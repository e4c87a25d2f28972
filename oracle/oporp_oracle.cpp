// Sign-OPORP 1-bit codes, matched-bit scoring and the V3 two-stage search — TEST INFRASTRUCTURE ONLY.
//
// Plain, slow CPU definitions of what the quantised path computes (arXiv 2407.13218 §3.2
// "Quantized KNN", Fig. 3 caption P:4310). Same rules as linr_oracle.cpp: only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
// this code; it shares nothing with paper_2407_13218_b200/csrc and does not include linr.h.
//
// Sign-OPORP ("single random projection with fixed-length binning scheme ... takes the
// sign of the projected embedding to generate 1-bit embedding"): the projection
// parameters are ONE permutation and ONE random sign vector of length L, passed in as
//   src[p]  = the input coordinate placed at position p (or -1: a zero padding entry),
//   sign[p] = +1 / -1,
// for p in [0, L), L = k * b. Bin j (of k) is the contiguous positions [j*b, (j+1)*b); its value
// is the sum, in position order, of sign[p] * x[src[p]] (each term widened exactly to double and
// summed in double); bit j = 1 iff the bin value >= 0 (sign(0) = +). Codes are packed
// LSB-first in k/64 u64 words (bit j = word j/64, bit j%64). How src/sign are drawn
// (permutation of the padded or replicated vector) is DESIGN.md reading R25; the oracle takes
// them as inputs.
//
// Matched bits (Fig. 3 caption: "bit-wise XOR ... integer bit-wise NOT ... number of matched
// bits"): m(a, b) = #{j : bit_j(a) == bit_j(b)}, here a literal per-bit loop.
// Multi-vector users (reading R12): m = max over the user's V query codes.
//
// Code search (Fig. 3 caption: "The quantized KNN module can be used without full precision
// matrix multiplication when K is large in top-K selection"; P:4665 top-50M of 1B): the passing
// items (the clause filter of linr_oracle.cpp) ordered by (m desc, id asc), the first
// min(K, pass) returned; K may be as large as the index (huge-K selection).
//
// V3 (Fig. 3 / P:4297 "leverage the approximated similarity as an extra pre-filtering step to
// reduce the computation of the full-precision matrix multiplication"):
//   stage 1 clause filter; stage 2 matched bits of every passing item, keep the first
//   K' = min(pass, max(K, ceil(keep * pass))) in (m desc, id asc) order; stage 3 full-precision
//   dot product (fp64 of exactly widened inputs, max over V) of the kept items, top-K by
//   (score desc, id asc). keep = 1 reproduces the exact search.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

namespace {

enum { O_F32 = 0, O_F16 = 1, O_BF16 = 2, O_I8 = 3 };

double widen16(uint16_t h) {   // IEEE binary16 -> double, exact
  const int s = (h >> 15) & 1, e = (h >> 10) & 0x1F, m = h & 0x3FF;
  double v;
  if (e == 0) v = std::ldexp((double)m, -24);
  else if (e == 31) v = m ? std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::infinity();
  else v = std::ldexp((double)(m + 1024), e - 25);
  return s ? -v : v;
}

double widenbf(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return (double)f;
}

double value(const void* base, int dtype, int64_t idx) {
  switch (dtype) {
    case O_F32: return (double)((const float*)base)[idx];
    case O_F16: return widen16(((const uint16_t*)base)[idx]);
    case O_BF16: return widenbf(((const uint16_t*)base)[idx]);
    default: return (double)((const int8_t*)base)[idx];
  }
}

// one vector x (d elements of dtype at base + row*d) -> k bits
void encode_one(const void* base, int dtype, int d, int64_t row, int k, int L, const int32_t* src,
                const int8_t* sign, uint64_t* code) {
  const int b = L / k;
  for (int w = 0; w < k / 64; ++w) code[w] = 0;
  for (int j = 0; j < k; ++j) {
    double s = 0.0;
    for (int p = j * b; p < (j + 1) * b; ++p) {
      const double x = src[p] < 0 ? 0.0 : value(base, dtype, row * d + src[p]);
      s = s + (sign[p] > 0 ? x : -x);
    }
    if (s >= 0.0) code[j / 64] |= 1ull << (j % 64);
  }
}

int matched(const uint64_t* a, const uint64_t* b, int k) {
  int m = 0;
  for (int j = 0; j < k; ++j) {
    const int ba = (int)((a[j / 64] >> (j % 64)) & 1ull);
    const int bb = (int)((b[j / 64] >> (j % 64)) & 1ull);
    if (ba == bb) ++m;
  }
  return m;
}

struct Clause {
  uint64_t mask;
  uint8_t word;
  uint8_t reverse;
  uint8_t pad[6];
};

bool passes(const uint64_t* attrs, int W, int64_t i, const Clause* cl, int ncl) {
  for (int c = 0; c < ncl; ++c) {
    const bool hit = (attrs[i * W + cl[c].word] & cl[c].mask) != 0;
    if (cl[c].reverse ? hit : !hit) return false;
  }
  return true;
}

bool clauses_ok(const Clause* cl, const int32_t* off, int B, int W) {
  for (int b = 0; b < B; ++b) {
    if (off[b + 1] < off[b]) return false;
    for (int c = off[b]; c < off[b + 1]; ++c)
      if (cl[c].word >= W || cl[c].mask == 0) return false;
  }
  return true;
}

struct IntCand {
  int m;
  int64_t id;
  int64_t row;
};
bool int_better(const IntCand& a, const IntCand& b) {
  if (a.m != b.m) return a.m > b.m;
  return a.id < b.id;
}
struct FCand {
  double s;
  int64_t id;
};
bool f_better(const FCand& a, const FCand& b) {
  if (a.s != b.s) return a.s > b.s;
  return a.id < b.id;
}

bool params_ok(int d, int k, int L, const int32_t* src, const int8_t* sign) {
  if (d < 1 || k < 64 || k % 64 || L < k || L % k) return false;
  for (int p = 0; p < L; ++p) {
    if (src[p] >= d || src[p] < -1) return false;
    if (sign[p] != 1 && sign[p] != -1) return false;
  }
  return true;
}

// per query b: matched bits of every passing item (max over V), sorted (m desc, id asc)
std::vector<IntCand> code_candidates(int dtype, int d, int64_t n, int64_t row0, const void* emb,
                                     const std::vector<uint64_t>& icodes, const uint64_t* attrs, int W,
                                     const uint8_t* live, const std::vector<uint64_t>& qcodes, int b, int V,
                                     const Clause* cl, int ncl, int k) {
  (void)dtype;
  (void)d;
  (void)emb;
  const int words = k / 64;
  std::vector<IntCand> C;
  for (int64_t i = 0; i < n; ++i) {
    if (!live[i] || !passes(attrs, W, i, cl, ncl)) continue;
    int m = -1;
    for (int v = 0; v < V; ++v)
      m = std::max(m, matched(&qcodes[((size_t)b * V + v) * words], &icodes[(size_t)i * words], k));
    C.push_back({m, row0 + i, i});
  }
  std::sort(C.begin(), C.end(), int_better);
  return C;
}

}  // namespace

extern "C" {

// codes [n][k/64] of rows emb [n][d] (dtype). Returns 0, or -1 on bad parameters.
int oracle_oporp_encode(int dtype, int d, int64_t n, const void* emb, int k, int L, const int32_t* src,
                        const int8_t* sign, uint64_t* out_codes) {
  if (!params_ok(d, k, L, src, sign) || n < 0) return -1;
  for (int64_t i = 0; i < n; ++i) encode_one(emb, dtype, d, i, k, L, src, sign, out_codes + i * (k / 64));
  return 0;
}

// m(a_i, b_i) for n pairs of k-bit codes (per-bit loop)
int oracle_matched_bits(int k, int64_t n, const uint64_t* a, const uint64_t* b, int32_t* out) {
  if (k < 64 || k % 64) return -1;
  for (int64_t i = 0; i < n; ++i) out[i] = matched(a + i * (k / 64), b + i * (k / 64), k);
  return 0;
}

// Code search: out_ids [B][K], out_m [B][K] (-1 padding), out_pass [B].
int oracle_code_search(int dtype, int d, int64_t n, int64_t row0, const void* emb, const uint64_t* attrs, int W,
                       const uint8_t* live, const void* queries, int B, int V, const void* clauses,
                       const int32_t* clause_off, int64_t K, int k, int L, const int32_t* src, const int8_t* sign,
                       int64_t* out_ids, int32_t* out_m, int64_t* out_pass) {
  const Clause* cl = (const Clause*)clauses;
  if (K < 1 || B < 1 || V < 1 || W < 1 || n < 0 || !params_ok(d, k, L, src, sign) || !clauses_ok(cl, clause_off, B, W))
    return -1;
  const int words = k / 64;
  std::vector<uint64_t> icodes((size_t)n * words), qcodes((size_t)B * V * words);
  for (int64_t i = 0; i < n; ++i) encode_one(emb, dtype, d, i, k, L, src, sign, &icodes[(size_t)i * words]);
  for (int64_t j = 0; j < (int64_t)B * V; ++j) encode_one(queries, dtype, d, j, k, L, src, sign, &qcodes[(size_t)j * words]);
  for (int b = 0; b < B; ++b) {
    std::vector<IntCand> C = code_candidates(dtype, d, n, row0, emb, icodes, attrs, W, live, qcodes, b, V,
                                             cl + clause_off[b], clause_off[b + 1] - clause_off[b], k);
    out_pass[b] = (int64_t)C.size();
    for (int64_t j = 0; j < K; ++j) {
      const int64_t at = (int64_t)b * K + j;
      out_ids[at] = j < (int64_t)C.size() ? C[j].id : -1;
      out_m[at] = j < (int64_t)C.size() ? C[j].m : -1;
    }
  }
  return 0;
}

// V3 two-stage search: out_ids [B][K], out_scores [B][K] (fp64; -inf padding), out_pass [B],
// out_kept [B] = K' (items reranked at full precision).
int oracle_search_v3(int dtype, int d, int64_t n, int64_t row0, const void* emb, const uint64_t* attrs, int W,
                     const uint8_t* live, const void* queries, int B, int V, const void* clauses,
                     const int32_t* clause_off, int K, double keep, int k, int L, const int32_t* src,
                     const int8_t* sign, int64_t* out_ids, double* out_scores, int64_t* out_pass, int64_t* out_kept) {
  const Clause* cl = (const Clause*)clauses;
  if (K < 1 || B < 1 || V < 1 || W < 1 || n < 0 || !(keep > 0.0 && keep <= 1.0) || !params_ok(d, k, L, src, sign) ||
      !clauses_ok(cl, clause_off, B, W))
    return -1;
  const int words = k / 64;
  std::vector<uint64_t> icodes((size_t)n * words), qcodes((size_t)B * V * words);
  for (int64_t i = 0; i < n; ++i) encode_one(emb, dtype, d, i, k, L, src, sign, &icodes[(size_t)i * words]);
  for (int64_t j = 0; j < (int64_t)B * V; ++j) encode_one(queries, dtype, d, j, k, L, src, sign, &qcodes[(size_t)j * words]);
  for (int b = 0; b < B; ++b) {
    std::vector<IntCand> C = code_candidates(dtype, d, n, row0, emb, icodes, attrs, W, live, qcodes, b, V,
                                             cl + clause_off[b], clause_off[b + 1] - clause_off[b], k);
    const int64_t pass = (int64_t)C.size();
    const int64_t want = (int64_t)std::ceil(keep * (double)pass);
    const int64_t kept = std::min(pass, std::max((int64_t)K, want));
    std::vector<FCand> F;
    for (int64_t j = 0; j < kept; ++j) {
      double s = -std::numeric_limits<double>::infinity();
      for (int v = 0; v < V; ++v) {
        double acc = 0.0;
        for (int t = 0; t < d; ++t)
          acc += value(emb, dtype, C[j].row * d + t) * value(queries, dtype, ((int64_t)b * V + v) * d + t);
        s = std::max(s, acc);
      }
      if (s == 0.0) s = 0.0;   // -0.0 -> +0.0
      F.push_back({s, C[j].id});
    }
    std::sort(F.begin(), F.end(), f_better);
    out_pass[b] = pass;
    out_kept[b] = kept;
    for (int j = 0; j < K; ++j) {
      const int64_t at = (int64_t)b * K + j;
      out_ids[at] = j < (int64_t)F.size() ? F[j].id : -1;
      out_scores[at] = j < (int64_t)F.size() ? F[j].s : -std::numeric_limits<double>::infinity();
    }
  }
  return 0;
}

}  // extern "C"
