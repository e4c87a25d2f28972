// LiNR pre-filtered exhaustive top-K oracle — TEST INFRASTRUCTURE ONLY.
//
// Plain, slow, obviously-correct CPU definition of what the GPU hot path computes
// (arXiv 2407.13218, §3.1 "Exhaustive Search with Attribute-Based Matching").
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load this library. It shares no code, header, table or helper with the CUDA library
// under paper_2407_13218_b200/csrc, and it does not include include/linr.h.
//
// What it computes, per query b:
//   C = { (s_i, id_i) : i < n, live[i], every clause of b passes on item i }
//     clause (mask m, word w, reverse r) passes  <=>  ((A[i][w] & m) != 0) XOR r
//        "Feasible items should satisfy all clauses, requiring at least one of the
//        attribute in each clauses is matched. Reverse clauses are also supported."
//        (attributes as a bitmask over a small universe: reading R2 in DESIGN.md)
//     s_i = max_v <q_{b,v}, x_i>   dot product ("dot-product similarity"); max over the
//        user's V query vectors (multi-embedding, reading R12); float inputs widened exactly to
//        double and summed in double in index order; int8 summed exactly in int64.
//   pass[b] = |C|
//   out[b]  = first min(K, |C|) of C sorted by (score desc, id asc)   ("Top-1 selection";
//        ties by lower id: reading R5), remaining slots (-1, -inf)     (reading R6)
//   Filtered items are excluded, never scored as 0 (reading R1; V1's "map ... to zero").
//
// Parity pins for every function here live in tests/test_oracle.py (-m "not gpu").

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

namespace {

enum { O_F32 = 0, O_F16 = 1, O_BF16 = 2, O_I8 = 3 };

// IEEE-754 binary16 -> double, exact (definition of the format, not a library call).
double widen_f16(uint16_t h) {
  const int sign = (h >> 15) & 1;
  const int e = (h >> 10) & 0x1F;
  const int m = h & 0x3FF;
  double v;
  if (e == 0) {
    v = std::ldexp((double)m, -24);                 // subnormal: m * 2^-24
  } else if (e == 31) {
    v = m ? std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::infinity();
  } else {
    v = std::ldexp((double)(m + 1024), e - 25);     // (1 + m/1024) * 2^(e-15)
  }
  return sign ? -v : v;
}

// bfloat16 -> double, exact: bf16 is the top half of an fp32 bit pattern.
double widen_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return (double)f;
}

double elem(const void* base, int dtype, int64_t idx) {
  switch (dtype) {
    case O_F32: return (double)((const float*)base)[idx];
    case O_F16: return widen_f16(((const uint16_t*)base)[idx]);
    case O_BF16: return widen_bf16(((const uint16_t*)base)[idx]);
    default: return (double)((const int8_t*)base)[idx];
  }
}

struct Clause {        // the oracle's own clause record (layout chosen to match the test marshalling)
  uint64_t mask;
  uint8_t word;
  uint8_t reverse;
  uint8_t pad[6];
};

bool item_passes(const uint64_t* attrs, int W, int64_t i, const Clause* cl, int ncl) {
  for (int c = 0; c < ncl; ++c) {
    const bool hit = (attrs[i * W + cl[c].word] & cl[c].mask) != 0;   // OR within the clause
    const bool ok = cl[c].reverse ? !hit : hit;                       // Reverse: no attribute matches
    if (!ok) return false;                                            // AND across clauses
  }
  return true;
}

double dot(const void* emb, const void* q, int dtype, int d, int64_t row) {
  if (dtype == O_I8) {
    int64_t acc = 0;
    const int8_t* x = (const int8_t*)emb + row * d;
    const int8_t* y = (const int8_t*)q;
    for (int j = 0; j < d; ++j) acc += (int64_t)x[j] * (int64_t)y[j];
    return (double)acc;
  }
  double acc = 0.0;
  for (int j = 0; j < d; ++j) acc += elem(emb, dtype, row * d + j) * elem(q, dtype, j);
  return acc;
}

struct Cand {
  double s;
  int64_t id;
};

bool better(const Cand& a, const Cand& b) {   // score desc, then id asc; -0.0 == +0.0 in double compare
  if (a.s != b.s) return a.s > b.s;
  return a.id < b.id;
}

}  // namespace

extern "C" {

int oracle_version(void) { return 1; }

// Exact widening of one stored element (pinned against IEEE bit patterns in the tests).
double oracle_widen(int dtype, uint32_t bits) {
  if (dtype == O_F16) return widen_f16((uint16_t)bits);
  if (dtype == O_BF16) return widen_bf16((uint16_t)bits);
  if (dtype == O_I8) return (double)(int8_t)(uint8_t)bits;
  float f;
  std::memcpy(&f, &bits, 4);
  return (double)f;
}

// Joint pre-filter mask (Fig. 2 caption: "a joint 0-1 mask vector").
// attrs: [n][W] row-major; live: [n] 0/1. Returns pass count.
int64_t oracle_filter(const uint64_t* attrs, int W, int64_t n, const uint8_t* live,
                      const void* clauses, int ncl, uint8_t* out_mask) {
  const Clause* cl = (const Clause*)clauses;
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    const bool p = live[i] && item_passes(attrs, W, i, cl, ncl);
    out_mask[i] = p ? 1 : 0;
    cnt += p;
  }
  return cnt;
}

// Scores of every row (no filter) for one query vector: s_i = <q, x_i>. Used by pins.
void oracle_scores(int dtype, int d, int64_t n, const void* emb, const void* q, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = dot(emb, q, dtype, d, i);
}

// The filtered exhaustive top-K (the whole hot path, one shard = the whole index).
//   emb     [n][d] in dtype (f32 / f16 bits / bf16 bits / int8)
//   attrs   [n][W] u64;   live [n] u8;   row0 = global id of local row 0
//   queries [B][V][d] in dtype;   clauses: CSR by clause_off[B+1]
//   out_ids [B][K] i64, out_scores [B][K] f64, out_pass [B] i64
// Returns 0, or -1 on a violated precondition (K<1, B<1, V<1, d<1, W<1, bad clause word,
// empty clause mask: reading R3).
int oracle_search(int dtype, int d, int64_t n, int64_t row0, const void* emb,
                  const uint64_t* attrs, int W, const uint8_t* live,
                  const void* queries, int B, int V,
                  const void* clauses, const int32_t* clause_off, int K,
                  int64_t* out_ids, double* out_scores, int64_t* out_pass) {
  if (K < 1 || B < 1 || V < 1 || d < 1 || W < 1 || n < 0) return -1;
  const Clause* cl_all = (const Clause*)clauses;
  const int64_t qstride = (int64_t)d * (dtype == O_F32 ? 4 : dtype == O_I8 ? 1 : 2);
  for (int b = 0; b < B; ++b) {
    const int c0 = clause_off[b], c1 = clause_off[b + 1];
    if (c1 < c0) return -1;
    for (int c = c0; c < c1; ++c)
      if (cl_all[c].word >= W || cl_all[c].mask == 0) return -1;
  }
  for (int b = 0; b < B; ++b) {
    const Clause* cl = cl_all + clause_off[b];
    const int ncl = clause_off[b + 1] - clause_off[b];
    std::vector<Cand> C;
    for (int64_t i = 0; i < n; ++i) {
      if (!live[i]) continue;
      if (!item_passes(attrs, W, i, cl, ncl)) continue;
      double s = -std::numeric_limits<double>::infinity();
      for (int v = 0; v < V; ++v) {
        const void* q = (const char*)queries + ((int64_t)b * V + v) * qstride;
        s = std::max(s, dot(emb, q, dtype, d, i));
      }
      if (s == 0.0) s = 0.0;   // canonicalise -0.0
      C.push_back({s, row0 + i});
    }
    std::sort(C.begin(), C.end(), better);
    out_pass[b] = (int64_t)C.size();
    for (int j = 0; j < K; ++j) {
      if (j < (int64_t)C.size()) {
        out_ids[(int64_t)b * K + j] = C[j].id;
        out_scores[(int64_t)b * K + j] = C[j].s;
      } else {
        out_ids[(int64_t)b * K + j] = -1;
        out_scores[(int64_t)b * K + j] = -std::numeric_limits<double>::infinity();
      }
    }
  }
  return 0;
}

// ID-list clauses ("Each query clause could contain multiple attributes. Feasible
// items should satisfy all clauses, requiring at least one of the attribute in each clauses is
// matched. Reverse clauses are also supported ... we store all clause attributes in a single
// matrix ... and have an extra counting matrix to record the number of attributes for each item in
// each clause"; attributes "converted to 64-bit integers"). Item i's attribute set in slot
// s = the first counts[s][i] entries of ids[s][i][0..A_s); a clause (slot, reverse, query id list)
// passes iff (item set INTERSECT query set is non-empty) XOR reverse -- a literal double loop here.
struct IdClause {       // the oracle's own record: 16 B
  const uint64_t* ids;
  int32_t n;
  uint8_t slot;
  uint8_t reverse;
  uint8_t pad[2];
};

bool id_clause_passes(const uint64_t* const* slot_ids, const int32_t* slot_width, const uint8_t* const* slot_counts,
                      int64_t i, const IdClause& c) {
  const int A = slot_width[c.slot];
  const int cnt = slot_counts[c.slot][i];
  bool hit = false;
  for (int a = 0; a < cnt; ++a)
    for (int q = 0; q < c.n; ++q)
      if (slot_ids[c.slot][i * A + a] == c.ids[q]) hit = true;
  return c.reverse ? !hit : hit;
}

// Filtered top-K with bitmask clauses AND ID-list clauses (same definition as oracle_search plus
// the ID-list clauses of each query). slot_ids[s]: [n][A_s] u64 row-major, slot_counts[s]: [n].
int oracle_search_idc(int dtype, int d, int64_t n, int64_t row0, const void* emb, const uint64_t* attrs, int W,
                      const uint8_t* live, int S, const uint64_t* const* slot_ids, const int32_t* slot_width,
                      const uint8_t* const* slot_counts, const void* queries, int B, int V, const void* clauses,
                      const int32_t* clause_off, const void* id_clauses, const int32_t* id_off, int K,
                      int64_t* out_ids, double* out_scores, int64_t* out_pass) {
  if (K < 1 || B < 1 || V < 1 || d < 1 || W < 1 || n < 0 || S < 0) return -1;
  const Clause* cl_all = (const Clause*)clauses;
  const IdClause* ic_all = (const IdClause*)id_clauses;
  const int64_t qstride = (int64_t)d * (dtype == O_F32 ? 4 : dtype == O_I8 ? 1 : 2);
  for (int b = 0; b < B; ++b) {
    if (clause_off[b + 1] < clause_off[b] || id_off[b + 1] < id_off[b]) return -1;
    for (int c = clause_off[b]; c < clause_off[b + 1]; ++c)
      if (cl_all[c].word >= W || cl_all[c].mask == 0) return -1;
    for (int c = id_off[b]; c < id_off[b + 1]; ++c)
      if (ic_all[c].slot >= S || ic_all[c].n < 1) return -1;   // an empty ID list is rejected (reading R3)
  }
  for (int b = 0; b < B; ++b) {
    const Clause* cl = cl_all + clause_off[b];
    const int ncl = clause_off[b + 1] - clause_off[b];
    std::vector<Cand> C;
    for (int64_t i = 0; i < n; ++i) {
      if (!live[i]) continue;
      if (!item_passes(attrs, W, i, cl, ncl)) continue;
      bool ok = true;
      for (int c = id_off[b]; c < id_off[b + 1]; ++c)
        if (!id_clause_passes(slot_ids, slot_width, slot_counts, i, ic_all[c])) ok = false;
      if (!ok) continue;
      double s = -std::numeric_limits<double>::infinity();
      for (int v = 0; v < V; ++v) {
        const void* q = (const char*)queries + ((int64_t)b * V + v) * qstride;
        s = std::max(s, dot(emb, q, dtype, d, i));
      }
      if (s == 0.0) s = 0.0;
      C.push_back({s, row0 + i});
    }
    std::sort(C.begin(), C.end(), better);
    out_pass[b] = (int64_t)C.size();
    for (int j = 0; j < K; ++j) {
      const int64_t at = (int64_t)b * K + j;
      out_ids[at] = j < (int64_t)C.size() ? C[j].id : -1;
      out_scores[at] = j < (int64_t)C.size() ? C[j].s : -std::numeric_limits<double>::infinity();
    }
  }
  return 0;
}

// Union of L result lists for the same B queries (one per shard), then top-K by the same order.
// ids/scores: [L][B][Kin] (-1 padded); pass: [L][B]. Output [B][K], pass summed.
// Definition used for sharding (reading R13): result on the concatenated index.
int oracle_merge(int L, int B, int Kin, const int64_t* ids, const double* scores,
                 const int64_t* pass, int K, int64_t* out_ids, double* out_scores,
                 int64_t* out_pass) {
  if (L < 1 || B < 1 || Kin < 1 || K < 1) return -1;
  for (int b = 0; b < B; ++b) {
    std::vector<Cand> C;
    int64_t p = 0;
    for (int l = 0; l < L; ++l) {
      p += pass[(int64_t)l * B + b];
      for (int j = 0; j < Kin; ++j) {
        const int64_t at = ((int64_t)l * B + b) * Kin + j;
        if (ids[at] >= 0) C.push_back({scores[at], ids[at]});
      }
    }
    std::sort(C.begin(), C.end(), better);
    out_pass[b] = p;
    for (int j = 0; j < K; ++j) {
      const int64_t at = (int64_t)b * K + j;
      if (j < (int64_t)C.size()) { out_ids[at] = C[j].id; out_scores[at] = C[j].s; }
      else { out_ids[at] = -1; out_scores[at] = -std::numeric_limits<double>::infinity(); }
    }
  }
  return 0;
}

}  // extern "C"
