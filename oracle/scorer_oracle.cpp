// Learned similarity scorers for the filtered exhaustive search — TEST INFRASTRUCTURE ONLY.
//
// Plain fp64 forward passes (arXiv 2407.13218 §3.3 "Similarity Modeling"; SPEC
// S:240-262 for the layer conventions), used in place of the dot product by the same filtered
// top-K definition as linr_oracle.cpp. Same rules: only tests/, smoke() and bench.py's CPU legs
// load this; it shares nothing with the CUDA library.
//
// Hadamard MLP ("A MLP block is applied to member and item embedding respectively, whose
// output performs hadamard product and then passes to another MLP block to output the final
// logit"; Table 1 "Member & Item MLP [50]+[10, 1]"): member and item MLPs are one linear layer
// each (dim -> F), the head is Linear(F -> H) + ReLU + Linear(H -> 1) (ReLU hidden,
// linear outputs):
//     s(q, x) = w2 . ReLU(W1 (h_q (.) h_x) + b1) + b2,   h_q = Wm q + bm,  h_x = Wi x + bi.
// Mixture-of-Logits ("phi_MoL(x, u) = sum_k pi_k(x, u) delta_k(x, u) ... soft-max gate
// given input of user and item features"): K components with user / item projections
// f_k(u) = Fk u, g_k(x) = Gk x (dc each), delta_k = <f_k(u), g_k(x)>; the gate is one hidden
// ReLU layer over the concatenated user and item features, a = ReLU(Wgu u + Wgx x + bg), then
// logits = Wo a + bo, pi = softmax(logits):
//     s(u, x) = sum_k pi_k delta_k.
// All weights are float32 inputs (synthetic; training is out of scope), widened exactly to fp64.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

namespace {

enum { O_F32 = 0, O_F16 = 1, O_BF16 = 2, O_I8 = 3 };

double w16(uint16_t h) {
  const int s = (h >> 15) & 1, e = (h >> 10) & 0x1F, m = h & 0x3FF;
  double v;
  if (e == 0) v = std::ldexp((double)m, -24);
  else if (e == 31) v = m ? std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::infinity();
  else v = std::ldexp((double)(m + 1024), e - 25);
  return s ? -v : v;
}
double wbf(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return (double)f;
}
double val(const void* base, int dtype, int64_t idx) {
  switch (dtype) {
    case O_F32: return (double)((const float*)base)[idx];
    case O_F16: return w16(((const uint16_t*)base)[idx]);
    case O_BF16: return wbf(((const uint16_t*)base)[idx]);
    default: return (double)((const int8_t*)base)[idx];
  }
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

}  // namespace

extern "C" {

// The oracle's view of the scorer weights (all float32, row-major). kind 1 = Hadamard, 2 = MoL.
struct OracleScorer {
  int32_t kind;
  int32_t F, H;            // Hadamard: F = member/item width, H = head hidden width
  int32_t K, dc, G;        // MoL: K components of width dc, gate hidden width G
  const float* Wm; const float* bm;     // [F][d], [F]
  const float* Wi; const float* bi;     // [F][d], [F]
  const float* W1; const float* b1;     // [H][F], [H]
  const float* w2; const float* b2;     // [H], [1]
  const float* Fk; const float* Gk;     // [K*dc][d] each
  const float* Wgu; const float* Wgx; const float* bg;   // [G][d], [G][d], [G]
  const float* Wo; const float* bo;     // [K][G], [K]
};

// score of item x (row of emb) for query q (both of dtype, length d)
double oracle_scorer_score(const OracleScorer* S, int dtype, int d, const void* q, int64_t qrow, const void* emb,
                           int64_t row) {
  auto Q = [&](int j) { return val(q, dtype, qrow * d + j); };
  auto X = [&](int j) { return val(emb, dtype, row * d + j); };
  if (S->kind == 1) {
    std::vector<double> hq(S->F), hx(S->F);
    for (int f = 0; f < S->F; ++f) {
      double a = S->bm[f], b = S->bi[f];
      for (int j = 0; j < d; ++j) {
        a += (double)S->Wm[f * d + j] * Q(j);
        b += (double)S->Wi[f * d + j] * X(j);
      }
      hq[f] = a;
      hx[f] = b;
    }
    double s = S->b2[0];
    for (int h = 0; h < S->H; ++h) {
      double z = S->b1[h];
      for (int f = 0; f < S->F; ++f) z += (double)S->W1[h * S->F + f] * (hq[f] * hx[f]);
      if (z < 0.0) z = 0.0;   // ReLU
      s += (double)S->w2[h] * z;
    }
    return s;
  }
  // MoL
  std::vector<double> delta(S->K), a(S->G), logit(S->K);
  for (int k = 0; k < S->K; ++k) {
    double dk = 0.0;
    for (int c = 0; c < S->dc; ++c) {
      double f = 0.0, g = 0.0;
      const int r = k * S->dc + c;
      for (int j = 0; j < d; ++j) {
        f += (double)S->Fk[r * d + j] * Q(j);
        g += (double)S->Gk[r * d + j] * X(j);
      }
      dk += f * g;
    }
    delta[k] = dk;
  }
  for (int h = 0; h < S->G; ++h) {
    double z = S->bg[h];
    for (int j = 0; j < d; ++j) z += (double)S->Wgu[h * d + j] * Q(j) + (double)S->Wgx[h * d + j] * X(j);
    a[h] = z < 0.0 ? 0.0 : z;
  }
  double mx = -std::numeric_limits<double>::infinity();
  for (int k = 0; k < S->K; ++k) {
    double l = S->bo[k];
    for (int h = 0; h < S->G; ++h) l += (double)S->Wo[k * S->G + h] * a[h];
    logit[k] = l;
    mx = std::max(mx, l);
  }
  double den = 0.0;
  for (int k = 0; k < S->K; ++k) den += std::exp(logit[k] - mx);
  double s = 0.0;
  for (int k = 0; k < S->K; ++k) s += std::exp(logit[k] - mx) / den * delta[k];
  return s;
}

// Filtered top-K under a learned scorer: passing items (live, every clause), ordered by
// (score desc, id asc), first min(K, pass), padded (-1, -inf). queries [B][d] (one vector each).
int oracle_search_scored(const OracleScorer* S, int dtype, int d, int64_t n, int64_t row0, const void* emb,
                         const uint64_t* attrs, int W, const uint8_t* live, const void* queries, int B,
                         const void* clauses, const int32_t* clause_off, int K, int64_t* out_ids, double* out_scores,
                         int64_t* out_pass) {
  if (!S || (S->kind != 1 && S->kind != 2) || K < 1 || B < 1 || d < 1 || W < 1 || n < 0) return -1;
  const Clause* cl_all = (const Clause*)clauses;
  for (int b = 0; b < B; ++b) {
    if (clause_off[b + 1] < clause_off[b]) return -1;
    for (int c = clause_off[b]; c < clause_off[b + 1]; ++c)
      if (cl_all[c].word >= W || cl_all[c].mask == 0) return -1;
  }
  struct C {
    double s;
    int64_t id;
  };
  for (int b = 0; b < B; ++b) {
    std::vector<C> cand;
    for (int64_t i = 0; i < n; ++i) {
      if (!live[i] || !passes(attrs, W, i, cl_all + clause_off[b], clause_off[b + 1] - clause_off[b])) continue;
      double s = oracle_scorer_score(S, dtype, d, queries, b, emb, i);
      if (s == 0.0) s = 0.0;
      cand.push_back({s, row0 + i});
    }
    std::sort(cand.begin(), cand.end(), [](const C& a, const C& c) { return a.s != c.s ? a.s > c.s : a.id < c.id; });
    out_pass[b] = (int64_t)cand.size();
    for (int j = 0; j < K; ++j) {
      const int64_t at = (int64_t)b * K + j;
      out_ids[at] = j < (int64_t)cand.size() ? cand[j].id : -1;
      out_scores[at] = j < (int64_t)cand.size() ? cand[j].s : -std::numeric_limits<double>::infinity();
    }
  }
  return 0;
}

}  // extern "C"
