"""Pins for the quantised-path oracle (oracle/oporp_oracle.cpp; -m "not gpu").

Each pin checks the oracle against something other than its own formula: hand-worked codes
(tests/golden/oporp_example.json), SPEC's printed invariants (zero vector, sign antisymmetry,
self/anti match), the paper's XOR/NOT formulation of matched bits (Fig. 3 caption) against the
oracle's per-bit loop, the sign-random-projection collision law (the estimator
cos(pi(1 - m/k)) tracks the true cosine), brute force for the code search, and the V3 identities
(keep = 1 is the exact search; kept = min(pass, max(K, ceil(keep*pass)))).
"""
import json
import math
import os

import numpy as np
import pytest

import datagen as dg
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def popcount64(a):
    a = np.asarray(a, dtype=np.uint64)
    return np.array([bin(int(v)).count("1") for v in a.ravel()]).reshape(a.shape)


def _rules(case):
    k, rule_src, rule_sign = case["k"], case["src_rule"], case["sign_rule"]
    b = {"one coordinate per bit (b=1), signs + then -": 1, "128-bit code, second word from the negated vector": 1}.get(
        case["name"], 2)
    L = k * b
    p = np.arange(L)
    if rule_src == "src[p] = p % 4":
        src = p % 4
    else:
        src = np.where(p % 2 == 1, -1, (p // 2) % 4)
    if rule_sign == "sign[p] = +1":
        sign = np.ones(L)
    elif rule_sign.startswith("sign[p] = +1 for p < "):
        half = int(rule_sign.split("p < ")[1].split(",")[0])
        sign = np.where(p < half, 1, -1)
    else:
        sign = np.where((p // 2) % 4 == 2, -1, 1)
    return src.astype(np.int32), sign.astype(np.int8)


def test_golden_hand_worked_codes():
    g = json.load(open(os.path.join(GOLD, "oporp_example.json")))
    for case in g["cases"]:
        x = np.zeros((1, 4), np.float32)
        x[0] = case["x"]
        code = oracle.oporp_encode(oracle.F32, x, case["k"], _rules(case))
        assert [f"0x{int(w):016X}" for w in code[0]] == case["expect_words"], case["name"]
        # the same values stored as int8 / bf16 give the same bits (exact widening)
        for dt, store in ((oracle.I8, x.astype(np.int8)), (oracle.BF16, dg.f32_to_bf16_bits(x))):
            assert np.array_equal(oracle.oporp_encode(dt, store, case["k"], _rules(case)), code)


@pytest.mark.parametrize("d,k", [(64, 64), (128, 64), (128, 512), (16, 128), (100, 64)])
def test_zero_vector_all_ones_and_antisymmetry(d, k):
    """all-zero embedding -> every bin 0 -> every bit 1; encode(-x) is the bitwise
    complement of encode(x) when no bin sums to exactly 0 (dense random f32 values)."""
    prm = dg.oporp_params(dg.OPORP_SEED, d, k)
    z = oracle.oporp_encode(oracle.F32, np.zeros((1, d), np.float32), k, prm)
    assert np.all(z == np.uint64(0xFFFFFFFFFFFFFFFF))
    rng = np.random.default_rng(d * k)
    x = (rng.standard_normal((20, d)) + 1e-3).astype(np.float32)
    a = oracle.oporp_encode(oracle.F32, x, k, prm)
    b = oracle.oporp_encode(oracle.F32, -x, k, prm)
    # bins made only of zero padding sum to exactly 0 for x and -x (bit 1 in both): excluded
    src = prm[0].reshape(k, -1)
    real = np.zeros(k // 64, np.uint64)
    for j in range(k):
        if (src[j] >= 0).any():
            real[j // 64] |= np.uint64(1) << np.uint64(j % 64)
    assert np.all((a ^ b) & real == real)
    assert np.all(a & b & ~real == ~real & np.uint64(0xFFFFFFFFFFFFFFFF))


def test_params_reading_R25():
    """k <= d: a permutation of the zero-padded vector (every coordinate exactly once);
    k > d: a permutation of k copies (every coordinate exactly k times, bins of d entries)."""
    src, sign = dg.oporp_params(dg.OPORP_SEED, 100, 64)
    assert len(src) == 128 and sorted(src[src >= 0].tolist()) == list(range(100)) and (src == -1).sum() == 28
    src, sign = dg.oporp_params(dg.OPORP_SEED, 128, 512)
    assert len(src) == 512 * 128 and np.all(np.bincount(src, minlength=128) == 512)
    assert set(np.unique(sign).tolist()) == {-1, 1} and abs(int(sign.astype(np.int64).sum())) < 4 * math.sqrt(len(sign))
    src2, _ = dg.oporp_params(dg.OPORP_SEED, 128, 512)
    assert np.array_equal(src, src2)   # seed-deterministic


def test_matched_bits_vs_xor_not_formulation():
    """Fig. 3 caption: matched = popcount(NOT(a) XOR b); the oracle counts bit by bit."""
    rng = np.random.default_rng(5)
    for k in (64, 128, 512):
        a = rng.integers(0, 2 ** 63, size=(200, k // 64), dtype=np.int64).astype(np.uint64) * np.uint64(2) + \
            rng.integers(0, 2, size=(200, k // 64)).astype(np.uint64)
        b = rng.integers(0, 2 ** 63, size=(200, k // 64), dtype=np.int64).astype(np.uint64)
        m = oracle.matched_bits(k, a, b)
        ref = popcount64(~a ^ b).sum(axis=1)
        assert m.tolist() == ref.tolist()
        assert oracle.matched_bits(k, a, a).tolist() == [k] * 200          # self-match
        assert oracle.matched_bits(k, a, ~a).tolist() == [0] * 200         # anti-match


def test_collision_law_estimates_cosine():
    """SPEC S:176 / P:4291 (Sign-OPORP approximates cosine via matched bits): over random unit-vector
    pairs at d=128, k=512, the estimate cos(pi*(1 - m/k)) is within 0.06 of the true cosine on
    average, and the matched fraction tracks the sign-random-projection law 1 - theta/pi."""
    d, k, n = 128, 512, 1500
    prm = dg.oporp_params(dg.OPORP_SEED, d, k)
    rng = np.random.default_rng(11)
    x = rng.standard_normal((n, d))
    rho = rng.uniform(-0.95, 0.95, size=n)
    z = rng.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    z -= (z * x).sum(1, keepdims=True) * x
    z /= np.linalg.norm(z, axis=1, keepdims=True)
    y = rho[:, None] * x + np.sqrt(1 - rho[:, None] ** 2) * z
    cx = oracle.oporp_encode(oracle.F32, x.astype(np.float32), k, prm)
    cy = oracle.oporp_encode(oracle.F32, y.astype(np.float32), k, prm)
    m = oracle.matched_bits(k, cx, cy)
    true_cos = (x.astype(np.float32).astype(np.float64) * y.astype(np.float32).astype(np.float64)).sum(1) / (
        np.linalg.norm(x.astype(np.float32), axis=1) * np.linalg.norm(y.astype(np.float32), axis=1))
    est = np.cos(np.pi * (1 - m / k))
    assert np.mean(np.abs(est - true_cos)) <= 0.06
    law = 1 - np.arccos(np.clip(true_cos, -1, 1)) / np.pi
    assert abs(np.mean(m / k - law)) < 0.01
    # a dropped sign vector or a broken permutation would decorrelate: the fit must be tight
    assert np.corrcoef(m / k, law)[0, 1] > 0.97


def _brute_code_search(dtype, vals, attrs, live, Q, clauses, K, k, prm, row0=0):
    codes = oracle.oporp_encode(dtype, vals, k, prm)
    q = Q if Q.ndim == 3 else Q[:, None, :]
    B, V, d = q.shape
    qc = oracle.oporp_encode(dtype, q.reshape(B * V, d), k, prm).reshape(B, V, -1)
    ids = np.full((B, K), -1, np.int64)
    ms = np.full((B, K), -1, np.int64)
    ps = np.zeros(B, np.int64)
    for b in range(B):
        mask, cnt = oracle.filter_mask(attrs, live, clauses[b])
        rows = np.nonzero(mask)[0]
        # paper's formulation: popcount(NOT(q) XOR x), max over the user's V codes
        m = np.max([popcount64(~qc[b, v][None, :] ^ codes[rows]).sum(1) for v in range(V)], axis=0) if len(rows) else []
        order = sorted(range(len(rows)), key=lambda j: (-int(m[j]), int(rows[j])))
        ps[b] = len(rows)
        for j, o in enumerate(order[:K]):
            ids[b, j] = rows[o] + row0
            ms[b, j] = m[o]
    return ids, ms, ps


@pytest.mark.parametrize("k,V,K", [(64, 1, 10), (128, 2, 7), (512, 1, 300), (64, 3, 1000)])
def test_code_search_brute_force(k, V, K):
    n, d, B = 300, 64, 3
    vals, attrs = dg.gen_items(3, 0, n, d, dg.BF16, dg.MODE_DENSE)
    live = np.ones(n, np.uint8)
    live[::13] = 0
    Q = dg.gen_queries(4, 3, n, B, V, d, dg.BF16, dg.MODE_DENSE)
    cls = dg.gen_clauses(4, B, "HIGH")
    cls[2] = []
    prm = dg.oporp_params(dg.OPORP_SEED, d, k)
    got = oracle.code_search(dg.BF16, vals, attrs, live, Q, cls, K, k, prm, row0=1000)
    ref = _brute_code_search(dg.BF16, vals, attrs, live, Q, cls, K, k, prm, row0=1000)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]) and np.array_equal(got[2], ref[2])


def test_code_search_huge_K_returns_every_passer_in_order():
    """K = n (NEXT-3 regime): every passing item, (m desc, id asc), then padding."""
    n, d, k = 500, 32, 64
    vals, attrs = dg.gen_items(5, 0, n, d, dg.I8)
    Q = dg.gen_queries(6, 5, n, 1, 1, d, dg.I8)
    prm = dg.oporp_params(dg.OPORP_SEED, d, k)
    ids, m, ps = oracle.code_search(dg.I8, vals, attrs, np.ones(n), Q, [[(0xFF << 56, 0, 0)]], n, k, prm)
    assert ps[0] == n and sorted(ids[0].tolist()) == list(range(n))
    key = list(zip((-m[0]).tolist(), ids[0].tolist()))
    assert key == sorted(key)
    ids2, m2, _ = oracle.code_search(dg.I8, vals, attrs, np.ones(n), Q, [[(0xFF << 56, 0, 0)]], n + 50, k, prm)
    assert np.all(ids2[0, n:] == -1) and np.all(m2[0, n:] == -1)


@pytest.mark.parametrize("dtype,mode", [(dg.BF16, dg.MODE_DENSE), (dg.I8, dg.MODE_DENSE), (dg.F32, dg.MODE_GRID)])
def test_v3_keep_one_is_the_exact_search(dtype, mode):
    """keep_fraction = 1 reproduces V2 exactly (every passing item is reranked)."""
    n, d, B, K = 2000, 64, 3, 50
    vals, attrs = dg.gen_items(7, 0, n, d, dtype, mode)
    Q = dg.gen_queries(8, 7, n, B, 2, d, dtype, mode)
    cls = dg.gen_clauses(8, B, "HIGH")
    prm = dg.oporp_params(dg.OPORP_SEED, d, 128)
    ids, sc, ps, kept = oracle.search_v3(dtype, vals, attrs, np.ones(n), Q, cls, K, 1.0, 128, prm)
    ei, es, ep = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    assert np.array_equal(ids, ei) and np.array_equal(sc, es) and np.array_equal(ps, ep)
    assert kept.tolist() == ps.tolist()


def test_v3_kept_count_and_subset():
    """kept = min(pass, max(K, ceil(keep*pass))) (SPEC S:351 floor rule); the result is the exact
    top-K of the kept set, whose members are the top-K' of the code search."""
    n, d, K, k = 3000, 64, 40, 64
    vals, attrs = dg.gen_items(9, 0, n, d, dg.I8)
    Q = dg.gen_queries(10, 9, n, 2, 1, d, dg.I8)
    cls = dg.gen_clauses(10, 2, "HIGH")
    prm = dg.oporp_params(dg.OPORP_SEED, d, k)
    for keep in (1e-4, 0.01, 0.1, 0.5):
        ids, sc, ps, kept = oracle.search_v3(dg.I8, vals, attrs, np.ones(n), Q, cls, K, keep, k, prm)
        for b in range(2):
            want = min(ps[b], max(K, math.ceil(keep * ps[b])))
            assert kept[b] == want
            cid, cm, _ = oracle.code_search(dg.I8, vals, attrs, np.ones(n), Q[b:b + 1], [cls[b]], int(kept[b]), k, prm)
            pool = cid[0]
            s = oracle.scores(dg.I8, vals[pool], Q[b, 0])
            order = sorted(range(len(pool)), key=lambda j: (-s[j], pool[j]))[:K]
            assert ids[b].tolist() == [int(pool[j]) for j in order]
            assert sc[b].tolist() == [float(s[j]) for j in order]


def test_v3_recall_monotone_in_keep():
    """SPEC S:356 / Fig. 6 trade-off: recall@K against the exact search does not decrease with keep."""
    n, d, K, k = 20000, 64, 100, 256
    vals, attrs = dg.gen_items(12, 0, n, d, dg.BF16, dg.MODE_DENSE)
    Q = dg.gen_queries(13, 12, n, 2, 1, d, dg.BF16, dg.MODE_DENSE)
    cls = dg.gen_clauses(13, 2, "HIGH")
    prm = dg.oporp_params(dg.OPORP_SEED, d, k)
    exact = oracle.search(dg.BF16, vals, attrs, np.ones(n), Q, cls, K)[0]
    prev = -1.0
    for keep in (0.001, 0.01, 0.1, 0.5, 1.0):
        ids = oracle.search_v3(dg.BF16, vals, attrs, np.ones(n), Q, cls, K, keep, k, prm)[0]
        rec = np.mean([len(set(ids[b]) & set(exact[b])) / K for b in range(2)])
        assert rec >= prev - 1e-12
        prev = rec
    assert prev == 1.0
