"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: the hand-worked Fig. 1-style
example (tests/golden, values derived by hand from PAPER.md P:4266), SPEC.md's printed examples,
IEEE bit-pattern definitions, closed forms, brute force on tiny inputs, and invariants. A
plausible mistake (dropped clause, inverted Reverse, wrong tie order, zero-masking instead of
exclusion, transposed operand, lost V-max, wrong shard offset) fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import datagen as dg
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DTYPES = [oracle.F32, oracle.F16, oracle.BF16, oracle.I8]


def to_storage(x, dtype):
    x = np.asarray(x, dtype=np.float64)
    if dtype == oracle.F32:
        return x.astype(np.float32)
    if dtype == oracle.F16:
        return x.astype(np.float16).view(np.uint16)
    if dtype == oracle.BF16:
        return dg.f32_to_bf16_bits(x.astype(np.float32))
    return x.astype(np.int8)


def parse_clauses(cl):
    return [(int(m, 16), w, r) for (m, w, r) in cl]


def fscore(v):
    return -math.inf if v == "-inf" else float(v)


# ------------------------------------------------------------------ golden: Fig. 1-style example
@pytest.mark.parametrize("dtype", DTYPES)
def test_fig1_hand_worked(dtype):
    g = json.load(open(os.path.join(GOLD, "fig1_example.json")))
    d = 16
    X = np.zeros((5, d))
    A = np.zeros((5, 1), dtype=np.uint64)
    for it in g["items"]:
        X[it["id"], :2] = it["x"]
        A[it["id"], 0] = int(it["attrs"], 16)
    emb = to_storage(X, dtype)
    live = np.ones(5, np.uint8)
    for case in g["cases"]:
        q = np.zeros((1, d))
        q[0, :2] = case["q"]
        ids, sc, ps = oracle.search(dtype, emb, A, live, to_storage(q, dtype), [parse_clauses(case["clauses"])],
                                    case["K"])
        assert ids[0].tolist() == case["expect_ids"], case["name"]
        assert sc[0].tolist() == [fscore(v) for v in case["expect_scores"]], case["name"]
        assert ps[0] == case["expect_pass"], case["name"]


def test_spec_clause_examples():
    g = json.load(open(os.path.join(GOLD, "spec_clause_examples.json")))
    for c in g["clause_cases"]:
        item = sum(1 << b for b in c["item_bits"])
        qm = sum(1 << b for b in c["query_bits"])
        m, cnt = oracle.filter_mask(np.array([[item]], np.uint64), np.ones(1), [(qm, 0, c["reverse"])])
        assert int(m[0]) == c["expect"], c


def test_spec_topk_examples():
    g = json.load(open(os.path.join(GOLD, "spec_clause_examples.json")))
    d = 16
    for c in g["topk_cases"]:
        n = len(c["scores"])
        X = np.zeros((n, d), np.float32)
        X[:, 0] = c["scores"]
        A = np.array([[1 if m else 2] for m in c["mask"]], np.uint64)   # bit0 <=> mask=1
        q = np.zeros((1, d), np.float32)
        q[0, 0] = 1.0
        ids, sc, ps = oracle.search(oracle.F32, X, A, np.ones(n), q, [[(1, 0, 0)]], c["k"])
        assert ids[0].tolist() == c["expect_slots"]
        assert sc[0].tolist() == [float(np.float32(s)) for s in c["expect_scores"]]


# ------------------------------------------------------------------ widening = IEEE definitions
def test_widen_f16_bit_patterns():
    assert oracle.widen(oracle.F16, 0x3C00) == 1.0
    assert oracle.widen(oracle.F16, 0xC000) == -2.0
    assert oracle.widen(oracle.F16, 0x0001) == 2.0 ** -24       # smallest subnormal
    assert oracle.widen(oracle.F16, 0x03FF) == 1023 * 2.0 ** -24  # largest subnormal
    assert oracle.widen(oracle.F16, 0x0400) == 2.0 ** -14       # smallest normal
    assert oracle.widen(oracle.F16, 0x7BFF) == 65504.0          # largest finite
    assert oracle.widen(oracle.F16, 0x3555) == 0.333251953125
    assert math.copysign(1.0, oracle.widen(oracle.F16, 0x8000)) == -1.0


def test_widen_all_f16_and_bf16_patterns():
    bits = np.arange(65536, dtype=np.uint32)
    ref16 = bits.astype(np.uint16).view(np.float16).astype(np.float64)      # library special case
    refbf = (bits << np.uint32(16)).view(np.float32).astype(np.float64)
    for b in range(0, 65536, 7):   # stride keeps it fast; includes subnormals, normals, +-inf
        v16 = oracle.widen(oracle.F16, int(b))
        vbf = oracle.widen(oracle.BF16, int(b))
        if np.isnan(ref16[b]):
            assert np.isnan(v16)
        else:
            assert v16 == ref16[b]
        if np.isnan(refbf[b]):
            assert np.isnan(vbf)
        else:
            assert vbf == refbf[b]
    assert oracle.widen(oracle.BF16, 0x3F80) == 1.0
    assert oracle.widen(oracle.BF16, 0xBF80) == -1.0
    assert oracle.widen(oracle.I8, 0x80) == -128.0
    assert oracle.widen(oracle.I8, 0x7F) == 127.0


# ------------------------------------------------------------------ clause semantics
def test_clause_complementarity():
    rng = np.random.default_rng(1)
    A = rng.integers(0, 2 ** 63, size=(500, 2), dtype=np.int64).astype(np.uint64)
    A[::7] = 0
    live = np.ones(500)
    for _ in range(50):
        m = int(rng.integers(1, 2 ** 63))
        w = int(rng.integers(0, 2))
        a, _ = oracle.filter_mask(A, live, [(m, w, 0)])
        b, _ = oracle.filter_mask(A, live, [(m, w, 1)])
        assert np.all(a ^ b)   # Match(m) + Reverse(m) = 1 for every item


def test_clause_brute_force_sets():
    """Every non-zero mask of a 4-value field against every item, vs decoded set intersection."""
    items = []
    for bits in range(16):      # every subset of a 4-value field, in bits 8..11
        items.append(bits << 8)
    A = np.array(items, np.uint64)[:, None]
    live = np.ones(len(items))
    for qm in range(1, 16):
        for rev in (0, 1):
            got, cnt = oracle.filter_mask(A, live, [(qm << 8, 0, rev)])
            for i, bits in enumerate(range(16)):
                item_set = {v for v in range(4) if bits >> v & 1}
                q_set = {v for v in range(4) if qm >> v & 1}
                inter = bool(item_set & q_set)
                assert bool(got[i]) == (not inter if rev else inter)


def test_clause_and_across_or_within_and_liveness():
    rng = np.random.default_rng(2)
    A = rng.integers(0, 2 ** 63, size=(300, 3), dtype=np.int64).astype(np.uint64)
    live = (rng.random(300) < 0.8).astype(np.uint8)
    cls = [(int(rng.integers(1, 2 ** 62)), int(rng.integers(0, 3)), int(rng.integers(0, 2))) for _ in range(4)]
    got, cnt = oracle.filter_mask(A, live, cls)
    for i in range(300):
        ok = bool(live[i])
        for (m, w, r) in cls:
            hit = any((int(A[i, w]) >> bit) & 1 and (m >> bit) & 1 for bit in range(64))
            ok = ok and (hit != bool(r))
        assert bool(got[i]) == ok
    assert cnt == int(got.sum())


def test_empty_clause_rejected():
    X = np.zeros((2, 16), np.float32)
    with pytest.raises(ValueError):
        oracle.search(oracle.F32, X, np.zeros((2, 1), np.uint64), np.ones(2), np.zeros((1, 16), np.float32),
                      [[(0, 0, 0)]], 1)
    with pytest.raises(ValueError):   # clause word beyond W
        oracle.search(oracle.F32, X, np.zeros((2, 1), np.uint64), np.ones(2), np.zeros((1, 16), np.float32),
                      [[(1, 1, 0)]], 1)


# ------------------------------------------------------------------ scoring closed forms
@pytest.mark.parametrize("dtype", DTYPES)
def test_basis_query_gives_column(dtype):
    d = 32
    vals, _ = dg.gen_items(7, 0, 40, d, dtype, dg.MODE_GRID)
    for j in (0, 5, 31):
        q = np.zeros(d)
        q[j] = 1.0
        s = oracle.scores(dtype, vals, to_storage(q, dtype))
        col = dg.bits_to_f32(vals[:, j], dtype).astype(np.float64) if dtype != oracle.I8 else vals[:, j]
        assert np.array_equal(s, np.asarray(col, np.float64))


def test_int8_dot_exact_integer():
    rng = np.random.default_rng(3)
    X = rng.integers(-128, 128, size=(64, 1024)).astype(np.int8)
    q = rng.integers(-128, 128, size=1024).astype(np.int8)
    s = oracle.scores(oracle.I8, X, q)
    ref = [sum(int(a) * int(b) for a, b in zip(X[i], q)) for i in range(64)]
    assert s.tolist() == [float(v) for v in ref]
    Xm = np.full((1, 1024), -128, np.int8)
    assert oracle.scores(oracle.I8, Xm, np.full(1024, -128, np.int8))[0] == 1024 * 128 * 128


@pytest.mark.parametrize("dtype", [oracle.F32, oracle.F16, oracle.BF16])
def test_grid_mode_scores_are_exact_integers(dtype):
    """Integer-grid inputs k*2^-7: score * 2^14 equals the integer dot of the k's exactly."""
    d = 128
    vals, _ = dg.gen_items(11, 0, 30, d, dtype, dg.MODE_GRID)
    k8, _ = dg.gen_items(11, 0, 30, d, oracle.I8, dg.MODE_GRID)
    q = dg.gen_queries(5, 11, 30, 1, 1, d, dtype, dg.MODE_GRID)[0, 0]
    qk = dg.gen_queries(5, 11, 30, 1, 1, d, oracle.I8, dg.MODE_GRID)[0, 0]
    s = oracle.scores(dtype, vals, q)
    ref = [sum(int(a) * int(b) for a, b in zip(k8[i], qk)) for i in range(30)]
    assert (s * 2.0 ** 14).tolist() == [float(v) for v in ref]


def test_float_accumulation_is_fp64_cancellation():
    """Reading R8: the oracle widens exactly and sums in fp64 (not fp32). Cancellation vectors fix
    the precision: [2^24, 1, -2^24] . [1, 1, 1] is exactly 1; an fp32 running sum gives
    fl32(2^24 + 1) - 2^24 = 0, and a sum in any other order than index order still differs
    from the fp64 value for the second row (2^-30 below fp32 resolution at 1)."""
    X = np.zeros((2, 16), np.float32)
    X[0, :3] = [2.0 ** 24, 1.0, -(2.0 ** 24)]
    X[1, :3] = [1.0, 2.0 ** -30, 2.0 ** -30]
    q = np.zeros(16, np.float32)
    q[:3] = 1.0
    s = oracle.scores(oracle.F32, X, q)
    assert s[0] == 1.0                       # fp32 accumulation would give 0.0
    assert s[1] == 1.0 + 2.0 ** -29          # fp32 accumulation would give 1.0
    # the same through the search (the definition the GPU is compared against)
    ids, sc, _ = oracle.search(oracle.F32, X, np.ones((2, 1), np.uint64), np.ones(2), q[None], [[]], 2)
    assert ids[0].tolist() == [1, 0] and sc[0].tolist() == [1.0 + 2.0 ** -29, 1.0]
    # bf16 widening feeds the same fp64 sum: 2^24 and 1 are exact bf16 values
    b = dg.f32_to_bf16_bits(X[:1])
    assert oracle.scores(oracle.BF16, b, dg.f32_to_bf16_bits(q))[0] == 1.0


def test_zero_query_returns_first_passing_ids():
    rng = np.random.default_rng(4)
    n, d = 200, 16
    X = rng.standard_normal((n, d)).astype(np.float32)
    A = rng.integers(0, 2 ** 63, size=(n, 1), dtype=np.int64).astype(np.uint64)
    live = (rng.random(n) < 0.9).astype(np.uint8)
    cl = [(0x00FF00FF00FF00FF, 0, 0)]
    mask, cnt = oracle.filter_mask(A, live, cl)
    K = 17
    ids, sc, ps = oracle.search(oracle.F32, X, A, live, np.zeros((1, d), np.float32), [cl], K)
    exp = np.nonzero(mask)[0][:K]
    assert ids[0, :len(exp)].tolist() == exp.tolist()
    assert np.all(sc[0, :len(exp)] == 0.0)
    assert ps[0] == cnt


# ------------------------------------------------------------------ top-K brute force
def test_topk_brute_force_tiny():
    rng = np.random.default_rng(5)
    for trial in range(60):
        n = int(rng.integers(1, 13))
        d = 16
        X = np.zeros((n, d), np.float32)
        X[:, 0] = rng.integers(-3, 4, size=n)       # small integers -> many ties
        X[:, 1] = rng.integers(-3, 4, size=n)
        q = np.zeros((1, d), np.float32)
        q[0, :2] = rng.integers(-2, 3, size=2)
        A = rng.integers(0, 4, size=(n, 1)).astype(np.uint64)
        live = (rng.random(n) < 0.85).astype(np.uint8)
        cl = [] if trial % 3 == 0 else [(int(rng.integers(1, 4)), 0, int(rng.integers(0, 2)))]
        s = [float(X[i, 0]) * float(q[0, 0]) + float(X[i, 1]) * float(q[0, 1]) for i in range(n)]
        passing = []
        for i in range(n):
            ok = bool(live[i])
            for (m, w, r) in cl:
                ok = ok and (((int(A[i, 0]) & m) != 0) != bool(r))
            if ok:
                passing.append(i)
        # rank by counting who beats whom (no sort)
        rank = {i: sum(1 for j in passing if s[j] > s[i] or (s[j] == s[i] and j < i)) for i in passing}
        for K in range(1, n + 3):
            ids, sc, ps = oracle.search(oracle.F32, X, A, live, q, [cl], K, row0=1000)
            exp = [None] * K
            for i in passing:
                if rank[i] < K:
                    exp[rank[i]] = i
            exp_ids = [1000 + i if i is not None else -1 for i in exp]
            exp_sc = [s[i] if i is not None else -math.inf for i in exp]
            assert ids[0].tolist() == exp_ids
            assert sc[0].tolist() == exp_sc
            assert ps[0] == len(passing)


# ------------------------------------------------------------------ multi-vector (R12)
def test_multi_vector_max_and_v1_reduction():
    n, d, V = 300, 64, 4
    for dtype in (oracle.BF16, oracle.I8):
        vals, A = dg.gen_items(21, 0, n, d, dtype, dg.MODE_DENSE)
        live = np.ones(n)
        Q = dg.gen_queries(9, 21, n, 2, V, d, dtype, dg.MODE_DENSE)
        cls = dg.gen_clauses(9, 2, "HIGH")
        K = 25
        ids, sc, ps = oracle.search(dtype, vals, A, live, Q, cls, K)
        for b in range(2):
            per_v = np.stack([oracle.scores(dtype, vals, Q[b, v]) for v in range(V)])   # [V][n]
            mx = per_v.max(axis=0)
            mask, cnt = oracle.filter_mask(A, live, cls[b])
            cand = sorted([(-mx[i], i) for i in range(n) if mask[i]])[:K]
            assert ids[b, :len(cand)].tolist() == [i for _, i in cand]
            assert sc[b, :len(cand)].tolist() == [-s for s, _ in cand]
            # R12: union of per-vector top-Ks, dedupe keeping max, then top-K == max-sim top-K
            union = {}
            for v in range(V):
                iv, sv, _ = oracle.search(dtype, vals, A, live, Q[b:b + 1, v:v + 1], [cls[b]], K)
                for i, s in zip(iv[0], sv[0]):
                    if i >= 0:
                        union[int(i)] = max(union.get(int(i), -math.inf), float(s))
            merged = sorted(union.items(), key=lambda t: (-t[1], t[0]))[:K]
            assert ids[b, :len(merged)].tolist() == [i for i, _ in merged]
        # V=1 of a multi-vector query equals the single-vector call
        i1, s1, p1 = oracle.search(dtype, vals, A, live, Q[:, :1], cls, K)
        i2, s2, p2 = oracle.search(dtype, vals, A, live, Q[:, 0], cls, K)
        assert np.array_equal(i1, i2) and np.array_equal(s1, s2) and np.array_equal(p1, p2)


# ------------------------------------------------------------------ sharding (R13)
def test_shard_merge_equals_full_index():
    n, d, K = 1000, 32, 40
    vals, A = dg.gen_items(31, 0, n, d, oracle.I8, dg.MODE_DENSE)
    live = np.ones(n, np.uint8)
    live[::13] = 0
    Q = dg.gen_queries(3, 31, n, 3, 1, d, oracle.I8)
    cls = dg.gen_clauses(3, 3, "HIGH")
    full = oracle.search(oracle.I8, vals, A, live, Q, cls, K)
    for G in (1, 2, 3, 8):
        per = -(-n // G)
        outs = []
        for r in range(G):
            a, b = r * per, min(n, (r + 1) * per)
            outs.append(oracle.search(oracle.I8, vals[a:b], A[a:b], live[a:b], Q, cls, K, row0=a))
        ids = np.stack([o[0] for o in outs])
        sc = np.stack([o[1] for o in outs])
        ps = np.stack([o[2] for o in outs])
        m = oracle.merge(ids, sc, ps, K)
        for x, y in zip(m, full):
            assert np.array_equal(x, y), G


def test_merge_brute_force():
    rng = np.random.default_rng(6)
    L, B, Kin, K = 4, 2, 5, 7
    ids = rng.permutation(100)[:L * B * Kin].reshape(L, B, Kin).astype(np.int64)
    sc = rng.integers(-3, 3, size=(L, B, Kin)).astype(np.float64)
    ids[1, 0, 3:] = -1
    sc[1, 0, 3:] = -math.inf
    ps = rng.integers(0, 50, size=(L, B))
    oi, osc, op = oracle.merge(ids, sc, ps, K)
    for b in range(B):
        allc = [(sc[l, b, j], ids[l, b, j]) for l in range(L) for j in range(Kin) if ids[l, b, j] >= 0]
        rank = [(sum(1 for (s2, i2) in allc if s2 > s or (s2 == s and i2 < i)), i, s) for (s, i) in allc]
        exp = sorted(rank)[:K]
        assert oi[b].tolist() == [i for _, i, _ in exp]
        assert op[b] == ps[:, b].sum()


# ------------------------------------------------------------------ live update replay
def test_update_replay_equivalence():
    n, d, K = 500, 64, 30
    vals, A = dg.gen_items(41, 0, n, d, oracle.BF16)
    live = np.ones(n, np.uint8)
    Q = dg.gen_queries(4, 41, n, 2, 1, d, oracle.BF16)
    cls = dg.gen_clauses(4, 2, "HIGH")
    # apply: overwrite rows 10..59 with rows generated under another seed, delete 100..119
    rows = np.arange(10, 60)
    nv, na = dg.item_values(99, rows, d, oracle.BF16, dg.MODE_DENSE), dg.item_attrs(99, rows, 1)
    v2, a2, l2 = vals.copy(), A.copy(), live.copy()
    v2[rows], a2[rows] = nv, na
    l2[100:120] = 0
    r_upd = oracle.search(oracle.BF16, v2, a2, l2, Q, cls, K)
    # fresh build with the final rows (keep deleted rows out by not loading them)
    keep = np.ones(n, bool)
    keep[100:120] = False
    fv, fa = vals.copy(), A.copy()
    fv[rows], fa[rows] = nv, na
    r_new = oracle.search(oracle.BF16, fv, fa, keep.astype(np.uint8), Q, cls, K)
    for x, y in zip(r_upd, r_new):
        assert np.array_equal(x, y)
    assert not set(r_upd[0].ravel().tolist()) & set(range(100, 120))
