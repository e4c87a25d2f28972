"""GPU parity of the quantised path (§3.2, Fig. 3) through
the C ABI vs the oracle (oracle/oporp_oracle.cpp), element by element (-m gpu).

Codes, matched-bit counts, ids and the kept counts are integers decided by fp64 bin sums taken in
the same order on both sides: bit-exact. The V3 rerank scores follow the float path's bar (exact on
int8 / integer-grid inputs; R8/R9 tolerance on dense floats).
"""
import numpy as np
import pytest
import torch

import datagen as dg
import oracle
from parity import attrs_torch, check, make_index, to_torch

pytestmark = pytest.mark.gpu
DEV = "cuda"


def coded_index(dtype, d, n, k, mode, seed=dg.DATA_SEED, capacity=None):
    vals, attrs = dg.gen_items(seed, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype, capacity=capacity)
    prm = dg.oporp_params(dg.OPORP_SEED, d, k)
    ix.attach_codes(k, *prm)
    return ix, vals, attrs, prm


@pytest.mark.parametrize("dtype", [dg.F32, dg.F16, dg.BF16, dg.I8])
@pytest.mark.parametrize("d,k", [(64, 64), (128, 64), (128, 512), (16, 128), (32, 256), (64, 1024)])
def test_encode_bit_exact(dtype, d, k):
    n = 3000
    ix, vals, attrs, prm = coded_index(dtype, d, n, k, dg.MODE_DENSE)
    ref = oracle.oporp_encode(dtype, vals, k, prm)
    got = ix.codes(n).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, ref)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, 7, 1, d, dtype, dg.MODE_DENSE)[:, 0]
    qg = ix.encode(to_torch(Q, dtype, DEV)).cpu().numpy().view(np.uint64)
    assert np.array_equal(qg, oracle.oporp_encode(dtype, Q, k, prm))
    # the all-zero vector encodes to all ones
    z = torch.zeros((1, d), dtype=to_torch(Q[:1], dtype, DEV).dtype, device=DEV)
    assert np.all(ix.encode(z).cpu().numpy().view(np.uint64) == np.uint64(0xFFFFFFFFFFFFFFFF))


def run_code_case(dtype, d, n, k, B, V, K, preset, mode=dg.MODE_DENSE, live_frac=1.0):
    ix, vals, attrs, prm = coded_index(dtype, d, n, k, mode)
    live = np.ones(n, np.uint8)
    if live_frac < 1.0:
        dead = np.nonzero(np.random.default_rng(n).random(n) > live_frac)[0]
        live[dead] = 0
        ix.delete_rows(torch.from_numpy(dead).to(DEV))
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    gi, gm, gp = [t.cpu().numpy() for t in ix.code_search(to_torch(Q, dtype, DEV), cls, K)]
    oi, om, op = oracle.code_search(dtype, vals, attrs, live, Q, cls, K, k, prm)
    assert np.array_equal(gp, op), (gp, op)
    assert np.array_equal(gm, om)
    assert np.array_equal(gi, oi)
    return ix


@pytest.mark.parametrize("k,K,preset", [(64, 1000, "HIGH"), (64, 1, "ALL"), (128, 5000, "HIGH4"),
                                        (512, 300, "LOW"), (1024, 64, "HIGH"), (256, 20_000, "ALL")])
def test_code_search_bit_exact(k, K, preset):
    run_code_case(dg.BF16, 128, 60_011, k, 2, 1, K, preset)


@pytest.mark.parametrize("B,V", [(1, 2), (3, 4), (9, 1), (12, 2)])
def test_code_search_batches_multivector(B, V):
    """B > 8 runs several user groups (kCodeMaxUsers); V > 1 takes the max matched bits (R12)."""
    run_code_case(dg.I8, 64, 40_000, 64, B, V, 777, "HIGH", live_frac=0.8)


def test_code_search_huge_K_everything():
    """K >= pass: every passing item in (m desc, id asc) order, then padding (NEXT-3 regime)."""
    n = 50_000
    ix = run_code_case(dg.I8, 64, n, 64, 1, 1, n + 1000, "ALL")
    run_code_case(dg.F16, 64, 20_000, 128, 2, 1, 15_000, "HIGH4")
    assert ix.counters()["scan_overflow"] == 0


def test_code_search_tiny_and_empty():
    run_code_case(dg.BF16, 64, 100, 64, 2, 1, 10, "HIGH")
    run_code_case(dg.BF16, 64, 5, 64, 1, 1, 10, "ALL")
    from paper_2407_13218_b200 import Index
    ix = Index(1000, 64, dg.I8, 1)
    ix.attach_codes(64, *dg.oporp_params(dg.OPORP_SEED, 64, 64))
    Q = dg.gen_queries(1, 1, 10, 1, 1, 64, dg.I8)
    ids, m, ps = ix.code_search(to_torch(Q, dg.I8, DEV), [[]], 16)
    assert (ids.cpu() == -1).all() and (m.cpu() == -1).all() and int(ps.cpu()[0]) == 0


def test_codes_follow_live_updates():
    """Upserts re-encode the overwritten rows on the same stream (codes stay exact)."""
    n, d, k, K = 30_000, 128, 256, 500
    ix, vals, attrs, prm = coded_index(dg.BF16, d, n, k, dg.MODE_DENSE, capacity=n + 2000)
    rng = np.random.default_rng(3)
    rows = np.concatenate([rng.choice(n, 2000, replace=False), np.arange(n, n + 1000)])
    nv, na = dg.gen_items(dg.UPDATE_SEED, 0, len(rows), d, dg.BF16, dg.MODE_DENSE)
    ix.update_rows(torch.from_numpy(rows).to(DEV), to_torch(nv, dg.BF16, DEV), attrs_torch(na, DEV))
    dele = rng.choice(n, 3000, replace=False)
    ix.delete_rows(torch.from_numpy(dele).to(DEV))
    fv = np.concatenate([vals, np.zeros((1000, d), vals.dtype)])
    fa = np.concatenate([attrs, np.zeros((1000, 1), np.uint64)])
    fv[rows], fa[rows] = nv, na
    live = np.ones(n + 1000, np.uint8)
    live[dele] = 0
    assert np.array_equal(ix.codes(n + 1000).cpu().numpy().view(np.uint64), oracle.oporp_encode(dg.BF16, fv, k, prm))
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, 2, 1, d, dg.BF16, dg.MODE_DENSE)
    cls = dg.gen_clauses(dg.QUERY_SEED, 2, "HIGH")
    gi, gm, gp = [t.cpu().numpy() for t in ix.code_search(to_torch(Q, dg.BF16, DEV), cls, K)]
    oi, om, op = oracle.code_search(dg.BF16, fv, fa, live, Q, cls, K, k, prm)
    assert np.array_equal(gi, oi) and np.array_equal(gm, om) and np.array_equal(gp, op)


@pytest.mark.parametrize("dtype,mode,keep,K,k,B,V", [
    (dg.I8, dg.MODE_DENSE, 0.01, 100, 64, 2, 1),
    (dg.I8, dg.MODE_DENSE, 0.1, 1000, 128, 3, 2),
    (dg.BF16, dg.MODE_GRID, 0.05, 500, 512, 2, 1),
    (dg.BF16, dg.MODE_GRID, 1.0, 200, 64, 1, 1),
    (dg.BF16, dg.MODE_DENSE, 0.02, 1000, 256, 4, 1),
    (dg.F32, dg.MODE_DENSE, 0.001, 50, 64, 1, 1),
])
def test_search_v3_parity(dtype, mode, keep, K, k, B, V):
    n, d = 80_000, 128
    ix, vals, attrs, prm = coded_index(dtype, d, n, k, mode)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    g = ix.search_v3(to_torch(Q, dtype, DEV), cls, K, keep)
    gi, gs, gp, gk = [t.cpu().numpy() for t in g]
    oi, osc, op, ok = oracle.search_v3(dtype, vals, attrs, np.ones(n), Q, cls, K, keep, k, prm)
    assert np.array_equal(gp, op) and np.array_equal(gk, ok), (gp, op, gk, ok)
    exact = dtype == dg.I8 or mode == dg.MODE_GRID
    if exact:
        assert np.array_equal(gi, oi) and np.array_equal(gs.astype(np.float64), osc)
    else:
        # the kept set is integer-exact; within it the rerank is the float path: R8/R9. check()
        # re-derives R9 against the exact scores of the kept items via a restricted oracle search.
        for b in range(B):
            cid, _, _ = oracle.code_search(dtype, vals, attrs, np.ones(n), Q[b:b + 1], [cls[b]], int(ok[b]), k, prm)
            pool = np.sort(cid[0][cid[0] >= 0])
            ref = oracle.search(dtype, vals[pool], attrs[pool], np.ones(len(pool)), Q[b:b + 1], [cls[b]], K)
            ref = (np.where(ref[0] >= 0, pool[np.maximum(ref[0], 0)], -1), ref[1], op[b:b + 1])
            check(dtype, vals, attrs, np.ones(n), Q[b:b + 1], [cls[b]], K,
                  (gi[b:b + 1], gs[b:b + 1], gp[b:b + 1]), ref, False, what=f"v3 b{b}")
    if keep == 1.0:   # keep = 1 is the exact search
        ei, es, ep = [t.cpu().numpy() for t in ix.search(to_torch(Q, dtype, DEV), cls, K)]
        assert np.array_equal(gi, ei) and np.array_equal(gs, es)
