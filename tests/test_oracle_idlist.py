"""Pins for the ID-list clauses of the oracle (oracle_search_idc; -m "not gpu").

PAPER.md P:4266 defines a clause as a list of attribute ids with at-least-one-match semantics
(Reverse: none matches) over per-item attribute lists stored with a count matrix; P:4564 stores
them as 64-bit integers. Pinned against: SPEC's printed example, brute-force Python set
intersection, Match/Reverse complementarity, and -- a cross-representation pin -- the bitmask
clauses of oracle_search on the same sets encoded as bits (ids < 64).
"""
import numpy as np
import pytest

import datagen as dg
import oracle


def _one_item_index(ids_list, A=4):
    ids = np.full((1, A), dg.ID_SENTINEL, np.uint64)
    ids[0, :len(ids_list)] = sorted(ids_list)
    return ids, np.array([len(ids_list)], np.uint8)


def test_spec_example():
    """item attrs {3,7}, query {7,9}: Match -> 1, ReverseMatch -> 0."""
    X = np.zeros((1, 16), np.float32)
    A = np.zeros((1, 1), np.uint64)
    q = np.zeros((1, 16), np.float32)
    idl = [_one_item_index([3, 7])]
    _, _, pm = oracle.search_idc(oracle.F32, X, A, np.ones(1), idl, q, [[]], [[(0, 0, [7, 9])]], 1)
    _, _, pr = oracle.search_idc(oracle.F32, X, A, np.ones(1), idl, q, [[]], [[(0, 1, [7, 9])]], 1)
    assert pm[0] == 1 and pr[0] == 0
    _, _, p2 = oracle.search_idc(oracle.F32, X, A, np.ones(1), idl, q, [[]], [[(0, 0, [8, 9])]], 1)
    assert p2[0] == 0


def test_brute_force_sets_and_complementarity():
    n, d, S = 800, 16, 2
    rng = np.random.default_rng(4)
    X = rng.standard_normal((n, d)).astype(np.float32)
    A = np.ones((n, 1), np.uint64)
    live = (rng.random(n) < 0.9).astype(np.uint8)
    idl = [dg.gen_idlists(7, 0, n, s, 5 if s == 0 else 2, 40 if s == 0 else 9) for s in range(S)]
    q = rng.standard_normal((3, d)).astype(np.float32)
    id_cl = [[(0, 0, np.unique(dg.id_of(7, [1, 5, 9, 30])))],
             [(1, 1, np.unique(dg.id_of(7, [2])))],
             [(0, 0, np.unique(dg.id_of(7, [0, 3]))), (1, 0, np.unique(dg.id_of(7, [4, 8])))]]
    ids, sc, ps = oracle.search_idc(oracle.F32, X, A, live, idl, q, [[], [], []], id_cl, n)
    for b in range(3):
        want = []
        for i in range(n):
            ok = bool(live[i])
            for (slot, rev, qids) in id_cl[b]:
                items = set(idl[slot][0][i, :idl[slot][1][i]].tolist())
                hit = bool(items & set(np.asarray(qids).tolist()))
                ok = ok and (hit != bool(rev))
            if ok:
                want.append(i)
        assert ps[b] == len(want)
        assert sorted(ids[b, :ps[b]].tolist()) == want
    # Match + Reverse of the same clause partition the live items
    _, _, pm = oracle.search_idc(oracle.F32, X, A, live, idl, q[:1], [[]], [[id_cl[0][0]]], 1)
    c = id_cl[0][0]
    _, _, pr = oracle.search_idc(oracle.F32, X, A, live, idl, q[:1], [[]], [[(c[0], 1, c[2])]], 1)
    assert pm[0] + pr[0] == int(live.sum())


@pytest.mark.parametrize("rev", [0, 1])
def test_equals_bitmask_clauses_on_small_universe(rev):
    """Ids in [0, 64): an item's ID list {v} <-> attribute word with bits v; a query ID clause with
    values Q <-> bitmask clause mask = sum 2^v. Both oracle functions must give identical results."""
    n, d, K = 3000, 32, 200
    vals, _ = dg.gen_items(21, 0, n, d, dg.I8)
    ids, cnt = dg.gen_idlists(21, 0, n, 0, 6, 64, raw=True)
    word = np.zeros((n, 1), np.uint64)
    for i in range(n):
        for v in ids[i, :cnt[i]]:
            word[i, 0] |= np.uint64(1) << np.uint64(int(v))
    Q = dg.gen_queries(22, 21, n, 4, 2, d, dg.I8)
    qsets = [[3, 17, 40], [0], [63, 62, 1, 2, 5], [10, 11]]
    id_cl = [[(0, rev, np.array(sorted(s_), np.uint64))] for s_ in qsets]
    bm_cl = [[(sum(1 << v for v in s_), 0, rev)] for s_ in qsets]
    live = np.ones(n, np.uint8)
    a = oracle.search_idc(dg.I8, vals, np.zeros((n, 1), np.uint64), live, [(ids, cnt)], Q, [[]] * 4, id_cl, K)
    b = oracle.search(dg.I8, vals, word, live, Q, bm_cl, K)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_empty_id_list_and_bad_slot_rejected():
    X = np.zeros((2, 16), np.float32)
    idl = [_one_item_index([1]), _one_item_index([2])]
    idl = [(np.concatenate([idl[0][0], idl[1][0]]), np.concatenate([idl[0][1], idl[1][1]]))]
    with pytest.raises(ValueError):
        oracle.search_idc(oracle.F32, X, np.ones((2, 1), np.uint64), np.ones(2), idl, X[:1], [[]], [[(0, 0, [])]], 1)
    with pytest.raises(ValueError):
        oracle.search_idc(oracle.F32, X, np.ones((2, 1), np.uint64), np.ones(2), idl, X[:1], [[]], [[(1, 0, [1])]], 1)


def test_generator_lists_sorted_distinct_padded():
    ids, cnt = dg.gen_idlists(5, 100, 2000, 1, 8, 1000)
    assert cnt.min() >= 1 and cnt.max() <= 8
    for i in range(0, 2000, 37):
        row = ids[i, :cnt[i]]
        assert np.all(row[1:] > row[:-1])
        assert np.all(ids[i, cnt[i]:] == dg.ID_SENTINEL)
