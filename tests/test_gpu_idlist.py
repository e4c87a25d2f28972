"""GPU parity of ID-list clauses through the C ABI
vs oracle.search_idc, element by element (-m gpu). Integer filter decisions: ids, pass counts and
(int8 / integer-grid) scores are bit-exact."""
import numpy as np
import pytest
import torch

import datagen as dg
import oracle
from parity import check, make_index, to_torch

pytestmark = pytest.mark.gpu
DEV = "cuda"

SLOTS = [(4, 1000), (8, 60), (1, 24)]   # (width, universe): company-like, skills-like, geo-like


def idl_index(dtype, d, n, mode, slots=SLOTS, capacity=None):
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype, capacity=capacity)
    ix.attach_idlists([w for w, _ in slots])
    lists = []
    for s, (w, u) in enumerate(slots):
        ids, cnt = dg.gen_idlists(dg.DATA_SEED, 0, n, s, w, u)
        lists.append((ids, cnt))
        ix.set_idlists(s, torch.from_numpy(ids.view(np.int64)).to(DEV), torch.from_numpy(cnt).to(DEV), row0=0)
    return ix, vals, attrs, lists


def queries_for(B, n, slots=SLOTS):
    out = []
    for b in range(B):
        cl = []
        for s, (w, u) in enumerate(slots):
            if (b + s) % 3 == 2:
                continue
            c = dg.gen_id_clauses(dg.QUERY_SEED + s, dg.DATA_SEED, 1 + b, s, w, u, 1 + 5 * (s + b % 2), n,
                                  reverse=(b + s) % 4 == 3)[b]
            cl.extend(c)
        out.append(cl)
    return out


@pytest.mark.parametrize("dtype,mode,d,B,V,K,preset", [
    (dg.I8, dg.MODE_DENSE, 64, 3, 1, 500, "HIGH"),
    (dg.BF16, dg.MODE_GRID, 128, 4, 2, 100, "ALL"),
    (dg.F32, dg.MODE_GRID, 64, 2, 1, 2048, "LOW"),
    (dg.BF16, dg.MODE_GRID, 128, 20, 1, 300, "HIGH"),   # B*V >= 16 also runs per user (bitmaps)
])
def test_search_idc_parity(dtype, mode, d, B, V, K, preset):
    n = 70_000
    ix, vals, attrs, lists = idl_index(dtype, d, n, mode)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    icl = queries_for(B, n)
    g = ix.search_idc(to_torch(Q, dtype, DEV), cls, icl, K)
    torch.cuda.synchronize()
    ref = oracle.search_idc(dtype, vals, attrs, np.ones(n), lists, Q, cls, icl, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, True, what=f"idc dt{dtype} B{B}")
    assert ix.stats()["overflow"] == 0


def test_idc_live_updates_and_deletes():
    """Upserted rows get new ID lists (set_idlists with row ids), deletes clear liveness."""
    n, d, K = 40_000, 64, 300
    ix, vals, attrs, lists = idl_index(dg.I8, d, n, dg.MODE_DENSE, capacity=n + 1000)
    rng = np.random.default_rng(5)
    rows = np.concatenate([rng.choice(n, 1500, replace=False), np.arange(n, n + 1000)])
    nv, na = dg.gen_items(dg.UPDATE_SEED, 0, len(rows), d, dg.I8)
    from parity import attrs_torch
    ix.update_rows(torch.from_numpy(rows).to(DEV), to_torch(nv, dg.I8, DEV), attrs_torch(na, DEV))
    fl = []
    for s, (w, u) in enumerate(SLOTS):
        ni, nc = dg.gen_idlists(dg.UPDATE_SEED, 0, len(rows), s, w, u)
        ix.set_idlists(s, torch.from_numpy(ni.view(np.int64)).to(DEV), torch.from_numpy(nc).to(DEV),
                       rows=torch.from_numpy(rows).to(DEV))
        ids, cnt = lists[s]
        ids = np.concatenate([ids, np.full((1000, w), dg.ID_SENTINEL, np.uint64)])
        cnt = np.concatenate([cnt, np.zeros(1000, np.uint8)])
        ids[rows], cnt[rows] = ni, nc
        fl.append((ids, cnt))
    dele = rng.choice(n, 2000, replace=False)
    ix.delete_rows(torch.from_numpy(dele).to(DEV))
    fv = np.concatenate([vals, np.zeros((1000, d), vals.dtype)])
    fa = np.concatenate([attrs, np.zeros((1000, 1), np.uint64)])
    fv[rows], fa[rows] = nv, na
    live = np.ones(n + 1000, np.uint8)
    live[dele] = 0
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, 3, 1, d, dg.I8)
    cls = dg.gen_clauses(dg.QUERY_SEED, 3, "ALL")
    icl = queries_for(3, n)
    g = ix.search_idc(to_torch(Q, dg.I8, DEV), cls, icl, K)
    ref = oracle.search_idc(dg.I8, fv, fa, live, fl, Q, cls, icl, K)
    check(dg.I8, fv, fa, live, Q, cls, K, g, ref, True, what="idc updates")


def test_idc_invalid_arguments():
    from paper_2407_13218_b200 import LinrError
    n, d = 1000, 64
    ix, vals, attrs, lists = idl_index(dg.I8, d, n, dg.MODE_DENSE)
    q = torch.zeros((1, d), dtype=torch.int8, device=DEV)
    with pytest.raises(LinrError):
        ix.search_idc(q, [[]], [[(0, 0, [])]], 10)       # empty ID list (reading R3)
    with pytest.raises(LinrError):
        ix.search_idc(q, [[]], [[(7, 0, [1])]], 10)      # slot beyond the attached ones
