"""GPU parity of the union path (2 <= B*V <= 8 on bf16/f16/int8, d = 64/128): sample-derived
per-user thresholds, ONE ring-scan launch over the union of the users' passing rows, merge with
certification flags, exact device-side recomputation of flagged users (readings
R23/R33). Compared with the oracle element by element (-m gpu)."""
import numpy as np
import pytest
import torch

import datagen as dg
import oracle
from parity import check, make_index, to_torch

pytestmark = pytest.mark.gpu
DEV = "cuda"


def run(dtype, d, n, B, V, K, preset, mode, expect_union=None):
    if expect_union is None:
        expect_union = V == 1 and 3 <= B <= 8   # the dispatch rule
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    ix.profile(True)
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    prof = ix.profile_read()
    if expect_union:   # sample, threshold, scan, merge, fallback: one scan launch for all B users
        assert prof["launches"] == 5, prof
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    exact = dtype == dg.I8 or mode == dg.MODE_GRID
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, exact, what=f"union dt{dtype} d{d} B{B} V{V} {preset}")
    return ix


@pytest.mark.parametrize("dtype,d,B,V,K,preset,mode,n", [
    (dg.BF16, 128, 3, 1, 1000, "HIGH", dg.MODE_GRID, 300_000),
    (dg.BF16, 128, 2, 1, 1000, "HIGH", dg.MODE_GRID, 300_000),      # per-user launches (B = 2)
    (dg.BF16, 128, 8, 1, 1000, "HIGH", dg.MODE_GRID, 300_000),
    (dg.BF16, 128, 4, 2, 500, "HIGH4", dg.MODE_GRID, 200_000),
    (dg.F16, 64, 3, 1, 2048, "ALL", dg.MODE_GRID, 150_000),
    (dg.I8, 128, 5, 1, 300, "LOW", dg.MODE_DENSE, 600_000),
    (dg.I8, 64, 2, 4, 1000, "HIGH", dg.MODE_DENSE, 250_000),
    (dg.BF16, 128, 6, 1, 100, "HIGH", dg.MODE_DENSE, 200_000),
    (dg.BF16, 64, 7, 1, 1, "ALL", dg.MODE_GRID, 50_000),
])
def test_union_path_parity(dtype, d, B, V, K, preset, mode, n):
    run(dtype, d, n, B, V, K, preset, mode)


def test_union_path_small_index_and_K_exceeds_pass():
    # fewer passers than K for some users: thresholds are 0 (no filtering) or certification fails
    run(dg.BF16, 128, 3000, 4, 1, 1500, "HIGH", dg.MODE_GRID)


def test_union_path_forced_fallback(monkeypatch):
    """LINR_UNION_FORCE_FB puts every user's threshold above every key: the scan keeps nothing,
    the merge flags every user, and the fallback kernel recomputes them exactly."""
    monkeypatch.setenv("LINR_UNION_FORCE_FB", "1")
    ix = run(dg.I8, 64, 120_000, 3, 1, 700, "HIGH", dg.MODE_DENSE)
    assert ix.counters()["tc_fallbacks"] >= 3


def test_union_path_disabled_matches(monkeypatch):
    monkeypatch.setenv("LINR_UNION", "0")
    run(dg.BF16, 128, 100_000, 4, 1, 1000, "HIGH", dg.MODE_GRID, expect_union=False)


def test_union_path_multiword_clauses_and_deleted_rows():
    """Clauses on attribute words 1..3, users without clauses, deleted rows, W = 4."""
    n, d, W, K, B = 60_000, 64, 4, 300, 5
    vals, attrs = dg.gen_items(3, 0, n, d, dg.I8, dg.MODE_DENSE, W=W)
    ix = make_index(vals, attrs, dg.I8)
    live = np.ones(n, np.uint8)
    dead = np.random.default_rng(5).choice(n, 9000, replace=False)
    live[dead] = 0
    ix.delete_rows(torch.from_numpy(dead).to(DEV))
    Q = dg.gen_queries(4, 3, n, B, 1, d, dg.I8)
    cls = [[(0x00F0_0000_0000_00F0, 1, 0), (0x1, 3, 1), (0xFFFF << 24, 0, 1)],
           [(0x8000_0000_0000_0001, 2, 0)],
           [],
           [(0xFF, 0, 0), (0xF0F0, 1, 1), (0x3, 2, 0), (0x10, 3, 1)],
           [(0xFFFF_FFFF, 0, 1)]]
    ix.profile(True)
    g = ix.search(to_torch(Q, dg.I8, DEV), cls, K)
    torch.cuda.synchronize()
    assert ix.profile_read()["launches"] == 5
    ref = oracle.search(dg.I8, vals, attrs, live, Q, cls, K)
    check(dg.I8, vals, attrs, live, Q, cls, K, g, ref, True, what="union multiword")


def test_union_path_after_updates():
    """Upserts (incl. rows past the high-water mark) between union searches: the sample, the
    thresholds and the scan all see the updated rows (stream order, reading R16)."""
    n, d, K, B = 80_000, 128, 800, 4
    dtype = dg.BF16
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, dg.MODE_GRID)
    ix = make_index(vals, attrs, dtype, capacity=n + 4000)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dtype, dg.MODE_GRID)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    ix.search(to_torch(Q, dtype, DEV), cls, K)
    rng = np.random.default_rng(11)
    rows = np.concatenate([rng.choice(n, 5000, replace=False), np.arange(n, n + 4000)])
    nv, na = dg.gen_items(dg.UPDATE_SEED, 0, len(rows), d, dtype, dg.MODE_GRID)
    from parity import attrs_torch
    ix.update_rows(torch.from_numpy(rows).to(DEV), to_torch(nv, dtype, DEV), attrs_torch(na, DEV))
    fv = np.concatenate([vals, np.zeros((4000, d), vals.dtype)])
    fa = np.concatenate([attrs, np.zeros((4000, 1), np.uint64)])
    fv[rows], fa[rows] = nv, na
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    ref = oracle.search(dtype, fv, fa, np.ones(n + 4000, np.uint8), Q, cls, K)
    check(dtype, fv, fa, np.ones(n + 4000, np.uint8), Q, cls, K, g, ref, True, what="union after updates")


@pytest.mark.parametrize("B,V", [(8, 1), (7, 1), (4, 2)])
def test_small_batch_without_pass_counts_takes_tcgen05(monkeypatch, B, V):
    """LINR_TC_NOPASS=1: B*V in [7, 8] without requested pass counts runs the dense tcgen05 pass
    (sample, threshold, main, finalize, fallback: 5 launches, no count kernel); exact results."""
    monkeypatch.setenv("LINR_TC_NOPASS", "1")
    dtype, d, n, K = dg.BF16, 128, 200_000, 500
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, dg.MODE_GRID)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, dg.MODE_GRID)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    ix.profile(True)
    ids, sc, _ = ix.search(to_torch(Q, dtype, DEV), cls, K, want_pass=False)
    torch.cuda.synchronize()
    assert ix.profile_read()["launches"] == 5
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, (ids, sc, torch.from_numpy(ref[2])), ref, True,
          what=f"tc no-pass B{B} V{V}")


@pytest.mark.parametrize("preset", ["HIGH", "LOW", "ALL"])
def test_union_gate_device_choice(preset):
    """B*V >= 7 without pass counts: the union path launches both the dense tcgen05 pass and the
    union scan behind a device-side gate (every user has a sample threshold -> tcgen05); whichever
    runs, the result is the oracle's (8 launches: sample, threshold, decide, tc main, finalize,
    union scan, merge, fallback)."""
    dtype, d, n, K, B = dg.I8, 128, 300_000, 700, 8
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, dg.MODE_DENSE)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dtype, dg.MODE_DENSE)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    ix.profile(True)
    ids, sc, _ = ix.search(to_torch(Q, dtype, DEV), cls, K, want_pass=False)
    torch.cuda.synchronize()
    assert ix.profile_read()["launches"] == 8
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, (ids, sc, torch.from_numpy(ref[2])), ref, True,
          what=f"union gate {preset}")


@pytest.mark.parametrize("B,preset", [(16, "LOW"), (12, "HIGH"), (16, "ALL"), (9, "LOW")])
def test_union_gate_two_groups(B, preset):
    """9 <= B <= 16 without pass counts: union scans over two groups of <= 8 users (or the dense
    tcgen05 pass, chosen on the device); exact either way."""
    dtype, d, n, K = dg.I8, 64, 250_000, 600
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, dg.MODE_DENSE)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dtype, dg.MODE_DENSE)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    ix.profile(True)
    ids, sc, _ = ix.search(to_torch(Q, dtype, DEV), cls, K, want_pass=False)
    torch.cuda.synchronize()
    assert ix.profile_read()["launches"] == 9
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, (ids, sc, torch.from_numpy(ref[2])), ref, True,
          what=f"union two groups B{B} {preset}")
