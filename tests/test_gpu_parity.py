"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element (-m gpu).

Exactness bar (BASELINE.json north_star / DESIGN.md R8-R10): int8 and integer-grid float inputs
are bit-exact (ids and scores); dense float inputs match per reading R9 (scores within the R8
tolerance, id sets equal except ties within tolerance at the K-th boundary).
"""
import numpy as np
import pytest
import torch

import datagen as dg
import oracle
from parity import check, make_index, to_torch, attrs_torch

pytestmark = pytest.mark.gpu
DEV = "cuda"


def run_case(dtype, d, n, B, V, K, preset, mode, live_frac=1.0, seed=dg.DATA_SEED, W=1, what=""):
    vals, attrs = dg.gen_items(seed, 0, n, d, dtype, mode, W=W)
    live = np.ones(n, np.uint8)
    ix = make_index(vals, attrs, dtype)
    if live_frac < 1.0:
        rng = np.random.default_rng(n + d)
        dead = np.nonzero(rng.random(n) > live_frac)[0]
        live[dead] = 0
        ix.delete_rows(torch.from_numpy(dead).to(DEV))
    Q = dg.gen_queries(dg.QUERY_SEED, seed, max(n, 1), B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    ref = oracle.search(dtype, vals, attrs, live, Q, cls, K)
    exact = dtype == dg.I8 or mode == dg.MODE_GRID
    check(dtype, vals, attrs, live, Q, cls, K, g, ref, exact, what=what)
    assert ix.stats()["overflow"] == 0
    return ix


def test_config_c1_full():
    """c1: 100k items, d=64 fp32, 4 clauses, 1 query, K=100 (BASELINE.json configs[0])."""
    run_case(dg.F32, 64, 100_000, 1, 1, 100, "HIGH4", dg.MODE_DENSE, what="c1 dense")
    run_case(dg.F32, 64, 100_000, 1, 1, 100, "HIGH4", dg.MODE_GRID, what="c1 grid")


@pytest.mark.parametrize("dtype", [dg.F32, dg.F16, dg.BF16, dg.I8])
@pytest.mark.parametrize("d", [16, 32, 64, 128, 256, 512, 1024])
def test_dtypes_dims_grid_exact(dtype, d):
    run_case(dtype, d, 20_011, 1, 1, 1000, "HIGH", dg.MODE_GRID, what=f"dt{dtype} d{d}")


@pytest.mark.parametrize("dtype", [dg.F16, dg.BF16])
def test_dense_tolerance(dtype):
    run_case(dtype, 128, 50_000, 2, 1, 500, "HIGH", dg.MODE_DENSE, what="dense")


@pytest.mark.parametrize("preset", ["ALL", "HIGH", "HIGH4", "LOW"])
@pytest.mark.parametrize("K", [1, 10, 1000, 2048])
def test_presets_and_K(preset, K):
    run_case(dg.I8, 128, 30_000 + 77, 1, 1, K, preset, dg.MODE_DENSE, what=f"{preset} K{K}")


@pytest.mark.parametrize("B,V", [(2, 1), (3, 1), (4, 1), (8, 1), (11, 1), (1, 2), (1, 8), (2, 4), (3, 2)])
def test_batches_and_multivector(B, V):
    run_case(dg.BF16, 128, 25_000, B, V, 300, "HIGH", dg.MODE_GRID, what=f"B{B} V{V}")
    run_case(dg.I8, 64, 25_000, B, V, 300, "LOW", dg.MODE_DENSE, what=f"i8 B{B} V{V}")


def test_liveness_and_multiword_attrs():
    run_case(dg.I8, 64, 40_000, 3, 1, 200, "HIGH", dg.MODE_DENSE, live_frac=0.7, what="live")
    # clauses on attribute words 1..3 (random 64-bit words)
    n, d, W = 20_000, 64, 4
    vals, attrs = dg.gen_items(3, 0, n, d, dg.I8, dg.MODE_DENSE, W=W)
    ix = make_index(vals, attrs, dg.I8)
    Q = dg.gen_queries(4, 3, n, 2, 1, d, dg.I8)
    cls = [[(0x00F0_0000_0000_00F0, 1, 0), (0x1, 3, 1), (0xFFFF << 24, 0, 1)],
           [(0x8000_0000_0000_0001, 2, 0)]]
    g = ix.search(to_torch(Q, dg.I8, DEV), cls, 100)
    ref = oracle.search(dg.I8, vals, attrs, np.ones(n), Q, cls, 100)
    check(dg.I8, vals, attrs, np.ones(n), Q, cls, 100, g, ref, True, what="multiword")


def test_no_clauses_and_zero_query_tie_break():
    n, d = 10_000, 64
    vals, attrs = dg.gen_items(5, 0, n, d, dg.BF16, dg.MODE_GRID)
    ix = make_index(vals, attrs, dg.BF16)
    Q = np.zeros((2, 1, d), np.uint16)   # bf16 zeros: every score is 0 -> lowest ids first
    cls = [[], [(0xFF << 56, 0, 0)]]
    g = ix.search(to_torch(Q, dg.BF16, DEV), cls, 50)
    ref = oracle.search(dg.BF16, vals, attrs, np.ones(n), Q, cls, 50)
    check(dg.BF16, vals, attrs, np.ones(n), Q, cls, 50, g, ref, True, what="zero query")
    assert g[0][0, :50].cpu().tolist() == list(range(50))


def test_empty_index_and_K_exceeds_pass():
    d = 64
    from paper_2407_13218_b200 import Index
    ix = Index(1000, d, dg.I8, 1)
    Q = dg.gen_queries(1, 1, 10, 2, 1, d, dg.I8)
    ids, sc, ps = ix.search(to_torch(Q, dg.I8, DEV), dg.gen_clauses(1, 2, "HIGH"), 16)
    assert (ids.cpu() == -1).all() and torch.isinf(sc.cpu()).all() and (ps.cpu() == 0).all()
    run_case(dg.I8, d, 3_000, 2, 1, 2048, "LOW", dg.MODE_DENSE, what="K > pass")


def test_adversarial_increasing_scores():
    """Scores increase with row id: every item beats the running threshold, so the CTA buffers
    compact as often as possible; the result must still be the last K passing rows."""
    n, d, K = 300_000, 16, 1000
    vals = np.zeros((n, d), np.float32)
    vals[:, 0] = np.arange(n, dtype=np.float32)
    attrs = np.full((n, 1), 1, np.uint64)
    ix = make_index(vals, attrs, dg.F32)
    q = np.zeros((1, d), np.float32)
    q[0, 0] = 1.0
    g = ix.search(torch.from_numpy(q).to(DEV), [[(1, 0, 0)]], K)
    ref = oracle.search(dg.F32, vals, attrs, np.ones(n), q, [[(1, 0, 0)]], K)
    check(dg.F32, vals, attrs, np.ones(n), q, [[(1, 0, 0)]], K, g, ref, True, what="increasing")
    assert ix.stats()["overflow"] == 0


def test_live_updates_replay_equivalence():
    """Upsert + delete in place (§4.3) then search == oracle on the final rows."""
    n, d, K = 60_000, 128, 500
    dtype = dg.BF16
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, dg.MODE_GRID)
    ix = make_index(vals, attrs, dtype, capacity=n + 5000)
    rng = np.random.default_rng(9)
    upd = rng.choice(n, 3000, replace=False)
    new_rows = np.concatenate([upd, np.arange(n, n + 2000)])          # overwrite + append beyond hwm
    nv, na = dg.gen_items(dg.UPDATE_SEED, 0, len(new_rows), d, dtype, dg.MODE_GRID)
    ix.update_rows(torch.from_numpy(new_rows).to(DEV), to_torch(nv, dtype, DEV), attrs_torch(na, DEV))
    dele = rng.choice(n, 4000, replace=False)
    ix.delete_rows(torch.from_numpy(dele).to(DEV))
    # out-of-shard ids are skipped and counted
    ix.delete_rows(torch.tensor([-5, n + 999_999], device=DEV))
    st = ix.stats()
    assert st["hwm"] == n + 2000 and st["skipped"] == 2
    fv = np.concatenate([vals, np.zeros((2000, d), vals.dtype)])
    fa = np.concatenate([attrs, np.zeros((2000, 1), np.uint64)])
    fv[new_rows], fa[new_rows] = nv, na
    live = np.ones(n + 2000, np.uint8)
    live[dele] = 0
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, 3, 1, d, dtype, dg.MODE_GRID)
    cls = dg.gen_clauses(dg.QUERY_SEED, 3, "HIGH")
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    ref = oracle.search(dtype, fv, fa, live, Q, cls, K)
    check(dtype, fv, fa, live, Q, cls, K, g, ref, True, what="updates")


@pytest.mark.parametrize("dtype", [dg.F32, dg.F16, dg.BF16, dg.I8])
@pytest.mark.parametrize("mode", [dg.MODE_GRID, dg.MODE_DENSE])
def test_device_generator_matches_datagen(dtype, mode):
    from paper_2407_13218_b200 import generate_rows
    d, W = 128, 3
    emb, att = generate_rows(dtype, d, W, dg.DATA_SEED, mode, 123_456, 5000)
    v, a = dg.gen_items(dg.DATA_SEED, 123_456, 5000, d, dtype, mode, W=W)
    ge = emb.cpu()
    if dtype in (dg.F16, dg.BF16):
        ge = ge.view(torch.int16).numpy().view(np.uint16)
    else:
        ge = ge.numpy()
    assert np.array_equal(ge, v)
    assert np.array_equal(att.cpu().numpy().view(np.uint64), a)


def test_index_generate_equals_load():
    n, d = 50_000, 64
    from paper_2407_13218_b200 import Index
    ix = Index(n, d, dg.I8, 1, global_row0=1000)
    ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, n)
    vals, attrs = dg.gen_items(dg.DATA_SEED, 1000, n, d, dg.I8)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, 2, 1, d, dg.I8)
    cls = dg.gen_clauses(dg.QUERY_SEED, 2, "HIGH")
    g = ix.search(to_torch(Q, dg.I8, DEV), cls, 100)
    ref = oracle.search(dg.I8, vals, attrs, np.ones(n), Q, cls, 100, row0=1000)
    check(dg.I8, vals, attrs, np.ones(n), Q, cls, 100, g, ref, True, row0=1000, what="generate")


@pytest.mark.parametrize("G", [2, 3, 8])
def test_virtual_shards_merge(G):
    """Row-sharded search on one GPU: G shards with global_row0 offsets, shard-local keys, then
    the merge kernel (the same kernel the multi-GPU all-gather feeds) == one index == oracle."""
    from paper_2407_13218_b200 import Index, merge_keys
    n, d, K, B = 80_000, 128, 1000, 2
    dtype = dg.I8
    per = -(-n // G)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dtype)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    qt = to_torch(Q, dtype, DEV)
    keys, ps = [], []
    for r in range(G):
        lo, hi = r * per, min(n, (r + 1) * per)
        ix = Index(per, d, dtype, 1, global_row0=lo)
        ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, hi - lo)
        k, p = ix.search_keys(qt, cls, K)
        keys.append(k)
        ps.append(p)
    g = merge_keys(torch.stack(keys), torch.stack(ps), K)
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype)
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, True, what=f"shards{G}")


def test_search_host_e2e_path():
    n, d, K = 30_000, 128, 100
    vals, attrs = dg.gen_items(1, 0, n, d, dg.BF16, dg.MODE_GRID)
    ix = make_index(vals, attrs, dg.BF16)
    Q = dg.gen_queries(2, 1, n, 3, 1, d, dg.BF16, dg.MODE_GRID)
    cls = dg.gen_clauses(2, 3, "HIGH")
    qh = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).contiguous().pin_memory()
    g = ix.search_host(qh, cls, K)
    ref = oracle.search(dg.BF16, vals, attrs, np.ones(n), Q, cls, K)
    check(dg.BF16, vals, attrs, np.ones(n), Q, cls, K, g, ref, True, what="host")


def test_search_host_async_pipelined():
    """linr_search_host_async: searches of different queries in flight on two streams (own
    workspaces, pinned host buffers), each equal to the oracle after its stream is synchronised."""
    n, d, K = 200_000, 128, 1000
    vals, attrs = dg.gen_items(3, 0, n, d, dg.BF16, dg.MODE_GRID)
    ix = make_index(vals, attrs, dg.BF16)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    cases = []
    for j, preset in enumerate(["HIGH", "ALL", "LOW", "HIGH4"]):
        Q = dg.gen_queries(10 + j, 3, n, 1, 1, d, dg.BF16, dg.MODE_GRID)
        cls = dg.gen_clauses(10 + j, 1, preset)
        qh = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).contiguous().pin_memory()
        out = (torch.empty((1, K), dtype=torch.int64, pin_memory=True),
               torch.empty((1, K), dtype=torch.float32, pin_memory=True),
               torch.empty(1, dtype=torch.int64, pin_memory=True))
        cases.append((Q, cls, qh, out))
    wss = [ix.new_workspace(1, 1, K, host_extra=True) for _ in streams]
    for j, (Q, cls, qh, out) in enumerate(cases):
        s = streams[j % 2]
        s.synchronize()
        if j >= 2:   # this stream's previous search has completed: check it before reuse
            pQ, pcls, _, pout = cases[j - 2]
            ref = oracle.search(dg.BF16, vals, attrs, np.ones(n), pQ, pcls, K)
            check(dg.BF16, vals, attrs, np.ones(n), pQ, pcls, K, tuple(t.clone() for t in pout), ref, True, what="async")
            cases[j - 2] = None
        with torch.cuda.stream(s):
            ix.search_host(qh, cls, K, out=out, ws=wss[j % 2], sync=False)
    for s in streams:
        s.synchronize()
    for c in cases:
        if c is None:
            continue
        Q, cls, _, out = c
        ref = oracle.search(dg.BF16, vals, attrs, np.ones(n), Q, cls, K)
        check(dg.BF16, vals, attrs, np.ones(n), Q, cls, K, out, ref, True, what="async")


def test_concurrent_searches_on_streams():
    """Searches of one index in flight on several streams (own workspaces; the fused merge's
    per-search ticket slots) give the same results as the oracle, for many interleaved calls."""
    n, d, K = 120_000, 128, 200
    vals, attrs = dg.gen_items(3, 0, n, d, dg.BF16, dg.MODE_GRID)
    ix = make_index(vals, attrs, dg.BF16)
    presets = ["HIGH", "LOW", "ALL", "HIGH4"]
    Qs = [dg.gen_queries(10 + i, 3, n, 1, 1, d, dg.BF16, dg.MODE_GRID) for i in range(4)]
    cls = [dg.gen_clauses(10 + i, 1, presets[i]) for i in range(4)]
    qd = [to_torch(Q, dg.BF16, DEV) for Q in Qs]
    streams = [torch.cuda.Stream(DEV) for _ in range(3)]
    wss = [ix.new_workspace(1, 1, K) for _ in range(3)]
    outs = []
    torch.cuda.synchronize()
    for k in range(24):
        j, i = k % 3, k % 4
        with torch.cuda.stream(streams[j]):
            outs.append((i, ix.search(qd[i], cls[i], K, ws=wss[j])))
            outs[-1] = (i, tuple(t.clone() for t in outs[-1][1]))   # snapshot before the stream reuses ws
    torch.cuda.synchronize()
    refs = [oracle.search(dg.BF16, vals, attrs, np.ones(n), Qs[i], cls[i], K) for i in range(4)]
    for k, (i, g) in enumerate(outs):
        check(dg.BF16, vals, attrs, np.ones(n), Qs[i], cls[i], K, g, refs[i], True, what=f"stream call {k}")


def test_invalid_arguments_raise():
    from paper_2407_13218_b200 import Index, LinrError
    ix = Index(1000, 64, dg.I8, 1)
    q = torch.zeros((1, 64), dtype=torch.int8, device=DEV)
    with pytest.raises(LinrError):
        ix.search(q, [[(0, 0, 0)]], 10)          # empty clause mask (reading R3)
    with pytest.raises(LinrError):
        ix.search(q, [[(1, 1, 0)]], 10)          # word >= W
    with pytest.raises(LinrError):
        ix.search(q, [[]], 4096)                 # K > 2048
    with pytest.raises(LinrError):
        ix.load(torch.zeros((10, 64), dtype=torch.int8, device=DEV),
                torch.zeros((10, 1), dtype=torch.int64, device=DEV), row0=995)   # ERANGE


# ---------------------------------------------------------------- batched tcgen05 path (B*V >= 16)
@pytest.mark.parametrize("dtype,d,B,V,K,preset,n", [
    (dg.BF16, 128, 32, 1, 100, "HIGH", 100_000),
    (dg.BF16, 128, 17, 1, 1000, "ALL", 60_000),
    (dg.F16, 128, 64, 1, 50, "HIGH4", 40_000),
    (dg.I8, 128, 16, 1, 1000, "LOW", 300_000),
    (dg.I8, 64, 256, 1, 20, "HIGH", 30_000),
    (dg.BF16, 64, 4, 8, 300, "HIGH", 80_000),
    (dg.BF16, 128, 256, 1, 1000, "HIGH", 200_000),
    (dg.BF16, 128, 32, 8, 1000, "HIGH", 100_000),     # c5 U=32: 256 query vectors, max-merged per user
    (dg.I8, 128, 16, 8, 500, "HIGH4", 60_000),
    (dg.F16, 64, 64, 2, 200, "LOW", 200_000),
    (dg.BF16, 128, 12, 1, 1000, "HIGH", 100_000),     # B*V in [LINR_TC_MIN, 16): NP = 16, padded columns
    (dg.I8, 64, 5, 2, 300, "LOW", 200_000),
])
def test_batched_tensor_core_path(dtype, d, B, V, K, preset, n):
    mode = dg.MODE_DENSE if dtype == dg.I8 else dg.MODE_GRID
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    ix.profile(True)
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    prof = ix.profile_read()
    assert prof["launches"] == 6, prof   # sample, threshold, main, finalize, fallback, pass count: the tcgen05 path ran
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, True, what=f"tc dt{dtype} d{d} B{B} V{V}")


# Kernel variants selected by the library's tuning knobs (read at plan time, per search): the
# per-warp scan for tensor-core shapes (LINR_NO_WS), the merge fused into the scan's last CTAs
# (LINR_FUSE_MERGE), a tiny per-user buffer (LINR_WS_CMAX: many consumer-side compactions while
# the producers keep gathering) and a small ring (LINR_WS_RING_KB: slot reuse every few groups).
@pytest.mark.parametrize("env", [{"LINR_NO_WS": "1"}, {"LINR_FUSE_MERGE": "1"}, {"LINR_WS_CMAX": "1280"},
                                 {"LINR_WS_RING_KB": "16"}, {"LINR_WS_CMAX": "1280", "LINR_WS_RING_KB": "16"}])
@pytest.mark.parametrize("dtype,d,B,V,preset", [(dg.BF16, 128, 1, 1, "ALL"), (dg.I8, 64, 1, 1, "HIGH"),
                                                (dg.BF16, 64, 3, 2, "ALL"), (dg.I8, 128, 2, 1, "LOW")])
def test_kernel_variants(monkeypatch, env, dtype, d, B, V, preset):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    run_case(dtype, d, 300_000, B, V, 1000, preset, dg.MODE_GRID, what=f"variant {env}")


@pytest.mark.parametrize("dtype,d,B,V,K,preset,n", [
    (dg.BF16, 128, 64, 1, 1000, "HIGH", 150_000),
    (dg.F16, 128, 32, 1, 200, "ALL", 60_000),
    (dg.BF16, 64, 8, 4, 300, "HIGH4", 80_000),
    (dg.F16, 64, 256, 1, 50, "HIGH", 40_000),
    (dg.BF16, 128, 32, 8, 1000, "HIGH", 100_000),
])
def test_batched_tensor_core_dense(dtype, d, B, V, K, preset, n):
    """The tcgen05 path on dense (full-mantissa) inputs: scores rebuilt as acc + t_eff (reading R22)
    must sit inside the R8 tolerance and the id sets obey R9."""
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, dg.MODE_DENSE)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, dg.MODE_DENSE)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    ix.profile(True)
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    assert ix.profile_read()["launches"] == 6
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, False, what=f"tc dense dt{dtype} d{d} B{B} V{V}")


@pytest.mark.parametrize("dtype,mode,d,B,V,K,preset", [
    (dg.BF16, dg.MODE_GRID, 128, 32, 1, 500, "HIGH"),
    (dg.I8, dg.MODE_DENSE, 64, 16, 1, 1000, "ALL"),
    (dg.F16, dg.MODE_DENSE, 128, 8, 2, 100, "HIGH4"),
    (dg.BF16, dg.MODE_GRID, 64, 4, 8, 2048, "LOW"),
])
def test_batched_certification_fallback_forced(monkeypatch, dtype, mode, d, B, V, K, preset):
    """LINR_TC_MAIN_CAP shrinks the per-(user, CTA) candidate regions of the main pass so they
    overflow: every affected user is flagged by the finalize kernel and recomputed exactly on the
    device (fallback.cu, reading R23). The result must still equal the oracle, and the device
    counter must show the recomputations."""
    monkeypatch.setenv("LINR_TC_MAIN_CAP", "2")
    n = 120_000
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    before = ix.counters()["tc_fallbacks"]
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    c = ix.counters()
    assert c["tc_fallbacks"] - before > 0, c
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    exact = dtype == dg.I8 or mode == dg.MODE_GRID
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, exact, what=f"fallback dt{dtype} B{B} V{V}")
    # keys form (shard-local search) takes the same fallback
    k, ps = ix.search_keys(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    assert ix.counters()["tc_fallbacks"] > c["tc_fallbacks"]
    from paper_2407_13218_b200 import merge_keys
    g2 = merge_keys(k[None], ps[None], K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g2, ref, exact, what="fallback keys")


@pytest.mark.parametrize("dtype,mode,d,B,K,preset", [
    (dg.BF16, dg.MODE_GRID, 128, 32, 500, "ALL"),
    (dg.I8, dg.MODE_DENSE, 64, 20, 1000, "HIGH"),
])
def test_batched_finalize_exact_select_from_regions(monkeypatch, dtype, mode, d, B, K, preset):
    """LINR_TC_FIN_ROOM shrinks the finalize's shared-memory room below a user's key count: the
    K-th key is then selected exactly from the regions in global memory (no fallback, no flag)."""
    monkeypatch.setenv("LINR_TC_FIN_ROOM", str(K))
    n = 200_000
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    f0 = ix.counters()["tc_fallbacks"]
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    assert ix.counters()["tc_fallbacks"] == f0
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, True, what="finalize global select")


@pytest.mark.parametrize("dtype,mode,d,B,V,K,preset,n", [
    (dg.BF16, dg.MODE_GRID, 128, 32, 1, 10, "HIGH", 500_000),
    (dg.I8, dg.MODE_DENSE, 64, 64, 1, 5, "ALL", 400_000),
    (dg.F16, dg.MODE_DENSE, 128, 8, 2, 20, "HIGH4", 600_000),
])
def test_batched_threshold_refinement(dtype, mode, d, B, V, K, preset, n):
    """Small K * sampled / rows (< 8): a second, main-style sample pass refines the thresholds
    (8 launches instead of 6); results stay exact (int8 / grid) or within R8/R9 (dense)."""
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    ix.profile(True)
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    assert ix.profile_read()["launches"] == 8
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    exact = dtype == dg.I8 or mode == dg.MODE_GRID
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, exact, what=f"refine dt{dtype} B{B}")


def test_batched_fallback_not_taken_normally():
    n, d, B, K = 200_000, 128, 64, 1000
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dg.BF16, dg.MODE_GRID)
    ix = make_index(vals, attrs, dg.BF16)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dg.BF16, dg.MODE_GRID)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    ix.search(to_torch(Q, dg.BF16, DEV), cls, K)
    assert ix.counters()["tc_fallbacks"] == 0


@pytest.mark.parametrize("B", [1, 64])
def test_search_does_not_block_the_host(B):
    """linr_search enqueues and returns (include/linr.h conventions): with a long spin kernel queued
    ahead of it on the stream, the call returns while the stream is still busy -- on the GEMV path
    and on the batched tcgen05 path (whose certification runs on the device)."""
    n, d, K = 100_000, 128, 100
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dg.BF16, dg.MODE_GRID)
    ix = make_index(vals, attrs, dg.BF16)
    Q = to_torch(dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dg.BF16, dg.MODE_GRID), dg.BF16, DEV)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    ix.search(Q, cls, K)   # warm-up: workspace allocation, attributes
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    torch.cuda._sleep(2_000_000_000)   # ~1 s of device time ahead of the search
    ix.search(Q, cls, K)
    busy = not s.query()
    torch.cuda.synchronize()
    assert busy, "linr_search synchronised the stream"


@pytest.mark.parametrize("B,dtype,mode", [(2, dg.I8, dg.MODE_DENSE), (32, dg.BF16, dg.MODE_GRID)])
def test_nccl_communicator_search_world1(B, dtype, mode):
    """The library's own NCCL exchange (linr_nccl_unique_id + linr_comm_init; linr_search then packs
    keys + pass counts, runs ncclAllGather and the merge kernel in the same call). One GPU here, so
    the communicator has one rank: the branch runs end to end and must equal the oracle."""
    from paper_2407_13218_b200 import nccl_unique_id
    n, d, K = 90_000, 128, 700
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype)
    ix.attach_comm(nccl_unique_id(), 0, 1)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    g = ix.search(to_torch(Q, dtype, DEV), cls, K)
    torch.cuda.synchronize()
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, True, what=f"nccl B{B}")
    qh = torch.from_numpy(np.ascontiguousarray(Q).view(np.int16 if dtype != dg.I8 else np.int8))
    if dtype == dg.BF16:
        qh = qh.view(torch.bfloat16)
    g2 = ix.search_host(qh.contiguous().pin_memory(), cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g2, ref, True, what=f"nccl host B{B}")


def test_update_duplicate_ids_last_writer_wins():
    """an id repeated within one update call is written by its last occurrence only."""
    n, d, K = 5_000, 64, 50
    vals, attrs = dg.gen_items(1, 0, n, d, dg.I8)
    ix = make_index(vals, attrs, dg.I8)
    rows = np.array([7, 9, 7, 7, 100, 9], np.int64)
    nv, na = dg.gen_items(2, 0, len(rows), d, dg.I8)
    ix.update_rows(torch.from_numpy(rows).to(DEV), to_torch(nv, dg.I8, DEV), attrs_torch(na, DEV))
    fv, fa = vals.copy(), attrs.copy()
    for j, r in enumerate(rows):   # sequential application == last writer wins
        fv[r], fa[r] = nv[j], na[j]
    Q = dg.gen_queries(3, 1, n, 2, 1, d, dg.I8)
    cls = [[], [(0xFF << 56, 0, 0)]]
    g = ix.search(to_torch(Q, dg.I8, DEV), cls, K)
    ref = oracle.search(dg.I8, fv, fa, np.ones(n), Q, cls, K)
    check(dg.I8, fv, fa, np.ones(n), Q, cls, K, g, ref, True, what="dup updates")
    assert ix.emb_storage[:n * d].view(torch.int8).reshape(n, d)[7].cpu().numpy().tolist() == nv[3].tolist()
