"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py times (-m gpu).

The index is generated in place on the device (linr_index_generate, the configuration bench.py
uses); the oracle side regenerates the same rows on the host with datagen/ in row chunks and
composes per-chunk oracle results with oracle.merge (exact by reading R13, pinned in
tests/test_oracle.py::test_shard_merge_equals_full_index).
"""
import numpy as np
import pytest
import torch

import datagen as dg
import oracle
from parity import check, to_torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda"


def chunked_oracle(dtype, d, n, mode, Q, cls, K, chunk=1 << 21):
    outs = []
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        vals, attrs = dg.gen_items(dg.DATA_SEED, a, b - a, d, dtype, mode)
        outs.append(oracle.search(dtype, vals, attrs, np.ones(b - a, np.uint8), Q, cls, K, row0=a))
    ids = np.stack([o[0] for o in outs])
    sc = np.stack([o[1] for o in outs])
    ps = np.stack([o[2] for o in outs])
    return oracle.merge(ids, sc, ps, K)


def sampled_rows(dtype, d, mode, ids):
    vals = dg.item_values(dg.DATA_SEED, ids, d, dtype, mode)
    attrs = dg.item_attrs(dg.DATA_SEED, ids, 1)
    return vals, attrs


def run_full(dtype, d, n, B, V, K, preset, mode, check_queries=None):
    from paper_2407_13218_b200 import Index
    ix = Index(n, d, dtype, 1)
    ix.generate(dg.DATA_SEED, mode, 0, n)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    gi, gs, gp = [t.cpu().numpy() for t in ix.search(to_torch(Q, dtype, DEV), cls, K)]
    assert ix.stats()["overflow"] == 0
    sel = list(range(B)) if check_queries is None else check_queries
    Qs = Q[sel]
    clss = [cls[b] for b in sel]
    ref = chunked_oracle(dtype, d, n, mode, Qs, clss, K)
    # the oracle side only has the rows it needs: build a compact view of the returned + oracle ids
    need = np.unique(np.concatenate([gi[sel].ravel(), ref[0].ravel()]))
    need = need[need >= 0]
    vals, attrs = sampled_rows(dtype, d, mode, need)
    remap = {int(g): i for i, g in enumerate(need)}
    # check() expects dense local rows: translate ids to positions in the sampled set
    gl = np.vectorize(lambda x: remap.get(int(x), -1))(gi[sel]) if len(need) else gi[sel]
    rl = np.vectorize(lambda x: remap.get(int(x), -1))(ref[0]) if len(need) else ref[0]
    exact = dtype == dg.I8 or mode == dg.MODE_GRID
    check(dtype, vals, attrs, np.ones(len(need), np.uint8), Qs, clss, K,
          (gl, gs[sel], gp[sel]), (rl, ref[1], ref[2]), exact, what=f"full dt{dtype} n{n}")


def test_c2_bf16_10M_B1_high():
    run_full(dg.BF16, 128, 10_000_000, 1, 1, 1000, "HIGH", dg.MODE_DENSE)


def test_c2_bf16_10M_B1_all_grid_exact():
    run_full(dg.BF16, 128, 10_000_000, 1, 1, 1000, "ALL", dg.MODE_GRID)


def test_c3_int8_shard_12p5M_high():
    """c3 per-GPU shard at G=8 (100M/8 rows, int8 d=128), exact."""
    run_full(dg.I8, 128, 12_500_000, 1, 1, 1000, "HIGH", dg.MODE_DENSE)


def test_c4_int8_d64_shard_low():
    """c4-shaped shard (int8 d=64, 1B/8 rows would be 125M; 20M here), exact, LOW preset."""
    run_full(dg.I8, 64, 20_000_000, 1, 1, 1000, "LOW", dg.MODE_DENSE)


def test_c2_bf16_10M_B256_dense_tcgen05():
    """c2 at B=256 (the batched tcgen05 path bench.py times) on dense inputs: R8/R9 tolerance,
    checked on sampled queries (first, middle, last) against the chunked oracle."""
    run_full(dg.BF16, 128, 10_000_000, 256, 1, 1000, "HIGH", dg.MODE_DENSE, check_queries=[0, 101, 255])
