"""Live updates interleaved with searches: version-tag snapshot pin (SURVEY §8(c) "Live update";
PAPER.md P:4427-4429 Upsert/Delete with "minimal data access serialization"; SPEC S:81 snapshot
consistency; reading R16: a search sees every row wholly old or wholly new).

Row r at version v stores v in embedding coordinate 0 and in attribute bits 56-63 (the level
field). The query is the basis vector e_0, so a row's score IS the version its embedding holds;
the clause selects rows whose attribute byte holds an odd version. After every update call the
next search (same stream) must equal the oracle on the host replica of the index at that point
of the stream, and every returned row's score (embedding version) must be odd (attribute
version): a row whose new attributes were seen with its old embedding would break either check.
"""
import numpy as np
import pytest
import torch

import datagen as dg
import oracle
from parity import check, make_index, to_torch, attrs_torch

pytestmark = pytest.mark.gpu
DEV = "cuda"
LEVEL_OFF = 56


def _odd_version_clause():
    # one Match clause over the attribute byte 56..63 holding the version: odd versions have bit 56
    return [(1 << LEVEL_OFF, 0, 0)]


def _set_version(vals, attrs, rows, v, base_attrs):
    vals[rows, 0] = v
    attrs[rows, 0] = (base_attrs[rows, 0] & np.uint64((1 << LEVEL_OFF) - 1)) | (np.uint64(v) << np.uint64(LEVEL_OFF))


@pytest.mark.parametrize("dtype,d", [(dg.I8, 64), (dg.BF16, 128)])
@pytest.mark.parametrize("B", [1, 16])
def test_version_tags_interleaved_updates(dtype, d, B):
    n, K, steps, per_call = 40_000, 1500, 24, 700
    vals, attrs0 = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, dg.MODE_GRID)
    vals = vals.copy()
    attrs = attrs0.copy()
    ver = np.zeros(n, np.int64)
    if dtype == dg.I8:
        enc = lambda v: np.int8(v)                                   # noqa: E731
    else:
        enc = lambda v: dg._store(np.array([v], np.float32), dtype)[0]   # noqa: E731  (small ints are exact)
    rng = np.random.default_rng(4429)
    start = rng.integers(0, 4, n)
    for v in range(4):
        rows = np.nonzero(start == v)[0]
        ver[rows] = v
        _set_version(vals, attrs, rows, enc(v), attrs0)
    ix = make_index(vals, attrs, dtype)
    live = np.ones(n, np.uint8)
    q = np.zeros((B, 1, d), np.float32)
    q[:, 0, 0] = 1.0
    Q = q.astype(np.int8) if dtype == dg.I8 else dg._store(q, dtype)
    Qt = to_torch(Q, dtype, DEV)
    cls = [_odd_version_clause() for _ in range(B)]
    for step in range(steps):
        rows = rng.choice(n, per_call, replace=False)
        ver[rows] += 1 + rng.integers(0, 2, per_call)                # sometimes parity flips, sometimes not
        for r in rows:
            _set_version(vals, attrs, np.array([r]), enc(int(ver[r])), attrs0)
        ix.update_rows(torch.from_numpy(rows).to(DEV), to_torch(vals[rows], dtype, DEV),
                       attrs_torch(attrs[rows], DEV))
        live[rows] = 1                                               # an upsert revives a deleted row (R7)
        if step % 3 == 2:                                            # deletes on the same stream too
            dele = rng.choice(n, 50, replace=False)
            live[dele] = 0
            ix.delete_rows(torch.from_numpy(dele).to(DEV))
        g = ix.search(Qt, cls, K)
        torch.cuda.synchronize()
        ref = oracle.search(dtype, vals, attrs, live, Q, cls, K)
        check(dtype, vals, attrs, live, Q, cls, K, g, ref, True, what=f"step {step}")
        gi, gs = g[0].cpu().numpy(), g[1].cpu().numpy()
        for b in range(B):
            m = gi[b] >= 0
            assert np.all(gs[b][m].astype(np.int64) % 2 == 1), "a row's embedding version disagrees with its attributes"
            assert np.all(gs[b][m].astype(np.int64) == ver[gi[b][m]]), "a row is seen at a stale version"
    assert int(ver.max()) < 127
