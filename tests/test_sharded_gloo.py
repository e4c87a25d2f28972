"""Multi-process (world_size 2, gloo, CPU) tests of the row-sharding host logic (-m "not gpu").

What runs on CPU: shard_range partitioning, the key exchange (sharded.exchange over
torch.distributed all_gather, keys and pass counts in one collective), single-owner update
routing (sharded.route_rows / owner_of). The per-shard top-K on each
rank comes from the oracle (no GPU here) packed into the ABI's u64 key format by this test; the
gathered lists are merged with oracle.merge and must equal the oracle on the unsharded index
(reading R13). The GPU side of the same path (linr_search_keys + linr_merge_keys) is covered by
tests/test_gpu_parity.py::test_virtual_shards_merge.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen as dg
import oracle
from paper_2407_13218_b200.sharded import exchange, owner_of, route_rows, shard_range

N, D, K, B = 6_000, 64, 50, 3


def pack_keys(ids, scores):
    """ABI key: (ordered_u32(fp32 score) << 32) | (0xFFFFFFFF - id); 0 for padding."""
    out = np.zeros(ids.shape, dtype=np.uint64)
    for idx in np.ndindex(ids.shape):
        i = int(ids[idx])
        if i < 0:
            continue
        u = int(np.float32(scores[idx]).view(np.uint32))
        if (u << 1) & 0xFFFFFFFF == 0:
            u = 0
        o = (~u) & 0xFFFFFFFF if u & 0x80000000 else (u | 0x80000000)
        out[idx] = (o << 32) | (0xFFFFFFFF - i)
    return out


def unpack_keys(keys):
    ids = np.full(keys.shape, -1, dtype=np.int64)
    sc = np.full(keys.shape, -np.inf)
    for idx in np.ndindex(keys.shape):
        k = int(keys[idx])
        if k == 0:
            continue
        o = k >> 32
        u = (o & 0x7FFFFFFF) if o & 0x80000000 else (~o) & 0xFFFFFFFF
        sc[idx] = float(np.uint32(u).view(np.float32))
        ids[idx] = 0xFFFFFFFF - (k & 0xFFFFFFFF)
    return ids, sc


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi, per = shard_range(N, world, rank)
        vals, attrs = dg.gen_items(dg.DATA_SEED, lo, hi - lo, D, dg.I8)
        Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, N, B, 1, D, dg.I8)
        cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
        ids, sc, ps = oracle.search(dg.I8, vals, attrs, np.ones(hi - lo, np.uint8), Q, cls, K, row0=lo)
        keys = torch.from_numpy(pack_keys(ids, sc).view(np.int64))
        gk, gp = exchange(keys, torch.from_numpy(ps), None)
        gids, gsc = unpack_keys(gk.numpy().view(np.uint64))
        merged = oracle.merge(gids, gsc, gp.numpy(), K)
        # update routing: every rank sees the same replicated batch, keeps only its rows
        rows = torch.tensor([0, per - 1, per, N - 1, N + 5, -1])
        mine = rows[route_rows(rows, rank, per, world)].tolist()
        out.put((rank, [m.tolist() for m in merged], mine, (lo, hi)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_exchange_and_merge_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, N, D, dg.I8)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, N, B, 1, D, dg.I8)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, "HIGH")
    full = oracle.search(dg.I8, vals, attrs, np.ones(N, np.uint8), Q, cls, K)
    per = -(-N // world)
    for rank, merged, mine, (lo, hi) in res:
        assert np.array_equal(np.array(merged[0]), full[0]), rank
        assert np.array_equal(np.array(merged[1]), full[1]), rank
        assert np.array_equal(np.array(merged[2]), full[2]), rank
        # single owner per id: [r*per, (r+1)*per), the last rank also takes growth rows, rank 0 the
        # invalid negative ids (skipped and counted on the device)
        rows = [0, per - 1, per, N - 1, N + 5, -1]
        want = [r for r in rows if min(max(r // per, 0), world - 1) == rank]
        assert mine == want
    owned = sorted(sum((m for _, _, m, _ in res), []))
    assert owned == sorted([0, per - 1, per, N - 1, N + 5, -1])   # every id routed exactly once


def test_key_packing_roundtrip_and_order():
    ids = np.array([[3, 7, 1, -1]])
    sc = np.array([[2.5, -1.0, 2.5, -np.inf]])
    k = pack_keys(ids, sc)
    # order: score desc, then id asc
    assert k[0, 2] > k[0, 0] > k[0, 1] > k[0, 3] == 0
    i2, s2 = unpack_keys(k)
    assert i2.tolist() == ids.tolist()
    assert s2[0, :3].tolist() == sc[0, :3].tolist()


def test_shard_range_covers_exactly():
    for n in (1, 7, 100, 1001):
        for g in (1, 2, 3, 8):
            cov = []
            for r in range(g):
                lo, hi, per = shard_range(n, g, r)
                assert hi - lo <= per
                cov.extend(range(lo, hi))
            assert cov == list(range(n))


def test_owner_routing_is_unique_with_empty_shards():
    """shard_range(10, 8) used to give ranks 5-7 the same lo (overlapping routing)."""
    n, g = 10, 8
    los = [shard_range(n, g, r)[0] for r in range(g)]
    assert los == sorted(set(los))                  # disjoint, ordered
    rows = torch.arange(-3, 40)
    own = owner_of(rows, shard_range(n, g, 0)[2], g)
    for r in range(g):
        sel = route_rows(rows, r, shard_range(n, g, 0)[2], g)
        assert torch.equal(own[sel], torch.full_like(sel, r))
    counts = sum(route_rows(rows, r, 2, g).numel() for r in range(g))
    assert counts == rows.numel()                   # each id goes to exactly one rank
