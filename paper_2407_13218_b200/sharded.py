"""Row-sharded index over the GPUs of one node (BASELINE.json north_star: "The item index is
sharded row-wise across the 8 GPUs of one B200 box, each shard produces its local top-K, and an
NCCL allgather of K (score, item-id) pairs over NVLink feeds a final merge").

One process per GPU. Rank r owns global rows [r*per, (r+1)*per) with per = ceil(N/G) (the last
rank also owns every id past the end: growth rows), so every global id has exactly one owner.
Queries and clauses are replicated.

On NCCL process groups the whole search is ONE library call per rank: the index handle carries
an NCCL communicator (linr_comm_init, id created by linr_nccl_unique_id on rank 0 and broadcast),
and linr_search runs the fused scan, packs the shard's sorted keys + pass counts into one buffer,
all-gathers it and merges on every rank (exact by reading R13). On other backends (gloo: the CPU
tests of this host logic) the same exchange is composed here: linr_search_keys, all_gather of the
packed keys through torch.distributed, linr_merge_keys.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .linr import Index, merge_keys, nccl_unique_id


def shard_range(n_total: int, world: int, rank: int):
    """[lo, hi) of the rows rank owns among the first n_total, and per = ceil(n_total / world).
    Ranges are disjoint and ordered by rank even when trailing shards are empty."""
    per = max(1, -(-n_total // world)) if world > 0 else max(1, n_total)
    lo = rank * per
    hi = max(lo, min(n_total, lo + per))
    return lo, hi, per


def owner_of(rows: torch.Tensor, per: int, world: int) -> torch.Tensor:
    """Owning rank of each global row id: floor(id / per), the last rank taking every id beyond
    its range (growth rows); negative ids map to rank 0, which skips and counts them."""
    return torch.clamp(torch.div(rows, per, rounding_mode="floor"), 0, world - 1)


def _dist_info(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def exchange(keys: torch.Tensor, pas: torch.Tensor, group=None):
    """All-gather the shard results (non-NCCL groups): keys [B][K], pass [B] -> [G][B][K], [G][B].
    Keys and pass counts travel in ONE collective (packed [B][K+1] int64 per rank)."""
    rank, world = _dist_info(group)
    if world == 1:
        return keys[None], pas[None]
    B, K = keys.shape
    packed = torch.cat([keys.reshape(-1), pas.reshape(-1)]).contiguous()
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    g = torch.stack(parts)
    return g[:, :B * K].reshape(world, B, K).contiguous(), g[:, B * K:].contiguous()


def route_rows(rows: torch.Tensor, rank: int, per: int, world: int) -> torch.Tensor:
    """Positions of the update rows this rank owns (§4.3 updates, routed by row id)."""
    return torch.nonzero(owner_of(rows, per, world) == rank, as_tuple=False).flatten()


class ShardedIndex:
    def __init__(self, n_total: int, dim: int, dtype: int, attr_words: int = 1, group=None,
                 growth: int = 0, device=None):
        """growth: extra capacity on the LAST rank for rows appended past n_total."""
        self.group = group
        self.rank, self.world = _dist_info(group)
        self.n_total = n_total
        self.lo, self.hi, self.per = shard_range(n_total, self.world, self.rank)
        cap = self.per + (growth if self.rank == self.world - 1 else 0)
        self.local = Index(cap, dim, dtype, attr_words, global_row0=self.lo, device=device)
        self.lib_comm = False
        if self.world > 1 and dist.get_backend(group) == "nccl":
            uid = torch.zeros(128, dtype=torch.uint8, device=self.local.device)
            if self.rank == 0:
                uid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast(uid, src=src, group=group)
            self.local.attach_comm(bytes(uid.cpu().numpy().tobytes()), self.rank, self.world)
            self.lib_comm = True

    def generate(self, seed: int, mode: int):
        """Fill this shard with the synthetic recipe (counters are global row ids)."""
        if self.hi > self.lo:
            self.local.generate(seed, mode, 0, self.hi - self.lo)

    def load(self, emb: torch.Tensor, attrs: torch.Tensor):
        """emb/attrs hold THIS shard's rows [lo, hi)."""
        self.local.load(emb, attrs, row0=self.lo)

    def update_rows(self, rows: torch.Tensor, emb: torch.Tensor, attrs: torch.Tensor):
        """Replicated update batch: each rank applies exactly the rows it owns."""
        sel = route_rows(rows, self.rank, self.per, self.world)
        if sel.numel():
            self.local.update_rows(rows[sel], emb[sel], attrs[sel])

    def delete_rows(self, rows: torch.Tensor):
        sel = route_rows(rows, self.rank, self.per, self.world)
        if sel.numel():
            self.local.delete_rows(rows[sel])

    def search(self, queries: torch.Tensor, clauses, K: int):
        if self.lib_comm or self.world == 1:
            return self.local.search(queries, clauses, K)   # scan + allgather + merge in one C call
        keys, ps = self.local.search_keys(queries, clauses, K)
        gk, gp = exchange(keys, ps, self.group)
        return merge_keys(gk, gp, K)
