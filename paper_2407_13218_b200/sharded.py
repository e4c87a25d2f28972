"""Row-sharded index over the GPUs of one node (BASELINE.json north_star: "The item index is
sharded row-wise across the 8 GPUs of one B200 box, each shard produces its local top-K, and an
NCCL allgather of K (score, item-id) pairs over NVLink feeds a final merge").

One process per GPU. Rank r owns global rows [r*ceil(N/G), min(N, (r+1)*ceil(N/G))). Queries and
clauses are replicated. Each rank runs the fused scan on its shard (linr_search_keys), the packed
u64 keys [B][K] + pass counts are all-gathered through torch.distributed (NCCL on GPUs), and every
rank merges the G lists with the library's merge kernel (linr_merge_keys). Exact by reading R13.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .linr import Index, merge_keys


def shard_range(n_total: int, world: int, rank: int):
    per = -(-n_total // world) if world > 0 else n_total
    lo = min(n_total, rank * per)
    hi = min(n_total, lo + per)
    return lo, hi, per


def _dist_info(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def exchange(keys: torch.Tensor, pas: torch.Tensor, group=None):
    """All-gather the shard results: keys [B][K], pass [B] -> [G][B][K], [G][B] (same device)."""
    rank, world = _dist_info(group)
    if world == 1:
        return keys[None], pas[None]
    backend = dist.get_backend(group)
    if backend == "nccl":
        gk = torch.empty((world,) + tuple(keys.shape), dtype=keys.dtype, device=keys.device)
        gp = torch.empty((world,) + tuple(pas.shape), dtype=pas.dtype, device=pas.device)
        dist.all_gather_into_tensor(gk, keys.contiguous(), group=group)
        dist.all_gather_into_tensor(gp, pas.contiguous(), group=group)
        return gk, gp
    lk = [torch.empty_like(keys) for _ in range(world)]
    lp = [torch.empty_like(pas) for _ in range(world)]
    dist.all_gather(lk, keys.contiguous(), group=group)
    dist.all_gather(lp, pas.contiguous(), group=group)
    return torch.stack(lk), torch.stack(lp)


def route_rows(rows: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Positions of the update rows this shard owns (§4.3 updates, routed by row id)."""
    return torch.nonzero((rows >= lo) & (rows < hi), as_tuple=False).flatten()


class ShardedIndex:
    def __init__(self, n_total: int, dim: int, dtype: int, attr_words: int = 1, group=None,
                 capacity: int | None = None, device=None):
        self.group = group
        self.rank, self.world = _dist_info(group)
        self.n_total = n_total
        self.lo, self.hi, self.per = shard_range(n_total, self.world, self.rank)
        cap = capacity if capacity is not None else max(1, self.per)
        self.local = Index(cap, dim, dtype, attr_words, global_row0=self.lo, device=device)
        self._out = {}

    def generate(self, seed: int, mode: int):
        """Fill this shard with the synthetic recipe (counters are global row ids)."""
        if self.hi > self.lo:
            self.local.generate(seed, mode, 0, self.hi - self.lo)

    def load(self, emb: torch.Tensor, attrs: torch.Tensor):
        """emb/attrs hold THIS shard's rows [lo, hi)."""
        self.local.load(emb, attrs, row0=self.lo)

    def update_rows(self, rows: torch.Tensor, emb: torch.Tensor, attrs: torch.Tensor):
        """Replicated update batch: each rank applies the rows it owns."""
        sel = route_rows(rows, self.lo, self.lo + self.local.capacity)
        if sel.numel():
            self.local.update_rows(rows[sel], emb[sel], attrs[sel])

    def delete_rows(self, rows: torch.Tensor):
        sel = route_rows(rows, self.lo, self.lo + self.local.capacity)
        if sel.numel():
            self.local.delete_rows(rows[sel])

    def search(self, queries: torch.Tensor, clauses, K: int):
        keys, ps = self.local.search_keys(queries, clauses, K)
        gk, gp = exchange(keys, ps, self.group)
        return merge_keys(gk, gp, K)
