"""Merge-kernel latency probe: is merge_kernel bound by its algorithm or by cold instruction /
data fetch? Times linr_merge_keys on L = 147 sorted partition lists (the scan merge's shape,
K = 1000) back to back (warm) and with a 512 MB copy between calls (L2 flushed, cold), CUDA events
around the merge only. Run on the GPU box; prints one line per mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2407_13218_b200.linr import merge_keys

dev = torch.device("cuda", 0)
L, B, K = 147, 1, 1000
g = torch.Generator(device="cpu").manual_seed(7)
# distinct positive keys, a cluster of high scores spread over the partitions like a real scan
keys = torch.randint(1 << 40, 1 << 62, (L, B, K), generator=g, dtype=torch.int64)
keys = torch.sort(keys, dim=-1, descending=True).values.to(dev)
pas = torch.full((L, B), 5000, dtype=torch.int64, device=dev)
out = (torch.empty((B, K), dtype=torch.int64, device=dev), torch.empty((B, K), dtype=torch.float32, device=dev),
       torch.empty(B, dtype=torch.int64, device=dev))
big_a = torch.empty(256 << 20, dtype=torch.int16, device=dev)
big_b = torch.empty_like(big_a)
st = torch.cuda.current_stream(dev)


def run(n, flush):
    ts = []
    for _ in range(n):
        if flush:
            big_b.copy_(big_a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        merge_keys(keys, pas, K, out=out)
        e1.record(st)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
    return v[len(v) // 2], v[0]


run(5, False)
for flush in (False, True):
    med, mn = run(200, flush)
    print(f"merge L={L} K={K} {'cold (L2 flushed)' if flush else 'warm'}: median {med:.2f} us, min {mn:.2f} us "
          f"(LINR_MERGE_BUCKET={os.environ.get('LINR_MERGE_BUCKET', '0')})")
