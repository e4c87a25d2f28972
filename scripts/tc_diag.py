"""Batched-path diagnostics on a large shard: fallback count and per-user thresholds / key counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses

n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dt = dg.I8 if (len(sys.argv) < 4 or sys.argv[3] == "i8") else dg.BF16
B, K = 256, 1000
ix = Index(n, d, dt, 1)
ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, n)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, d, dt)
q = torch.from_numpy(Q if dt == dg.I8 else Q.view(np.int16)).view(torch.int8 if dt == dg.I8 else torch.bfloat16).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, B, "HIGH"))
c0 = ix.counters()["tc_fallbacks"]
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ix.search(q, cls, K, want_pass=False)
    torch.cuda.synchronize()
    print(f"search {it}: {1e3 * (time.perf_counter() - t0):.2f} ms, fallbacks so far {ix.counters()['tc_fallbacks'] - c0}")
ws = ix.workspace(B, 1, K)
print("ws bytes", ws.numel())
