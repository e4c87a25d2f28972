"""Profiling driver: build the bench workload (c2) and run a few searches (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses

ap = argparse.ArgumentParser()
ap.add_argument("--items", type=int, default=10_000_000)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--V", type=int, default=1)
ap.add_argument("--K", type=int, default=1000)
ap.add_argument("--preset", default="HIGH")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--no-pass", action="store_true", help="no pass counts (the bench configuration for B > 8)")
a = ap.parse_args()
dt = dg.DTYPE_NAMES[a.dtype]
ix = Index(a.items, a.dim, dt, 1)
ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, a.items)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, a.items, a.batch, a.V, a.dim, dt)
tq = {dg.I8: torch.int8, dg.BF16: torch.bfloat16, dg.F16: torch.float16, dg.F32: torch.float32}[dt]
if dt in (dg.BF16, dg.F16):
    q = torch.from_numpy(Q.view(np.int16)).view(tq).cuda()
else:
    q = torch.from_numpy(Q).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, a.batch, a.preset))
torch.cuda.synchronize()
for _ in range(a.iters):
    r = ix.search(q, cls, a.K, want_pass=not a.no_pass)
torch.cuda.synchronize()
print("pass", r[2].tolist()[:4], "top", r[1][0, :3].tolist())
