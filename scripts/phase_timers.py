"""Read the library's device phase timers for one search of the bench workload."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses, library

ap = argparse.ArgumentParser()
ap.add_argument("--items", type=int, default=10_000_000)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--preset", default="HIGH")
ap.add_argument("--K", type=int, default=1000)
ap.add_argument("--V", type=int, default=1)
a = ap.parse_args()
dt = dg.DTYPE_NAMES[a.dtype]
ix = Index(a.items, a.dim, dt, 1)
ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, a.items)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, a.items, 1, a.V, a.dim, dt)
tq = {dg.I8: torch.int8, dg.BF16: torch.bfloat16, dg.F16: torch.float16, dg.F32: torch.float32}[dt]
q = torch.from_numpy(Q.view(np.int16) if dt in (dg.BF16, dg.F16) else Q).view(tq).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, 1, a.preset))
L = library()
for _ in range(3):
    ix.search(q, cls, a.K)
torch.cuda.synchronize()
L.linr_debug_timers(1)
ix.search(q, cls, a.K)
torch.cuda.synchronize()
buf = np.zeros(8192, np.uint64)
L.linr_debug_read(buf.ctypes.data, 8192)
L.linr_debug_timers(0)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
sc = buf[: nsm * 8].reshape(nsm, 8).astype(np.int64)
used = sc[:, 0] > 0
sc = sc[used]
t0 = sc[:, 0].min()
st = (sc[:, 0] - t0) / 1e3
rel = lambda k: (sc[:, k] - sc[:, 0]) / 1e3
def q(x):
    return f"min {x.min():7.2f} med {np.median(x):7.2f} max {x.max():7.2f}"
print(f"scan CTAs {used.sum()}: start spread {st.max():.2f} us")
if (sc[:, 4] > 0).all():
    print(f"  first producer done  {q(rel(4))}")
    print(f"  last producer done   {q(rel(5))}")
print(f"  scan loop end        {q(rel(1))}")
print(f"  sample selected      {q(rel(2))}")
print(f"  sample written       {q(rel(6))}")
print(f"  tail end             {q(rel(3))}")
print(f"  absolute tail end (from first start) max {((sc[:, 3] - t0) / 1e3).max():.2f} us")
print(f"  compactions per CTA: min {sc[:,7].min()} med {np.median(sc[:,7])} max {sc[:,7].max()}")
m = buf[4096:4104].astype(np.int64)
if m[0] > 0:
    mr = (m[:7] - t0) / 1e3
    print(f"merge: start {mr[0]:.2f}  gather-done {mr[1]-mr[0]:.2f}  lb {mr[2]-mr[1]:.2f}  prune {mr[3]-mr[2]:.2f}  select {mr[4]-mr[3]:.2f}  sort {mr[5]-mr[4]:.2f}  out {mr[6]-mr[5]:.2f}  n={m[7]}  (us)")
