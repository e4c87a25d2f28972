import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses, library
n, B, K = 10_000_000, int(sys.argv[1]), 1000
ix = Index(n, 128, dg.BF16, 1)
ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, n)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, 128, dg.BF16)
q = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, B, "HIGH"))
ix.search(q, cls, K, want_pass=False); torch.cuda.synchronize()
L = library(); L.linr_debug_timers(1)
ix.search(q, cls, K, want_pass=False); torch.cuda.synchronize()
buf = np.zeros(8192, np.uint64); L.linr_debug_read(buf.ctypes.data, 8192); L.linr_debug_timers(0)
t = buf[:256].reshape(64, 4).astype(np.int64)
t0 = t[0, 0]
for i in range(0, 24):
    print(i, ((t[i] - t0) / 1000).round(2).tolist())
d = np.diff(t[:, 3]) / 1000
print("epilogue-end spacing us: median", np.median(d[5:60]))
