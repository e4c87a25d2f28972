"""Check the folded threshold K-step: accumulator of tile 0 (CTA 0, chunk 0) + t_eff == dot product."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses, library
n, B, K = 200_000, int(sys.argv[1]) if len(sys.argv) > 1 else 16, 1000
dt = dg.BF16
ix = Index(n, 128, dt, 1)
ix.generate(dg.DATA_SEED, dg.MODE_GRID, 0, n)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, 128, dt)
q = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, B, "HIGH"))
ix.search(q, cls, K, want_pass=False); torch.cuda.synchronize()
L = library(); L.linr_debug_timers(1)
ix.search(q, cls, K, want_pass=False); torch.cuda.synchronize()
buf = np.zeros(8192, np.uint64); L.linr_debug_read(buf.ctypes.data, 8192); L.linr_debug_timers(0)
d32 = buf[1024:].view(np.uint32)
acc = d32[:128 * 32].view(np.float32).reshape(128, 32)
cq = d32[128 * 32:128 * 32 + 32].view(np.float32)
vals, _ = dg.gen_items(dg.DATA_SEED, 0, 128, 128, dt, dg.MODE_GRID)
def tof(a):
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)
Xf = tof(vals.view(np.uint16)) if vals.dtype != np.float64 else vals
Qf = tof(Q.view(np.uint16).reshape(B, 128))
sc = Xf @ Qf.T
print("cq", cq[:B])
rec = acc[:, :B] + cq[:B]
err = np.abs(rec - sc)
print("max |acc+cq - s|", err.max(), "at", np.unravel_index(err.argmax(), err.shape))
bad = np.argwhere(err > 1e-3)
print("bad count", len(bad), bad[:20].tolist())
for r, c in bad[:6]:
    print(r, c, "acc", acc[r, c], "cq", cq[c], "s", sc[r, c], "acc - s", acc[r, c] - sc[r, c])
