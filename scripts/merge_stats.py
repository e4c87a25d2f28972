"""Emulate the merge's fast path on a real scan workspace: saturation count, survivors, bucket sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses
n = int(sys.argv[1]); preset = sys.argv[2]; K = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
ix = Index(n, 128, dg.BF16, 1)
ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, n)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, 1, 1, 128, dg.BF16)
q = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, 1, preset))
ids, sc, ps = ix.search(q, cls, K)
torch.cuda.synchronize()
ws = ix.workspace(1, 1, K).cpu().numpy()
grid = torch.cuda.get_device_properties(0).multi_processor_count
samp = ws[:grid * 32 * 8].view(np.uint64).reshape(grid, 32)
tot = ws.size
lo = ((grid * 32 * 8 + 255) // 256) * 256
for list_cap in range(256, 40000):
    co = lo + ((grid * list_cap * 8 + 255) // 256) * 256
    po = co + ((grid * 4 + 255) // 256) * 256
    if po + ((grid * 8 + 255) // 256) * 256 == tot:
        break
cnts = ws[co:co + grid * 4].view(np.int32)
sk = np.sort(samp[samp != 0])[::-1]
lb = sk[K - 1]
sat = int(((samp[:, 31] >= lb) & (samp[:, 31] != 0)).sum())
surv = sk[:K]
a = np.bitwise_and.reduce(surv); o = np.bitwise_or.reduce(surv)
hb = int(a ^ o).bit_length() - 1
shift = max(hb - 10, 0)
dig = (surv >> np.uint64(shift)) & np.uint64(2047)
b = np.bincount(dig.astype(np.int64), minlength=2048)
print(f"n={n} {preset}: list_cap {list_cap} cnt med {np.median(cnts)} max {cnts.max()}  saturated CTAs {sat}  hb {hb} max bucket {b.max()} buckets>8: {(b>8).sum()} nonempty {(b>0).sum()}")
