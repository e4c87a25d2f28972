import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses, library
n, B, K = 200_000, 256, 1000
ix = Index(n, 128, dg.BF16, 1)
ix.generate(dg.DATA_SEED, dg.MODE_GRID, 0, n)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, 128, dg.BF16, dg.MODE_GRID)
q = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, B, "HIGH"))
ids, sc, ps = ix.search(q, cls, K, want_pass=False)
torch.cuda.synchronize()
ws = ix.workspace(B, 1, K).cpu().numpy()
al = lambda x: (x + 255) // 256 * 256
sbuf = 0; scnt = al(sbuf + B * 40960 * 8); thr = al(scnt + B * 4); mbuf = al(thr + B * 8); mcnt = al(mbuf + B * 65536 * 8)
flags = al(mcnt + B * 4)
f = ws[flags:flags + 4 * B].view(np.int32)
mc = ws[mcnt:mcnt + 4 * B].view(np.int32)
sc_ = ws[scnt:scnt + 4 * B].view(np.int32)
th = ws[thr:thr + 8 * B].view(np.uint64)
bad = np.nonzero(f)[0]
print("flagged", len(bad), bad[:20])
print("main counts flagged", mc[bad][:10], "ok", mc[f == 0][:10])
print("sample counts flagged", sc_[bad][:10])
print("thr flagged", [hex(x) for x in th[bad][:4]])
