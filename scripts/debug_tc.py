"""Inspect the batched (tcgen05) search workspace: sample counts, thresholds, main counts, flags."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses
n = int(sys.argv[1]); B = int(sys.argv[2]); K = 1000
ix = Index(n, 128, dg.BF16, 1)
ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, n)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, 128, dg.BF16)
q = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, B, "HIGH"))
import time
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    ids, sc, ps = ix.search(q, cls, K, want_pass=False)
    torch.cuda.synchronize(); print("search s", time.time() - t0)
ws = ix.workspace(B, 1, K).cpu().numpy()
al = lambda x: (x + 255) // 256 * 256
sbuf = 0; scnt = al(sbuf + B * 40960 * 8); thr = al(scnt + B * 4); mbuf = al(thr + B * 8); mcnt = al(mbuf + B * 65536 * 8)
flags = al(mcnt + B * 4)
print("sample counts", ws[scnt:scnt + 4 * B].view(np.int32)[:8])
print("thr", [hex(x) for x in ws[thr:thr + 8 * B].view(np.uint64)[:4]])
print("main counts", ws[mcnt:mcnt + 4 * B].view(np.int32)[:8])
print("flags", ws[flags:flags + 4 * B].view(np.int32)[:8])
