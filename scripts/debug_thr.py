"""Dump the batched path's per-user thresholds, sample counts and main counts from the workspace."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as dg
from paper_2407_13218_b200 import Index
from paper_2407_13218_b200.linr import Clauses
n, B, K = int(sys.argv[1]), int(sys.argv[2]), 1000
G, SCAP, MCAP = 148, 256, 256
ix = Index(n, 128, dg.BF16, 1)
ix.generate(dg.DATA_SEED, dg.MODE_GRID, 0, n)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, 1, 128, dg.BF16)
q = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).cuda()
cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, B, "HIGH"))
ix.profile(True)
ids, sc, ps = ix.search(q, cls, K, want_pass=False)
torch.cuda.synchronize()
print("profile", ix.profile_read())
ws = ix.workspace(B, 1, K).cpu().numpy()
al = lambda x: (x + 255) // 256 * 256
sbuf = 0; scnt = al(sbuf + B * G * SCAP * 8); thr = al(scnt + B * G * 4); mbuf = al(thr + B * 8)
mcnt = al(mbuf + B * G * MCAP * 8); flags = al(mcnt + B * G * 4)
sc_ = ws[scnt:scnt + 4 * B * G].view(np.int32).reshape(B, G)
print("sample counts per user (sum over CTAs)", sc_.sum(1)[:8], "max region", sc_.max())
T = ws[thr:thr + 8 * B].view(np.uint64)
print("zero thresholds", int((T == 0).sum()), "of", B)
mc = ws[mcnt:mcnt + 4 * B * G].view(np.int32).reshape(B, G)
print("main counts per user", mc.sum(1)[:8], "max region", mc.max())
print("flags", ws[flags:flags + 4 * B].view(np.int32).sum())
