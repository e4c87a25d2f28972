"""Debug: inspect the scan workspace (per-CTA samples/lists) for one search vs host-computed keys."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen as dg, oracle
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity import make_index, to_torch

n, d, K, preset = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dg.I8, dg.MODE_DENSE)
ix = make_index(vals, attrs, dg.I8)
Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, 1, 1, d, dg.I8)
cls = dg.gen_clauses(dg.QUERY_SEED, 1, preset)
ids, sc, ps = ix.search(to_torch(Q, dg.I8, "cuda"), cls, K)
torch.cuda.synchronize()
ws = ix.workspace(1, 1, K).cpu().numpy()
grid = torch.cuda.get_device_properties(0).multi_processor_count
# host keys
mask, cnt = oracle.filter_mask(attrs, np.ones(n), cls[0])
s = oracle.scores(dg.I8, vals, Q[0, 0])
def key(score, gid):
    u = int(np.float32(score).view(np.uint32))
    if (u << 1) & 0xFFFFFFFF == 0: u = 0
    o = (~u) & 0xFFFFFFFF if u & 0x80000000 else (u | 0x80000000)
    return (int(o) << 32) | (0xFFFFFFFF - gid)
allkeys = {key(s[i], int(i)) for i in np.nonzero(mask)[0]}
samp = ws[:grid * 32 * 8].view(np.uint64).reshape(grid, 32)
list_off = ((grid * 32 * 8 + 255) // 256) * 256
# find list_cap from total size: layout samp | list | cnt | pass
tot = ws.size
# brute: try list_cap candidates
for list_cap in range(256, 40000):
    lo = list_off; co = lo + ((grid * list_cap * 8 + 255) // 256) * 256
    po = co + ((grid * 4 + 255) // 256) * 256
    end = po + ((grid * 8 + 255) // 256) * 256
    if end == tot:
        break
lists = ws[lo:lo + grid * list_cap * 8].view(np.uint64).reshape(grid, list_cap)
cnts = ws[co:co + grid * 4].view(np.int32)
print("list_cap", list_cap, "sum cnt", cnts.sum(), "pass", cnt)
got = set()
bad = 0
for c in range(grid):
    L = lists[c, :cnts[c]]
    got |= set(int(x) for x in L)
    top = sorted(L.tolist(), reverse=True)[:32]
    sm = [int(x) for x in samp[c] if x != 0]
    if top != sm:
        bad += 1
        if bad < 4:
            print("CTA", c, "sample mismatch: cnt", cnts[c], "sample", [hex(x) for x in sm[:4]], "top", [hex(x) for x in top[:4]])
print("CTAs with bad samples:", bad)
print("keys missing from lists:", len(allkeys - got), "extra:", len(got - allkeys))
np.savez("gpurun_out/debug_case.npz", samp=samp, lists=lists, cnts=cnts, ids=ids.cpu().numpy(), sc=sc.cpu().numpy(),
         allkeys=np.array(sorted(allkeys, reverse=True), dtype=np.uint64))
