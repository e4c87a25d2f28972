"""Small searches through every kernel of the search path, for compute-sanitizer runs:
    compute-sanitizer --tool {memcheck,racecheck,synccheck} python scripts/sanitize.py [case]
Cases: ws (warp-specialised ring scan + merge), gemv (per-warp scan, f32 + fused merge),
tc (batched tcgen05 sample/threshold/main/finalize/fallback/count), tcv (tcgen05 with V = 8 and
with padded columns), fb (forced fallback)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen as dg  # noqa: E402
import oracle  # noqa: E402
from parity import check, make_index, to_torch  # noqa: E402


def run(dtype, d, n, B, V, K, preset, mode):
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, n, d, dtype, mode)
    ix = make_index(vals, attrs, dtype)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, B, V, d, dtype, mode)
    cls = dg.gen_clauses(dg.QUERY_SEED, B, preset)
    g = ix.search(to_torch(Q, dtype, "cuda"), cls, K)
    torch.cuda.synchronize()
    ref = oracle.search(dtype, vals, attrs, np.ones(n), Q, cls, K)
    check(dtype, vals, attrs, np.ones(n), Q, cls, K, g, ref, True, what="sanitize")


case = sys.argv[1] if len(sys.argv) > 1 else "ws"
if case == "ws":
    run(dg.BF16, 128, 60_000, 1, 1, 500, "HIGH", dg.MODE_GRID)
    os.environ["LINR_WS_CMAX"] = "1280"
    run(dg.I8, 64, 60_000, 1, 1, 1000, "ALL", dg.MODE_DENSE)
elif case == "gemv":
    run(dg.F32, 64, 40_000, 2, 1, 300, "HIGH4", dg.MODE_GRID)
    os.environ["LINR_FUSE_MERGE"] = "1"
    run(dg.F32, 64, 40_000, 1, 1, 300, "ALL", dg.MODE_GRID)
elif case == "tc":
    run(dg.BF16, 128, 40_000, 32, 1, 200, "HIGH", dg.MODE_GRID)
elif case == "tcv":
    run(dg.BF16, 128, 30_000, 4, 8, 300, "HIGH", dg.MODE_GRID)
    run(dg.I8, 64, 30_000, 12, 1, 200, "LOW", dg.MODE_DENSE)
elif case == "fb":
    os.environ["LINR_TC_MAIN_CAP"] = "2"
    run(dg.I8, 64, 30_000, 16, 1, 300, "HIGH", dg.MODE_DENSE)
print("sanitize case", case, "ok")
