"""Seeded synthetic-input generator shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no clause evaluation, no dot products,
no top-K). It only turns (seed, stream, row, col) counters into item embeddings, item
attribute bitmasks, query vectors and query clause lists, following the recipe in
DESIGN.md §"Input recipe" (SURVEY.md §8(d) "Synthetic inputs").

The same counter-based generator is implemented a second time, independently, in CUDA
(`gen_rows_kernel` in `paper_2407_13218_b200/csrc/index_kernels.cu`, used only to fill 1B-row indexes in place on the
device); `tests/test_datagen.py` checks the two produce identical bytes. Oracle inputs
always come from THIS module, never from the CUDA one.

Workload shape follows the paper's benchmark (§5.3 "Model Inference
Benchmarking"): one attribute per clause per item, stored as 64-bit integers; d=128 fp16
(here f32/f16/bf16/int8); a high-pass (~11%) and a low-pass clause mix.
"""
from __future__ import annotations

import numpy as np

U64 = np.uint64
MASK64 = (1 << 64) - 1

DATA_SEED = 0x2407
QUERY_SEED = 0x13218
UPDATE_SEED = 0x4429

# counter streams
S_CLUSTER, S_CENTER, S_NOISE, S_ATTR, S_QROW, S_QNOISE, S_QCLAUSE, S_OPORP = 1, 2, 3, 4, 5, 6, 7, 8
S_IDL, S_IDVAL, S_QIDL = 9, 10, 11
S_SCORER = 12
SCORER_SEED = 0x4318   # PAPER.md P:4318 (Hadamard MLP)
ID_SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)   # padding of ID-list rows
OPORP_SEED = 0x4294   # PAPER.md P:4294 (Sign-OPORP)

N_CLUSTERS = 1024

# dtype codes (same numbering as include/linr.h; restated here, not imported)
F32, F16, BF16, I8 = 0, 1, 2, 3
DTYPE_NAMES = {"f32": F32, "f16": F16, "bf16": BF16, "i8": I8, "int8": I8}
ELEM_BYTES = {F32: 4, F16: 2, BF16: 2, I8: 1}

# value modes
MODE_GRID = 0   # x = k * 2^-7, |k| <= 127: every fp32 partial sum is exact (SURVEY §8(c) pins)
MODE_DENSE = 1  # full-mantissa uniform mixture, rounded to the storage dtype

# attribute word 0 field layout: geo bits 0-23, company 24-39, title 40-55, level 56-63
GEO_BITS, COMPANY_BITS, TITLE_BITS, LEVEL_BITS = 24, 16, 16, 8
GEO_OFF, COMPANY_OFF, TITLE_OFF, LEVEL_OFF = 0, 24, 40, 56

PRESETS = ("ALL", "HIGH", "HIGH4", "LOW")

_G = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_SC = 0xD6E8FEB86659FD93


def sm64(z):
    """SplitMix64 finaliser on a uint64 ndarray (wrapping arithmetic)."""
    z = np.asarray(z, dtype=U64)
    with np.errstate(over="ignore"):
        z = z + U64(_G)
        z = (z ^ (z >> U64(30))) * U64(_M1)
        z = (z ^ (z >> U64(27))) * U64(_M2)
    return z ^ (z >> U64(31))


def sm64_int(z: int) -> int:
    z = (z + _G) & MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def stream_base(seed: int, stream: int) -> int:
    return sm64_int((seed ^ ((stream * _SC) & MASK64)) & MASK64)


def h1(seed: int, stream: int, a):
    """hash of one counter: sm64(base(seed,stream) ^ a)."""
    return sm64(U64(stream_base(seed, stream)) ^ np.asarray(a, dtype=U64))


def h2(seed: int, stream: int, a, b):
    """hash of two counters: sm64(h1(a) ^ (b * golden))."""
    with np.errstate(over="ignore"):
        bb = np.asarray(b, dtype=U64) * U64(_G)
    return sm64(h1(seed, stream, a) ^ bb)


# ---------------------------------------------------------------- rounding helpers
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (u >> np.uint32(16)) & np.uint32(1)
    r += np.uint32(0x7FFF)
    r += u                      # finite inputs: no uint32 overflow (max 0xFF7FFFFF + 0x8000)
    r >>= np.uint32(16)
    return r.astype(np.uint16)


def f32_to_f16_bits(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32).astype(np.float16).view(np.uint16)


def bits_to_f32(bits: np.ndarray, dtype: int) -> np.ndarray:
    """Exact widening of stored values to fp32 (for building queries from item rows)."""
    if dtype == F32:
        return np.asarray(bits, dtype=np.float32)
    if dtype == F16:
        return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float32)
    if dtype == BF16:
        return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
    return np.asarray(bits, dtype=np.float32)


def _store(x32: np.ndarray, dtype: int) -> np.ndarray:
    if dtype == F32:
        return x32.astype(np.float32)
    if dtype == F16:
        return f32_to_f16_bits(x32)
    if dtype == BF16:
        return f32_to_bf16_bits(x32)
    raise ValueError(dtype)


# ---------------------------------------------------------------- items
_CENTER_CACHE: dict = {}


def _center_table(seed: int, d: int, kind: str) -> np.ndarray:
    """Per-cluster centers [N_CLUSTERS][d]: int16 codes in [-64,63] ('i8') or exact fp32 in [-0.5,0.5) ('f')."""
    key = (seed, d, kind)
    t = _CENTER_CACHE.get(key)
    if t is None:
        cl = np.arange(N_CLUSTERS, dtype=U64)
        if kind == "i8":
            nb = (d + 7) // 8
            h = h2(seed, S_CENTER, cl[:, None], np.arange(nb, dtype=U64)[None, :])      # [C, nb]
            t = (h.view(np.uint8).reshape(N_CLUSTERS, nb * 8)[:, :d] & np.uint8(0x7F)).astype(np.int16) - 64
        else:
            nc = (d + 1) // 2
            h = h2(seed, S_CENTER, cl[:, None], np.arange(nc, dtype=U64)[None, :])      # [C, nc]
            c24 = h.view(np.uint32).reshape(N_CLUSTERS, nc * 2)[:, :d] & np.uint32(0xFFFFFF)
            t = c24.astype(np.float32) * np.float32(2.0 ** -24) - np.float32(0.5)
        _CENTER_CACHE[key] = t
    return t


def _clusters(seed: int, rows: np.ndarray) -> np.ndarray:
    return (h1(seed, S_CLUSTER, rows) & U64(N_CLUSTERS - 1)).astype(np.int64)


def _int8_values(seed: int, rows: np.ndarray, d: int) -> np.ndarray:
    """int8 codes x = center[cluster(row)] + noise(row), center in [-64,63], noise in [-32,31].
    Byte k of a 64-bit hash feeds element 8*blk + k (little-endian byte order)."""
    rows = np.asarray(rows, dtype=U64)
    cen = _center_table(seed, d, "i8")[_clusters(seed, rows)]                    # [n, d] int16
    nb = (d + 7) // 8
    noi_h = h2(seed, S_NOISE, rows[:, None], np.arange(nb, dtype=U64)[None, :])  # [n, nb]
    noi = (noi_h.view(np.uint8).reshape(len(rows), nb * 8)[:, :d] & np.uint8(0x3F)).astype(np.int16) - 32
    return np.clip(cen + noi, -127, 127).astype(np.int8)


def _dense_values(seed: int, rows: np.ndarray, d: int) -> np.ndarray:
    """fp32 values fl32(c + n): c = u24*2^-24 - 0.5 per (cluster, j) from the low 24 bits of 32-bit
    half (j % 2) of h2(center, cluster, j//2); n = u16*2^-17 - 0.25 per (row, j) from 16-bit
    quarter (j % 4) of h2(noise, row, j//4)."""
    rows = np.asarray(rows, dtype=U64)
    c = _center_table(seed, d, "f")[_clusters(seed, rows)]                         # [n, d] fp32
    nn = (d + 3) // 4
    noi_h = h2(seed, S_NOISE, rows[:, None], np.arange(nn, dtype=U64)[None, :])   # [n, nn]
    n16 = noi_h.view(np.uint16).reshape(len(rows), nn * 4)[:, :d]
    n = n16.astype(np.float32) * np.float32(2.0 ** -17) - np.float32(0.25)
    return (c + n).astype(np.float32)


def item_values(seed: int, rows, d: int, dtype: int, mode: int) -> np.ndarray:
    """Embedding rows in storage representation: float32 (F32), uint16 bits (F16/BF16), int8 (I8)."""
    rows = np.asarray(rows, dtype=np.int64)
    if dtype == I8:
        return _int8_values(seed, rows, d)
    if mode == MODE_GRID:
        x = _int8_values(seed, rows, d).astype(np.float32) * np.float32(2.0 ** -7)
    else:
        x = _dense_values(seed, rows, d)
    return _store(x, dtype)


def item_attrs(seed: int, rows, W: int) -> np.ndarray:
    """[n][W] uint64 attribute words. Word 0: one bit per field (geo/company/title/level)."""
    rows = np.asarray(rows, dtype=U64)
    out = np.empty((len(rows), W), dtype=U64)
    h = h2(seed, S_ATTR, rows, U64(0))
    geo = ((h & U64(0xFFFF)) * U64(GEO_BITS)) >> U64(16)
    com = (((h >> U64(16)) & U64(0xFFFF)) * U64(COMPANY_BITS)) >> U64(16)
    tit = (((h >> U64(32)) & U64(0xFFFF)) * U64(TITLE_BITS)) >> U64(16)
    lev = (((h >> U64(48)) & U64(0xFFFF)) * U64(LEVEL_BITS)) >> U64(16)
    one = U64(1)
    out[:, 0] = (one << (geo + U64(GEO_OFF))) | (one << (com + U64(COMPANY_OFF))) | \
                (one << (tit + U64(TITLE_OFF))) | (one << (lev + U64(LEVEL_OFF)))
    for w in range(1, W):
        out[:, w] = h2(seed, S_ATTR, rows, U64(w))
    return out


def gen_items(seed: int, row_begin: int, n: int, d: int, dtype: int, mode: int = MODE_DENSE, W: int = 1,
              threads: int = 0):
    """Rows [row_begin, row_begin+n): (values [n][d] storage repr, attrs [n][W] uint64).
    Large requests are split into row chunks on a thread pool (numpy releases the GIL); the
    result is identical because every value is a function of its (row, col) counter."""
    chunk = 1 << 18
    if n <= chunk:
        rows = np.arange(row_begin, row_begin + n, dtype=np.int64)
        return item_values(seed, rows, d, dtype, mode), item_attrs(seed, rows, W)
    import concurrent.futures as cf
    import os
    vdt = {F32: np.float32, F16: np.uint16, BF16: np.uint16, I8: np.int8}[dtype]
    vals = np.empty((n, d), dtype=vdt)
    attrs = np.empty((n, W), dtype=U64)
    _center_table(seed, d, "i8" if (dtype == I8 or mode == MODE_GRID) else "f")

    def work(a):
        b = min(n, a + chunk)
        rows = np.arange(row_begin + a, row_begin + b, dtype=np.int64)
        vals[a:b] = item_values(seed, rows, d, dtype, mode)
        attrs[a:b] = item_attrs(seed, rows, W)

    with cf.ThreadPoolExecutor(threads or min(32, os.cpu_count() or 4)) as ex:
        list(ex.map(work, range(0, n, chunk)))
    return vals, attrs


# ---------------------------------------------------------------- queries
def query_source_rows(qseed: int, n_items: int, B: int, V: int) -> np.ndarray:
    b = np.arange(B, dtype=U64)[:, None]
    v = np.arange(V, dtype=U64)[None, :]
    return (h2(qseed, S_QROW, b, v) % U64(max(n_items, 1))).astype(np.int64)   # [B, V]


def gen_queries(qseed: int, dseed: int, n_items: int, B: int, V: int, d: int, dtype: int,
                mode: int = MODE_DENSE) -> np.ndarray:
    """[B][V][d] query vectors: a random item's row plus noise, in the index dtype."""
    src = query_source_rows(qseed, n_items, B, V).reshape(-1)
    ctr = (np.arange(B, dtype=U64)[:, None] * U64(16) + np.arange(V, dtype=U64)[None, :]).reshape(-1)
    if dtype == I8 or mode == MODE_GRID:
        base = _int8_values(dseed, src, d).astype(np.int16)
        nb = (d + 7) // 8
        hq = h2(qseed, S_QNOISE, ctr[:, None], np.arange(nb, dtype=U64)[None, :])
        nz = (hq.view(np.uint8).reshape(len(src), nb * 8)[:, :d] & np.uint8(0xF)).astype(np.int16) - 8
        q8 = np.clip(base + nz, -127, 127).astype(np.int8)
        if dtype == I8:
            out = q8
        else:
            out = _store(q8.astype(np.float32) * np.float32(2.0 ** -7), dtype)
    else:
        base = bits_to_f32(item_values(dseed, src, d, dtype, mode), dtype)
        nn = (d + 3) // 4
        hq = h2(qseed, S_QNOISE, ctr[:, None], np.arange(nn, dtype=U64)[None, :])
        n16 = hq.view(np.uint16).reshape(len(src), nn * 4)[:, :d]
        nz = n16.astype(np.float32) * np.float32(2.0 ** -18) - np.float32(0.125)
        out = _store((base + nz).astype(np.float32), dtype)
    return out.reshape(B, V, d)


# ---------------------------------------------------------------- clauses
def _bit(off: int, v: int) -> int:
    return 1 << (off + v)


def gen_clauses(qseed: int, B: int, preset: str):
    """Per-query clause lists [(mask, word, reverse), ...] for a pass-rate preset.

    ALL   : level Match on all 8 level bits                               -> pass 1
    HIGH  : geo Match 3/24, company Reverse 1/16                          -> ~11.7% (paper high-pass ~11%)
    HIGH4 : geo Match 6/24, company Rev 1/16, title Match 8/16, level Rev 1/8 -> ~10.25% (config c1 "4 clauses")
    LOW   : geo Match 1/24, company Rev 1/16, title Match 1/16             -> ~0.24% (paper low-pass)
    """
    preset = preset.upper()
    out = []
    for b in range(B):
        hq = int(h2(qseed, S_QCLAUSE, U64(b), U64(0)))
        g0, c0, t0, l0 = hq % 24, (hq >> 8) % 16, (hq >> 16) % 16, (hq >> 24) % 8
        if preset == "ALL":
            cl = [(0xFF << LEVEL_OFF, 0, 0)]
        elif preset == "HIGH":
            geo = sum(_bit(GEO_OFF, (g0 + 8 * k) % 24) for k in range(3))
            cl = [(geo, 0, 0), (_bit(COMPANY_OFF, c0), 0, 1)]
        elif preset == "HIGH4":
            geo = sum(_bit(GEO_OFF, (g0 + 4 * k) % 24) for k in range(6))
            tit = sum(_bit(TITLE_OFF, (t0 + 2 * k) % 16) for k in range(8))
            cl = [(geo, 0, 0), (_bit(COMPANY_OFF, c0), 0, 1), (tit, 0, 0), (_bit(LEVEL_OFF, l0), 0, 1)]
        elif preset == "LOW":
            cl = [(_bit(GEO_OFF, g0), 0, 0), (_bit(COMPANY_OFF, c0), 0, 1), (_bit(TITLE_OFF, t0), 0, 0)]
        else:
            raise ValueError(preset)
        out.append(cl)
    return out


def field_value_probs(nvals: int) -> np.ndarray:
    """Exact probability of each field value under the multiply-shift map of a uniform u16."""
    v = (np.arange(65536, dtype=np.uint64) * np.uint64(nvals)) >> np.uint64(16)
    return np.bincount(v.astype(np.int64), minlength=nvals) / 65536.0


def flatten_clauses(clauses):
    """CSR form: (masks u64[n], words u8[n], reverse u8[n], offsets i32[B+1])."""
    off = [0]
    m, w, r = [], [], []
    for cl in clauses:
        for (mask, word, rev) in cl:
            m.append(mask); w.append(word); r.append(rev)
        off.append(len(m))
    return (np.array(m, dtype=np.uint64), np.array(w, dtype=np.uint8),
            np.array(r, dtype=np.uint8), np.array(off, dtype=np.int32))


# ---------------------------------------------------------------- Sign-OPORP parameters
def oporp_params(seed: int, d: int, k: int):
    """The random draws of Sign-OPORP (one permutation, one sign vector), as the
    (src[L], sign[L]) arrays both the oracle and the library take (reading R25):
      k <= d: the vector zero-padded to L = k*ceil(d/k), one uniform permutation of
              the L positions: bins of ceil(d/k) entries (k = d: one coordinate per bit, the paper's
              "1-bit embedding of the same dimension");
      k >  d: padding would leave k-d constant bits, so the vector is replicated k times (L = k*d)
              and one uniform permutation of the L positions is taken: every bin sums d entries
              (a sign random projection per bit).
    src[p] = coordinate at position p (-1 = zero padding), sign[p] = +-1. Fisher-Yates over
    SplitMix64 counters (seed, S_OPORP, p); signs from (seed, S_OPORP + 16, p)."""
    if k % 64 or k < 64 or d < 1:
        raise ValueError("k must be a positive multiple of 64")
    if k <= d:
        b = -(-d // k)
        L = k * b
        base = np.concatenate([np.arange(d, dtype=np.int64), np.full(L - d, -1, np.int64)])
    else:
        L = k * d
        base = np.tile(np.arange(d, dtype=np.int64), k)
    r = h1(seed, S_OPORP, np.arange(L, dtype=U64))
    perm = base.copy()
    for i in range(L - 1, 0, -1):   # Fisher-Yates: swap i with j = r[i] mod (i+1)
        j = int(r[i] % U64(i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    sgn = np.where((h1(seed, S_OPORP + 16, np.arange(L, dtype=U64)) & U64(1)) == U64(1), 1, -1).astype(np.int8)
    return perm.astype(np.int32), sgn


# ---------------------------------------------------------------- ID-list attributes
def id_of(seed: int, values) -> np.ndarray:
    """64-bit attribute id of an attribute value (attributes "converted to 64-bit integers");
    never the padding sentinel."""
    h = h1(seed, S_IDVAL, np.asarray(values, dtype=U64))
    return np.where(h == ID_SENTINEL, U64(0), h)


def gen_idlists(seed: int, row_begin: int, n: int, slot: int, A: int, universe: int, raw: bool = False):
    """One ID-list slot for rows [row_begin, row_begin+n): ids [n][A] uint64 (each row's distinct ids
    sorted ascending, padded with ID_SENTINEL) and counts [n] uint8 in [1, A]. Row r draws
    1 + h % A values uniformly from [0, universe); raw=True keeps the values themselves as ids."""
    rows = np.arange(row_begin, row_begin + n, dtype=U64)
    hc = h2(seed, S_IDL, rows, U64(slot * 64))
    want = (hc % U64(A)).astype(np.int64) + 1
    vals = np.stack([(h2(seed, S_IDL, rows, U64(slot * 64 + 1 + a)) % U64(universe)) for a in range(A)], axis=1)
    ids = vals.astype(U64) if raw else id_of(seed, vals)
    out = np.full((n, A), ID_SENTINEL, dtype=U64)
    cnt = np.zeros(n, dtype=np.uint8)
    for i in range(n):
        u = np.unique(ids[i, :want[i]])   # sorted, distinct
        out[i, :len(u)] = u
        cnt[i] = len(u)
    return out, cnt


def gen_id_clauses(qseed: int, dseed: int, B: int, slot: int, A: int, universe: int, nq: int, n_items: int,
                   reverse: int = 0, raw: bool = False):
    """Per query one ID-list clause on `slot`: the first value of a random item's list plus nq-1 random
    values, as sorted distinct 64-bit ids. Returns [[(slot, reverse, ids)], ...]."""
    out = []
    for b in range(B):
        src = int(h2(qseed, S_QIDL, U64(b), U64(slot)) % U64(max(1, n_items)))
        first = int(h2(dseed, S_IDL, U64(src), U64(slot * 64 + 1)) % U64(universe))
        others = [int(h2(qseed, S_QIDL, U64(b), U64(slot * 64 + 1 + j)) % U64(universe)) for j in range(nq - 1)]
        vals = np.array([first] + others, dtype=U64)
        ids = vals if raw else id_of(dseed, vals)
        out.append([(slot, reverse, np.unique(ids))])
    return out


# ---------------------------------------------------------------- learned-scorer weights (synthetic)
def _uniform_weights(seed: int, tag: int, shape, scale: float) -> np.ndarray:
    """float32 weights uniform in [-scale, scale), multiples of scale * 2^-11 (counter-based)."""
    n = int(np.prod(shape))
    h = h2(seed, S_SCORER, U64(tag), np.arange(n, dtype=U64))
    u = ((h >> U64(53)).astype(np.int64) - 1024).astype(np.float32) * np.float32(scale / 1024.0)
    return u.reshape(shape)


def scorer_weights(seed: int, kind: str, d: int, F: int = 50, H: int = 10, K: int = 4, dc: int = 32, G: int = 16):
    """Synthetic weights of a learned scorer (§3.3; training is out of scope):
    'hadamard' -- member/item MLP width F (Table 1: [50]), head [H, 1] (Table 1: [10, 1]);
    'mol'      -- K components of width dc (user/item projections), gate hidden width G.
    Fan-in-scaled uniform values so scores stay O(1)."""
    s_in = 1.0 / np.sqrt(d)
    if kind == "hadamard":
        return {"kind": 1, "F": F, "H": H,
                "Wm": _uniform_weights(seed, 1, (F, d), s_in), "bm": _uniform_weights(seed, 2, (F,), 0.1),
                "Wi": _uniform_weights(seed, 3, (F, d), s_in), "bi": _uniform_weights(seed, 4, (F,), 0.1),
                "W1": _uniform_weights(seed, 5, (H, F), 1.0 / np.sqrt(F)), "b1": _uniform_weights(seed, 6, (H,), 0.1),
                "w2": _uniform_weights(seed, 7, (H,), 1.0 / np.sqrt(H)), "b2": _uniform_weights(seed, 8, (1,), 0.1)}
    if kind == "mol":
        return {"kind": 2, "K": K, "dc": dc, "G": G,
                "Fk": _uniform_weights(seed, 11, (K * dc, d), s_in), "Gk": _uniform_weights(seed, 12, (K * dc, d), s_in),
                "Wgu": _uniform_weights(seed, 13, (G, d), s_in), "Wgx": _uniform_weights(seed, 14, (G, d), s_in),
                "bg": _uniform_weights(seed, 15, (G,), 0.1), "Wo": _uniform_weights(seed, 16, (K, G), 1.0 / np.sqrt(G)),
                "bo": _uniform_weights(seed, 17, (K,), 0.1)}
    raise ValueError(kind)
