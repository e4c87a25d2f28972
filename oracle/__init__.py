"""CPU oracle for the LiNR pre-filtered top-K scan — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference legs) may
import this package. The product path (paper_2407_13218_b200) never imports it and shares no
code with it. See linr_oracle.cpp for the definition and the PAPER.md passages it follows.

oporp_oracle.cpp adds the quantised path (§3.2, Fig. 3): Sign-OPORP encoding, matched
bits, the code search (any K, incl. huge K) and the V3 two-stage search.

Parity status: every function is pinned in tests/test_oracle.py against values fixed by the
paper's semantics and by mathematics (hand-worked example, closed forms, brute force,
invariants). No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "linr_oracle.cpp")
_SRCS = [_SRC, os.path.join(_HERE, "oporp_oracle.cpp"), os.path.join(_HERE, "scorer_oracle.cpp")]
_LIB = os.path.join(_HERE, "liblinr_oracle.so")
_lib = None

F32, F16, BF16, I8 = 0, 1, 2, 3

CLAUSE_DTYPE = np.dtype([("mask", "<u8"), ("word", "u1"), ("reverse", "u1"), ("pad", "u1", 6)])


def build(force: bool = False) -> str:
    """Compile the oracle with plain g++ (no intrinsics, no BLAS)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", tmp, *_SRCS])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_widen.argtypes = [ctypes.c_int, ctypes.c_uint32]
        L.oracle_widen.restype = ctypes.c_double
        L.oracle_filter.argtypes = [P, ctypes.c_int, ctypes.c_int64, P, P, ctypes.c_int, P]
        L.oracle_filter.restype = ctypes.c_int64
        L.oracle_scores.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, P, P, P]
        L.oracle_scores.restype = None
        L.oracle_search.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, P,
                                    P, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int,
                                    P, P, ctypes.c_int, P, P, P]
        L.oracle_search.restype = ctypes.c_int
        L.oracle_merge.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P,
                                   ctypes.c_int, P, P, P]
        L.oracle_merge.restype = ctypes.c_int
        I, I64 = ctypes.c_int, ctypes.c_int64
        L.oracle_oporp_encode.argtypes = [I, I, I64, P, I, I, P, P, P]
        L.oracle_oporp_encode.restype = I
        L.oracle_matched_bits.argtypes = [I, I64, P, P, P]
        L.oracle_matched_bits.restype = I
        L.oracle_code_search.argtypes = [I, I, I64, I64, P, P, I, P, P, I, I, P, P, I64, I, I, P, P, P, P, P]
        L.oracle_code_search.restype = I
        L.oracle_search_v3.argtypes = [I, I, I64, I64, P, P, I, P, P, I, I, P, P, I, ctypes.c_double, I, I, P, P,
                                       P, P, P, P]
        L.oracle_search_v3.restype = I
        L.oracle_search_idc.argtypes = [I, I, I64, I64, P, P, I, P, I, P, P, P, P, I, I, P, P, P, P, I, P, P, P]
        L.oracle_search_idc.restype = I
        L.oracle_scorer_score.argtypes = [P, I, I, P, I64, P, I64]
        L.oracle_scorer_score.restype = ctypes.c_double
        L.oracle_search_scored.argtypes = [P, I, I, I64, I64, P, P, I, P, P, I, P, P, I, P, P, P]
        L.oracle_search_scored.restype = I
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def clause_array(clauses_flat):
    """list of (mask, word, reverse) -> structured array matching the 16-byte clause record."""
    arr = np.zeros(len(clauses_flat), dtype=CLAUSE_DTYPE)
    for i, (m, w, r) in enumerate(clauses_flat):
        arr[i]["mask"] = m
        arr[i]["word"] = w
        arr[i]["reverse"] = r
    return arr


def csr(clauses):
    flat, off = [], [0]
    for cl in clauses:
        flat.extend(cl)
        off.append(len(flat))
    return clause_array(flat), np.array(off, dtype=np.int32)


def widen(dtype: int, bits: int) -> float:
    return lib().oracle_widen(dtype, bits)


def filter_mask(attrs, live, clauses_one):
    attrs = np.ascontiguousarray(attrs, dtype=np.uint64)
    n, W = attrs.shape
    live = np.ascontiguousarray(live, dtype=np.uint8)
    ca = clause_array(clauses_one)
    out = np.zeros(n, dtype=np.uint8)
    cnt = lib().oracle_filter(_p(attrs), W, n, _p(live), _p(ca), len(ca), _p(out))
    return out.astype(bool), int(cnt)


def scores(dtype, emb, q):
    emb = np.ascontiguousarray(emb)
    q = np.ascontiguousarray(q)
    n, d = emb.shape
    out = np.zeros(n, dtype=np.float64)
    lib().oracle_scores(dtype, d, n, _p(emb), _p(q), _p(out))
    return out


def search(dtype, emb, attrs, live, queries, clauses, K, row0=0):
    """Oracle top-K. emb [n][d] storage repr; attrs [n][W]; live [n]; queries [B][V][d] or [B][d].

    Returns (ids [B][K] int64, scores [B][K] float64, pass [B] int64).
    """
    emb = np.ascontiguousarray(emb)
    attrs = np.ascontiguousarray(attrs, dtype=np.uint64)
    n, d = emb.shape if emb.ndim == 2 else (0, queries.shape[-1])
    if n == 0:
        emb = np.zeros((1, d), dtype=queries.dtype)
        attrs = np.zeros((1, max(1, attrs.shape[1] if attrs.ndim == 2 else 1)), dtype=np.uint64)
    W = attrs.shape[1]
    live = np.ascontiguousarray(live, dtype=np.uint8) if n else np.zeros(1, np.uint8)
    q = np.ascontiguousarray(queries)
    if q.ndim == 2:
        q = q[:, None, :]
    B, V, _ = q.shape
    ca, off = csr(clauses)
    if len(ca) == 0:
        ca = np.zeros(1, dtype=CLAUSE_DTYPE)
    ids = np.zeros((B, K), dtype=np.int64)
    sc = np.zeros((B, K), dtype=np.float64)
    ps = np.zeros(B, dtype=np.int64)
    rc = lib().oracle_search(dtype, d, n, row0, _p(emb), _p(attrs), W, _p(live), _p(q), B, V,
                             _p(ca), _p(off), K, _p(ids), _p(sc), _p(ps))
    if rc != 0:
        raise ValueError("oracle precondition violated")
    return ids, sc, ps


def merge(ids, scores_, pass_, K):
    """Union of per-shard results [L][B][Kin] -> top-K [B][K]."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    scores_ = np.ascontiguousarray(scores_, dtype=np.float64)
    pass_ = np.ascontiguousarray(pass_, dtype=np.int64)
    L, B, Kin = ids.shape
    oi = np.zeros((B, K), dtype=np.int64)
    osc = np.zeros((B, K), dtype=np.float64)
    op = np.zeros(B, dtype=np.int64)
    rc = lib().oracle_merge(L, B, Kin, _p(ids), _p(scores_), _p(pass_), K, _p(oi), _p(osc), _p(op))
    if rc != 0:
        raise ValueError("oracle precondition violated")
    return oi, osc, op


# ---------------------------------------------------------------- quantised path (oporp_oracle.cpp)
def _prm(prm):
    src, sign = prm
    src = np.ascontiguousarray(src, dtype=np.int32)
    sign = np.ascontiguousarray(sign, dtype=np.int8)
    return src, sign, len(src)


def oporp_encode(dtype, emb, k, prm):
    """Sign-OPORP codes [n][k/64] uint64 of rows emb [n][d] (storage repr). prm = (src, sign)."""
    emb = np.ascontiguousarray(emb)
    n, d = emb.shape
    src, sign, L = _prm(prm)
    out = np.zeros((n, k // 64), dtype=np.uint64)
    if lib().oracle_oporp_encode(dtype, d, n, _p(emb), k, L, _p(src), _p(sign), _p(out)) != 0:
        raise ValueError("oracle precondition violated")
    return out


def matched_bits(k, a, b):
    a = np.ascontiguousarray(a, dtype=np.uint64).reshape(-1, k // 64)
    b = np.ascontiguousarray(b, dtype=np.uint64).reshape(-1, k // 64)
    out = np.zeros(len(a), dtype=np.int32)
    if lib().oracle_matched_bits(k, len(a), _p(a), _p(b), _p(out)) != 0:
        raise ValueError("oracle precondition violated")
    return out


def _search_inputs(emb, attrs, live, queries, clauses):
    emb = np.ascontiguousarray(emb)
    attrs = np.ascontiguousarray(attrs, dtype=np.uint64)
    n, d = emb.shape
    live = np.ascontiguousarray(live, dtype=np.uint8)
    q = np.ascontiguousarray(queries)
    if q.ndim == 2:
        q = q[:, None, :]
    ca, off = csr(clauses)
    if len(ca) == 0:
        ca = np.zeros(1, dtype=CLAUSE_DTYPE)
    return emb, attrs, live, q, ca, off, n, d


def code_search(dtype, emb, attrs, live, queries, clauses, K, k, prm, row0=0):
    """Filtered top-K by matched bits (any K). Returns ids [B][K], m [B][K] int32 (-1 pad), pass [B]."""
    emb, attrs, live, q, ca, off, n, d = _search_inputs(emb, attrs, live, queries, clauses)
    B, V, _ = q.shape
    src, sign, L = _prm(prm)
    ids = np.zeros((B, K), dtype=np.int64)
    m = np.zeros((B, K), dtype=np.int32)
    ps = np.zeros(B, dtype=np.int64)
    rc = lib().oracle_code_search(dtype, d, n, row0, _p(emb), _p(attrs), attrs.shape[1], _p(live), _p(q), B, V,
                                  _p(ca), _p(off), K, k, L, _p(src), _p(sign), _p(ids), _p(m), _p(ps))
    if rc != 0:
        raise ValueError("oracle precondition violated")
    return ids, m, ps


def search_v3(dtype, emb, attrs, live, queries, clauses, K, keep, k, prm, row0=0):
    """V3: clause filter, keep K' by matched bits, full-precision rerank. Returns ids, scores (fp64),
    pass, kept [B]."""
    emb, attrs, live, q, ca, off, n, d = _search_inputs(emb, attrs, live, queries, clauses)
    B, V, _ = q.shape
    src, sign, L = _prm(prm)
    ids = np.zeros((B, K), dtype=np.int64)
    sc = np.zeros((B, K), dtype=np.float64)
    ps = np.zeros(B, dtype=np.int64)
    kept = np.zeros(B, dtype=np.int64)
    rc = lib().oracle_search_v3(dtype, d, n, row0, _p(emb), _p(attrs), attrs.shape[1], _p(live), _p(q), B, V,
                                _p(ca), _p(off), K, float(keep), k, L, _p(src), _p(sign), _p(ids), _p(sc), _p(ps),
                                _p(kept))
    if rc != 0:
        raise ValueError("oracle precondition violated")
    return ids, sc, ps, kept


# ---------------------------------------------------------------- ID-list clauses (linr_oracle.cpp)
ID_CLAUSE_DTYPE = np.dtype([("ids", "<u8"), ("n", "<i4"), ("slot", "u1"), ("reverse", "u1"), ("pad", "u1", 2)])


def search_idc(dtype, emb, attrs, live, idlists, queries, clauses, id_clauses, K, row0=0):
    """Filtered top-K with bitmask clauses and ID-list clauses.
    idlists: list over slots of (ids [n][A_s] uint64, counts [n] uint8);
    id_clauses: per query, list of (slot, reverse, sorted query ids)."""
    emb = np.ascontiguousarray(emb)
    attrs = np.ascontiguousarray(attrs, dtype=np.uint64)
    n, d = emb.shape
    live = np.ascontiguousarray(live, dtype=np.uint8)
    q = np.ascontiguousarray(queries)
    if q.ndim == 2:
        q = q[:, None, :]
    B, V, _ = q.shape
    ca, off = csr(clauses)
    if len(ca) == 0:
        ca = np.zeros(1, dtype=CLAUSE_DTYPE)
    S = len(idlists)
    keep = []
    sid = (ctypes.c_void_p * max(1, S))()
    scnt = (ctypes.c_void_p * max(1, S))()
    width = np.zeros(max(1, S), dtype=np.int32)
    for s_, (ids, cnt) in enumerate(idlists):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        cnt = np.ascontiguousarray(cnt, dtype=np.uint8)
        keep += [ids, cnt]
        sid[s_] = ids.ctypes.data
        scnt[s_] = cnt.ctypes.data
        width[s_] = ids.shape[1]
    flat, ioff = [], [0]
    for cl in id_clauses:
        flat.extend(cl)
        ioff.append(len(flat))
    ic = np.zeros(max(1, len(flat)), dtype=ID_CLAUSE_DTYPE)
    for i, (slot, rev, ids) in enumerate(flat):
        arr = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
        keep.append(arr)
        ic[i]["ids"] = arr.ctypes.data
        ic[i]["n"] = len(arr)
        ic[i]["slot"] = slot
        ic[i]["reverse"] = rev
    ioff = np.array(ioff, dtype=np.int32)
    ids_o = np.zeros((B, K), dtype=np.int64)
    sc = np.zeros((B, K), dtype=np.float64)
    ps = np.zeros(B, dtype=np.int64)
    rc = lib().oracle_search_idc(dtype, d, n, row0, _p(emb), _p(attrs), attrs.shape[1], _p(live), S,
                                 ctypes.cast(sid, ctypes.c_void_p), _p(width), ctypes.cast(scnt, ctypes.c_void_p),
                                 _p(q), B, V, _p(ca), _p(off), _p(ic), _p(ioff), K, _p(ids_o), _p(sc), _p(ps))
    if rc != 0:
        raise ValueError("oracle precondition violated")
    return ids_o, sc, ps


# ---------------------------------------------------------------- learned scorers (scorer_oracle.cpp)
class _Scorer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("F", ctypes.c_int32), ("H", ctypes.c_int32), ("K", ctypes.c_int32),
                ("dc", ctypes.c_int32), ("G", ctypes.c_int32)] + \
               [(nm, ctypes.c_void_p) for nm in ("Wm", "bm", "Wi", "bi", "W1", "b1", "w2", "b2", "Fk", "Gk",
                                                 "Wgu", "Wgx", "bg", "Wo", "bo")]


def _scorer(w):
    """w: dict from datagen.scorer_weights (float32 arrays). Returns (struct, keep-alive list)."""
    st = _Scorer()
    st.kind = w["kind"]
    for k in ("F", "H", "K", "dc", "G"):
        setattr(st, k, int(w.get(k, 0)))
    keep = []
    for nm, _ in _Scorer._fields_[6:]:
        if nm in w:
            a = np.ascontiguousarray(w[nm], dtype=np.float32)
            keep.append(a)
            setattr(st, nm, a.ctypes.data)
    return st, keep


def scorer_scores(w, dtype, emb, q):
    """Scores of every row of emb for one query vector q under the learned scorer w."""
    st, keep = _scorer(w)
    emb = np.ascontiguousarray(emb)
    q = np.ascontiguousarray(q).reshape(1, -1)
    n, d = emb.shape
    return np.array([lib().oracle_scorer_score(ctypes.byref(st), dtype, d, _p(q), 0, _p(emb), i) for i in range(n)])


def search_scored(w, dtype, emb, attrs, live, queries, clauses, K, row0=0):
    """Filtered top-K under a learned scorer (queries [B][d]). Returns ids, scores (fp64), pass."""
    st, keep = _scorer(w)
    emb = np.ascontiguousarray(emb)
    attrs = np.ascontiguousarray(attrs, dtype=np.uint64)
    n, d = emb.shape
    live = np.ascontiguousarray(live, dtype=np.uint8)
    q = np.ascontiguousarray(queries).reshape(-1, d)
    B = q.shape[0]
    ca, off = csr(clauses)
    if len(ca) == 0:
        ca = np.zeros(1, dtype=CLAUSE_DTYPE)
    ids = np.zeros((B, K), dtype=np.int64)
    sc = np.zeros((B, K), dtype=np.float64)
    ps = np.zeros(B, dtype=np.int64)
    rc = lib().oracle_search_scored(ctypes.byref(st), dtype, d, n, row0, _p(emb), _p(attrs), attrs.shape[1],
                                    _p(live), _p(q), B, _p(ca), _p(off), K, _p(ids), _p(sc), _p(ps))
    if rc != 0:
        raise ValueError("oracle precondition violated")
    return ids, sc, ps
