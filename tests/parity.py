"""Helpers for GPU-vs-oracle parity tests (test infrastructure; imports both sides)."""
from __future__ import annotations

import math

import numpy as np
import torch

import datagen as dg
import oracle

TORCH_OF = {dg.F32: torch.float32, dg.F16: torch.float16, dg.BF16: torch.bfloat16, dg.I8: torch.int8}


def to_torch(vals: np.ndarray, dtype: int, device) -> torch.Tensor:
    if dtype in (dg.F16, dg.BF16):
        return torch.from_numpy(np.ascontiguousarray(vals).view(np.int16)).view(TORCH_OF[dtype]).to(device)
    return torch.from_numpy(np.ascontiguousarray(vals)).to(device)


def attrs_torch(attrs: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(attrs).view(np.int64)).to(device)


def make_index(vals, attrs, dtype, device="cuda", capacity=None, row0=0):
    from paper_2407_13218_b200 import Index
    n, d = vals.shape
    W = attrs.shape[1]
    ix = Index(capacity or max(n, 1), d, dtype, W, global_row0=row0, device=device)
    if n:
        ix.load(to_torch(vals, dtype, device), attrs_torch(attrs, device))
    return ix


def tolerance(dtype: int, s_ref: float, absdot: float, d: int) -> float:
    """Reading R8: |s_gpu - s_ref| <= max(1e-3*|s_ref|, 2*d*2^-24 * sum_j |q_j x_j|)."""
    if dtype == dg.I8:
        return 0.0
    return max(1e-3 * abs(s_ref), 2.0 * d * 2.0 ** -24 * absdot)


def _ref_scores_for(dtype, vals, q_bv, ids_local):
    """Oracle scores (max over V) and sum|q x| bounds for selected rows."""
    rows = vals[ids_local]
    best = np.full(len(ids_local), -np.inf)
    absd = np.zeros(len(ids_local))
    for v in range(q_bv.shape[0]):
        s = oracle.scores(dtype, rows, q_bv[v])
        best = np.maximum(best, s)
        xa = np.abs(dg.bits_to_f32(rows, dtype).astype(np.float64)) if dtype != dg.I8 else np.abs(rows.astype(np.float64))
        qa = np.abs(dg.bits_to_f32(q_bv[v], dtype).astype(np.float64)) if dtype != dg.I8 else np.abs(q_bv[v].astype(np.float64))
        absd = np.maximum(absd, xa @ qa)
    return best, absd


def check(dtype, vals, attrs, live, queries, clauses, K, gpu, ref, exact: bool, row0=0, what=""):
    """Compare GPU (ids, scores, pass) with the oracle's, element by element (exact) or per R9."""
    gi, gs, gp = [t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t) for t in gpu]
    oi, os_, op = ref
    q = queries if queries.ndim == 3 else queries[:, None, :]
    B = q.shape[0]
    d = vals.shape[1] if vals.ndim == 2 else q.shape[-1]
    assert np.array_equal(gp, op), f"{what}: pass counts differ {gp} vs {op}"
    for b in range(B):
        n = int(min(K, op[b]))
        # padding
        assert np.all(gi[b, n:] == -1), f"{what}: padding ids"
        assert np.all(np.isneginf(gs[b, n:])), f"{what}: padding scores"
        if exact:
            assert np.array_equal(gi[b, :n], oi[b, :n]), f"{what} b={b}: ids differ\n{gi[b,:n][:20]}\n{oi[b,:n][:20]}"
            assert np.array_equal(gs[b, :n].astype(np.float64), os_[b, :n]), f"{what} b={b}: scores differ"
            continue
        if n == 0:
            continue
        ids = gi[b, :n]
        assert len(np.unique(ids)) == n, f"{what}: duplicate ids"
        loc = ids - row0
        assert np.all((loc >= 0) & (loc < len(vals))), f"{what}: id out of range"
        # soundness: every returned id is live and passes the clauses
        m, _ = oracle.filter_mask(attrs[loc], live[loc], clauses[b])
        assert m.all(), f"{what}: returned an item failing the filter"
        sref, absd = _ref_scores_for(dtype, vals, q[b], loc)
        tol = np.array([tolerance(dtype, s, a, d) for s, a in zip(sref, absd)])
        err = np.abs(gs[b, :n].astype(np.float64) - sref)
        assert np.all(err <= tol), f"{what}: score error {err.max()} > tol"
        # ordering: scores non-increasing, ties by ascending id
        assert np.all(np.diff(gs[b, :n]) <= 0), f"{what}: not sorted"
        eq = np.diff(gs[b, :n]) == 0
        assert np.all(np.diff(ids)[eq] > 0), f"{what}: tie order"
        # set equality up to ties within tolerance at the K-th boundary (reading R9)
        tau = os_[b, n - 1]
        diff = set(ids.tolist()) ^ set(oi[b, :n].tolist())
        if diff:
            for i in diff:
                sr, ad = _ref_scores_for(dtype, vals, q[b], np.array([i - row0]))
                t = tolerance(dtype, sr[0], ad[0], d)
                assert abs(sr[0] - tau) <= 2 * t + 1e-12, f"{what}: id {i} differs away from the boundary"
