"""Pins for the learned-scorer oracle (oracle/scorer_oracle.cpp; -m "not gpu").

Degenerate weights reduce each scorer to a closed form that another oracle function or
arithmetic fixes: a Hadamard MLP with identity member/item MLPs and a summing head IS the dot
product -- compared with oracle.search exactly on integer-grid data; zero head
weights give the constant bias; MoL with K = 1 is its lone component logit ("the
gates will collapse to a value of 1 if there is only one feature"); a uniform gate averages the
components; MoL softmax weights sum to 1; and a numpy re-derivation of the forward pass
(different association order: matrix products) agrees to 1e-12 relative.
"""
import numpy as np
import pytest

import datagen as dg
import oracle

d = 32


def _identity_hadamard(C=2.0 ** 20):
    # member/item MLPs = identity (F = d), head: one hidden unit = sum(h_q * h_x) + C (ReLU is the
    # identity above -C), output = z - C: exactly the dot product for |dot| < C
    I = np.eye(d, dtype=np.float32)
    return {"kind": 1, "F": d, "H": 1, "Wm": I, "bm": np.zeros(d, np.float32), "Wi": I, "bi": np.zeros(d, np.float32),
            "W1": np.ones((1, d), np.float32), "b1": np.array([C], np.float32), "w2": np.ones(1, np.float32),
            "b2": np.array([-C], np.float32)}


def test_hadamard_identity_is_dot_product():
    n, K = 2000, 100
    vals, attrs = dg.gen_items(31, 0, n, d, dg.F32, dg.MODE_GRID)
    Q = dg.gen_queries(32, 31, n, 3, 1, d, dg.F32, dg.MODE_GRID)[:, 0]
    cls = dg.gen_clauses(32, 3, "HIGH")
    a = oracle.search_scored(_identity_hadamard(), dg.F32, vals, attrs, np.ones(n), Q, cls, K)
    b = oracle.search(dg.F32, vals, attrs, np.ones(n), Q, cls, K)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_hadamard_zero_head_is_constant():
    n = 300
    vals, attrs = dg.gen_items(33, 0, n, d, dg.BF16, dg.MODE_DENSE)
    w = dg.scorer_weights(1, "hadamard", d)
    w["W1"] = np.zeros_like(w["W1"])
    w["b1"] = np.zeros_like(w["b1"])
    w["b2"] = np.array([0.375], np.float32)
    Q = dg.gen_queries(34, 33, n, 1, 1, d, dg.BF16, dg.MODE_DENSE)[:, 0]
    ids, sc, ps = oracle.search_scored(w, dg.BF16, vals, attrs, np.ones(n), Q, [[]], 10)
    assert ids[0].tolist() == list(range(10)) and np.all(sc[0] == 0.375)


def _numpy_forward(w, X, q):
    if w["kind"] == 1:
        hq = w["Wm"].astype(np.float64) @ q + w["bm"]
        hx = X @ w["Wi"].astype(np.float64).T + w["bi"]
        z = np.maximum((hx * hq) @ w["W1"].astype(np.float64).T + w["b1"], 0.0)
        return z @ w["w2"].astype(np.float64) + w["b2"][0]
    K, dc = w["K"], w["dc"]
    f = (w["Fk"].astype(np.float64) @ q).reshape(K, dc)
    g = (X @ w["Gk"].astype(np.float64).T).reshape(len(X), K, dc)
    delta = (g * f[None]).sum(-1)
    a = np.maximum(X @ w["Wgx"].astype(np.float64).T + (w["Wgu"].astype(np.float64) @ q) + w["bg"], 0.0)
    lg = a @ w["Wo"].astype(np.float64).T + w["bo"]
    pi = np.exp(lg - lg.max(1, keepdims=True))
    pi /= pi.sum(1, keepdims=True)
    return (pi * delta).sum(1), pi


@pytest.mark.parametrize("kind", ["hadamard", "mol"])
def test_forward_pass_vs_numpy(kind):
    n = 200
    vals, _ = dg.gen_items(35, 0, n, d, dg.F32, dg.MODE_DENSE)
    w = dg.scorer_weights(3, kind, d)
    q = dg.gen_queries(36, 35, n, 1, 1, d, dg.F32, dg.MODE_DENSE)[0, 0]
    s = oracle.scorer_scores(w, dg.F32, vals, q)
    ref = _numpy_forward(w, vals.astype(np.float64), q.astype(np.float64))
    ref = ref[0] if kind == "mol" else ref
    assert np.allclose(s, ref, rtol=1e-12, atol=1e-12)
    if kind == "mol":   # gate rows are a probability distribution
        pi = _numpy_forward(w, vals.astype(np.float64), q.astype(np.float64))[1]
        assert np.allclose(pi.sum(1), 1.0, atol=1e-12) and np.all(pi >= 0)


def test_mol_single_component_and_uniform_gate():
    n = 150
    vals, _ = dg.gen_items(37, 0, n, d, dg.F32, dg.MODE_DENSE)
    q = dg.gen_queries(38, 37, n, 1, 1, d, dg.F32, dg.MODE_DENSE)[0, 0]
    w1 = dg.scorer_weights(5, "mol", d, K=1, dc=8)
    s1 = oracle.scorer_scores(w1, dg.F32, vals, q)
    delta = (vals.astype(np.float64) @ w1["Gk"].astype(np.float64).T) @ (w1["Fk"].astype(np.float64) @ q)
    assert np.allclose(s1, delta, rtol=1e-12, atol=1e-12)     # pi_1 = 1
    w2 = dg.scorer_weights(5, "mol", d, K=2, dc=8)
    w2["Wo"] = np.zeros_like(w2["Wo"])
    w2["bo"] = np.zeros_like(w2["bo"])
    s2 = oracle.scorer_scores(w2, dg.F32, vals, q)
    f = (w2["Fk"].astype(np.float64) @ q).reshape(2, 8)
    g = (vals.astype(np.float64) @ w2["Gk"].astype(np.float64).T).reshape(n, 2, 8)
    assert np.allclose(s2, (g * f[None]).sum(-1).mean(1), rtol=1e-12, atol=1e-12)
