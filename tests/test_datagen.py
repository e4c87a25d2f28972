"""Generator checks (-m "not gpu"): determinism, counter-based subset consistency, value ranges,
and pass rates against their closed forms (SURVEY.md §8(d) presets)."""
import math

import numpy as np
import pytest

import datagen as dg
import oracle


def test_splitmix64_reference_values():
    # SplitMix64 with state 0: first outputs of the reference generator (Vigna), i.e. sm64(k*golden)
    # for k=0,1,2 taken from the published sequence for seed 0.
    assert dg.sm64_int(0) == 0xE220A8397B1DCDAF
    assert int(dg.sm64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF
    g = 0x9E3779B97F4A7C15
    assert dg.sm64_int(g) == 0x6E789E6AA1B965F4
    assert dg.sm64_int((2 * g) & dg.MASK64) == 0x06C45D188009454F


@pytest.mark.parametrize("dtype", [dg.F32, dg.F16, dg.BF16, dg.I8])
@pytest.mark.parametrize("mode", [dg.MODE_GRID, dg.MODE_DENSE])
def test_rows_are_counter_based(dtype, mode):
    v_all, a_all = dg.gen_items(5, 0, 300, 64, dtype, mode, W=2)
    v_sub, a_sub = dg.gen_items(5, 123, 77, 64, dtype, mode, W=2)
    assert np.array_equal(v_all[123:200], v_sub)
    assert np.array_equal(a_all[123:200], a_sub)
    v2, _ = dg.gen_items(5, 0, 300, 64, dtype, mode, W=2)
    assert np.array_equal(v_all, v2)


def test_value_ranges():
    v, a = dg.gen_items(1, 0, 2000, 128, dg.I8)
    assert v.min() >= -96 and v.max() <= 94
    g, _ = dg.gen_items(1, 0, 100, 128, dg.BF16, dg.MODE_GRID)
    k = dg.bits_to_f32(g, dg.BF16) * 128
    assert np.array_equal(k, np.round(k)) and np.abs(k).max() <= 127
    f, _ = dg.gen_items(1, 0, 500, 128, dg.F32, dg.MODE_DENSE)
    assert np.abs(f).max() <= 0.75 and np.isfinite(f).all()
    # every item sets exactly one bit per field in word 0
    w0 = a[:, 0]
    for off, nb in ((0, 24), (24, 16), (40, 16), (56, 8)):
        fld = (w0 >> np.uint64(off)) & np.uint64((1 << nb) - 1)
        assert all(bin(int(x)).count("1") == 1 for x in fld[:200])


def exact_pass_prob(clauses):
    """Closed form for independent fields: product over clauses of P(match) or 1-P(match)."""
    probs = {0: dg.field_value_probs(24), 24: dg.field_value_probs(16), 40: dg.field_value_probs(16),
             56: dg.field_value_probs(8)}
    p = 1.0
    for (m, w, r) in clauses:
        for off, nb in ((0, 24), (24, 16), (40, 16), (56, 8)):
            sub = (m >> off) & ((1 << nb) - 1)
            if sub:
                pm = sum(probs[off][v] for v in range(nb) if sub >> v & 1)
                p *= (1 - pm) if r else pm
    return p


@pytest.mark.parametrize("preset,approx", [("ALL", 1.0), ("HIGH", 0.1172), ("HIGH4", 0.1025), ("LOW", 0.00244)])
def test_preset_pass_rates_closed_form(preset, approx):
    n = 200_000
    _, A = dg.gen_items(dg.DATA_SEED, 0, n, 16, dg.I8)
    cls = dg.gen_clauses(dg.QUERY_SEED, 4, preset)
    live = np.ones(n)
    for cl in cls:
        p = exact_pass_prob(cl)
        assert abs(p - approx) < 0.02 * approx + 1e-4
        _, cnt = oracle.filter_mask(A, live, cl)
        sd = math.sqrt(n * p * (1 - p)) + 1e-9
        assert abs(cnt - n * p) <= 5 * sd + 1, (preset, cnt, n * p)


def test_queries_shape_and_source_rows():
    q = dg.gen_queries(3, 4, 1000, 5, 8, 64, dg.BF16)
    assert q.shape == (5, 8, 64) and q.dtype == np.uint16
    src = dg.query_source_rows(3, 1000, 5, 8)
    assert src.min() >= 0 and src.max() < 1000 and len(np.unique(src)) > 30
    q8 = dg.gen_queries(3, 4, 1000, 2, 1, 64, dg.I8)
    base = dg.item_values(4, src[:2, 0], 64, dg.I8, dg.MODE_DENSE)
    assert np.abs(q8[:, 0].astype(int) - base.astype(int)).max() <= 8
