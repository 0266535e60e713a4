"""Pins of the fp64 exact layered BP oracle (R26) against things other
than itself: the literal Eq.(6), the paper's/SPEC's box-plus values, closed forms, and exact
posterior marginals by brute force on cycle-free Tanner graphs (BP is exact on trees)."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_beta_matches_literal_eq6():
    """Stable form == 2 atanh(tanh(a/2) tanh(b/2)) wherever the literal form is accurate."""
    for a in np.linspace(0, 14, 57):
        for b in np.linspace(0, 14, 43):
            assert oracle.beta(a, b) == pytest.approx(oracle.beta_eq6(a, b), rel=1e-9, abs=1e-12)


def test_boxplus_golden_and_closed_forms():
    g = json.load(open(os.path.join(GOLD, "boxplus.json")))
    for a, b, v in g["pairs"]:
        assert oracle.beta(a, b) == pytest.approx(v, abs=g["tol"])
    for a, b, c, v in g["triples"]:   # Eq.(7): the 4th output of a degree-4 check with inputs a, b, c
        out = oracle.check_node_float([a, b, c, 5.0], 0)
        assert out[3] == pytest.approx(v, abs=g["tol"])
    # degree 2: each output is the other input, sign by Eq.(1) with the syndrome bit (R5)
    assert list(oracle.check_node_float([3.0, -7.0], 0)) == pytest.approx([-7.0, 3.0])
    assert list(oracle.check_node_float([3.0, -7.0], 1)) == pytest.approx([7.0, -3.0])
    # beta(a, 0) = 0; beta(a, large) = a; beta <= min
    assert oracle.beta(4.0, 0.0) == 0.0 and oracle.beta(3.0, oracle.LLR_KNOWN) == pytest.approx(3.0)
    rng = np.random.default_rng(3)
    for _ in range(200):
        a, b = rng.uniform(0, 30, 2)
        assert oracle.beta(a, b) <= min(a, b) + 1e-12
    # associativity of the exact box-plus: F/B order is immaterial up to rounding
    x = rng.normal(0, 4, 9)
    o = oracle.check_node_float(x, 0)
    o_rev = oracle.check_node_float(x[::-1].copy(), 0)[::-1]
    assert np.allclose(o, o_rev, rtol=1e-10, atol=1e-12)


def _exact_posterior(H, llr, s):
    """log P(x_j = 0 | y, Hx = s) / P(x_j = 1 | y, Hx = s) by enumerating every word."""
    n = H.shape[1]
    num = np.zeros(n)
    den = np.zeros(n)
    for bits in itertools.product((0, 1), repeat=n):
        x = np.array(bits)
        if ((H @ x) % 2 != s).any():
            continue
        w = np.exp(np.sum(llr * (1 - 2 * x)) / 2)
        num += w * (x == 0)
        den += w * (x == 1)
    return np.log(num / den)


@pytest.mark.parametrize("shifts,T", [
    ([[0, 0, 0, -1, -1], [-1, -1, 0, 0, 0]], 3),                                        # 2 checks
    ([[0, 0, 0, -1, -1, -1, -1], [-1, -1, 0, 0, 0, -1, -1], [-1, -1, -1, -1, 0, 0, 0]], 4),  # chain of 3
    ([[0, 0, 0, 0, -1, -1, -1, -1], [-1, 0, -1, -1, 0, 0, -1, -1], [-1, -1, 0, -1, -1, -1, 0, 0]], 4),  # star
])
def test_bp_is_exact_on_trees(shifts, T):
    """On a cycle-free graph layered BP converges to the exact posterior LLRs: pins Eq.(1), Eq.(2)/(6),
    Eq.(8), Eq.(9) and the syndrome sign rule (R5) together."""
    sh = np.array(shifts, dtype=np.int32)
    code = oracle.Code(sh, 1)                              # Z = 1: H is the base-matrix pattern
    H = (sh >= 0).astype(int)
    rng = np.random.default_rng(len(shifts) * 7 + T)
    for trial in range(20):
        llr = rng.normal(0, 2.5, code.n)
        s = rng.integers(0, 2, code.m)
        syn = np.packbits(s.astype(np.uint8), bitorder="little")
        r = oracle.decode_float(code, llr[None], syn[None], T, 0)
        assert np.allclose(r["E"][0], _exact_posterior(H, llr, s), rtol=1e-9, atol=1e-9)


def test_float_decoder_invariants():
    import synth

    w = synth.workload("C1")
    code = oracle.Code(w.shifts(), w.Z)
    x, y, _ = w.gen(0, 24)
    syn = code.syndrome(x)
    llr = oracle.build_llr_float(code.n, w.qber, y)
    assert np.allclose(np.abs(llr), np.log(0.95 / 0.05))
    r = oracle.decode_float(code, llr, syn, w.max_iter, 1)
    ok = r["success"] == 1
    assert ok.mean() > 0.9 and np.array_equal(code.syndrome(r["bits"][ok]), syn[ok])
    r0 = oracle.decode_float(code, oracle.build_llr_float(code.n, w.qber, x), syn, w.max_iter, 1)
    assert (r0["iters"] == 0).all() and np.array_equal(r0["bits"], x)


@pytest.mark.parametrize("shifts,T", [
    ([[0, 0, 0, -1, -1], [-1, -1, 0, 0, 0]], 3),
    ([[0, 0, 0, -1, -1, -1, -1], [-1, -1, 0, 0, 0, -1, -1], [-1, -1, -1, -1, 0, 0, 0]], 5),
])
def test_flooding_bp_is_exact_on_trees(shifts, T):
    """The flooding schedule reaches the same exact posteriors on a tree."""
    sh = np.array(shifts, dtype=np.int32)
    code = oracle.Code(sh, 1)
    H = (sh >= 0).astype(int)
    rng = np.random.default_rng(99 + T)
    for trial in range(10):
        llr = rng.normal(0, 2.5, code.n)
        s = rng.integers(0, 2, code.m)
        syn = np.packbits(s.astype(np.uint8), bitorder="little")
        r = oracle.decode_float(code, llr[None], syn[None], T, 0, flooding=True)
        assert np.allclose(r["E"][0], _exact_posterior(H, llr, s), rtol=1e-9, atol=1e-9)


def test_flooding_equals_layered_with_one_layer():
    """With one block row no variable is shared between layers, so both schedules coincide."""
    import synth

    sh = synth.qc_code(1, 6, 32, {1: 1.0}, 5)
    code = oracle.Code(sh, 32)
    rng = np.random.default_rng(1)
    llr = rng.normal(0, 3, (4, code.n))
    syn = rng.integers(0, 256, (4, (code.m + 7) // 8), dtype=np.uint8)
    a = oracle.decode_float(code, llr, syn, 5, 0)
    b = oracle.decode_float(code, llr, syn, 5, 0, flooding=True)
    for k in ("E", "L"):   # equal up to rounding: layered forms E - L + L_new, flooding llr + L_new
        assert np.allclose(a[k], b[k], rtol=1e-12, atol=1e-12)
