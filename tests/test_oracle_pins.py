"""Pins for the CPU oracle: each test checks the oracle against something the paper or the
mathematics fixes, never against a re-typed copy of the oracle's own formula.

PAPER.md = P:<line>, SPEC.md = S:<line>; DESIGN.md §3 readings R1..R21.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def beta(a, b):
    """Eq.(6) box-plus, numerically stable log-domain form."""
    if a == 0 or b == 0:
        return 0.0
    s = math.copysign(1.0, a) * math.copysign(1.0, b)
    a, b = abs(a), abs(b)
    return s * (min(a, b) + math.log1p(math.exp(-(a + b))) - math.log1p(math.exp(-abs(a - b))))


# ---------------------------------------------------------------- box-plus (test helper pin)
def test_beta_helper_matches_paper_numbers():
    g = _gold("boxplus.json")
    for a, b, v in g["pairs"]:
        assert abs(beta(a, b) - v) < g["tol"]
        # direct Eq.(6) evaluation where tanh does not saturate
        if b < 30:
            assert abs(2 * math.atanh(math.tanh(a / 2) * math.tanh(b / 2)) - v) < g["tol"]
    for a, b, c, v in g["triples"]:
        assert abs(beta(a, beta(b, c)) - v) < g["tol"]      # Eq.(7) right fold


# ---------------------------------------------------------------- tau (Algorithm 1)
def test_tau_hand_traces():
    g = _gold("tau_traces.json")
    for c in g["cases"]:
        assert oracle.tau(c["p"], c["q"]) == c["tau"], c["trace"]


def test_tau_invariants_exhaustive():
    # symmetric, <= min(p,q,MSG_max), tau(p,0) = 0; inputs beyond 63 clamp
    for p in range(0, 80):
        assert oracle.tau(p, 0) == 0
        for q in range(0, 80):
            t = oracle.tau(p, q)
            assert t == oracle.tau(q, p)
            assert 0 <= t <= min(p, q, 63)
            assert t == oracle.tau(min(p, 63), min(q, 63))


def test_tau_is_the_boxplus_correction_at_step_quarter():
    """l > 2 branch == l - floor(ln(1+e^{-d*Delta})/Delta) with Delta = 1/4 (R1; P:116 says
    tau is the integer form of beta(p*D + D/2, q*D + D/2); the large-l limit of beta is
    min - ln(1+e^{-|a-b|}))."""
    for l in range(3, 64):
        for d in range(0, 64 - l):
            corr = math.floor(math.log1p(math.exp(-d / 4.0)) * 4.0)
            assert oracle.tau(l, l + d) == l - corr, (l, d)


def test_tau_within_one_step_of_quantized_boxplus():
    """tau(p,q) is the integer representation of beta(p D + D/2, q D + D/2), D = 1/4.
    Integer k represents [kD, (k+1)D) (midpoint kD + D/2), so the exact integer is
    floor(beta/D).  Algorithm 1 is an approximation: allow one step."""
    D = 0.25
    exact = 0
    for p in range(64):
        for q in range(64):
            ref = math.floor(beta(p * D + D / 2, q * D + D / 2) / D)
            t = oracle.tau(p, q)
            assert abs(t - ref) <= 1, (p, q, t, ref)
            exact += t == ref
    assert exact >= 3400          # most of the table is exact, not merely within 1


# ---------------------------------------------------------------- quantization (R1, R2)
def test_llr_magnitude_values():
    g = _gold("quantization.json")
    for q, v in g["cases"]:
        assert oracle.llr_magnitude(q) == v, q
    for q in g["invalid"]:
        assert oracle.llr_magnitude(q) == -1


def test_llr_magnitude_monotone():
    qs = np.linspace(0.001, 0.499, 400)
    v = [oracle.llr_magnitude(q) for q in qs]
    assert all(a >= b for a, b in zip(v, v[1:]))


def test_build_llr_patterns():
    """P:157 rate adaptation: punctured -> 0, shortened -> +-127 by the known bit, payload
    +-Lq by Bob's bit (y=0 -> +)."""
    shifts = np.array([[0, 1, -1, 2], [1, -1, 0, 3]], dtype=np.int32)
    code = oracle.Code(shifts, 5)
    n = code.n
    rng = np.random.default_rng(1)
    y = rng.integers(0, 2, n)
    x = rng.integers(0, 2, n)
    kind = rng.integers(0, 3, n).astype(np.uint8)
    pk = lambda b: np.packbits(b.astype(np.uint8), bitorder="little")
    llr = code.build_llr(0.05, pk(y), kind, pk(x))[0]
    for j in range(n):
        if kind[j] == 0:
            assert llr[j] == (12 if y[j] == 0 else -12)
        elif kind[j] == 1:
            assert llr[j] == 0
        else:
            assert llr[j] == (127 if x[j] == 0 else -127)


# ---------------------------------------------------------------- code expansion
def test_expansion_examples():
    for c in _gold("expansion.json")["cases"]:
        code = oracle.Code(np.array(c["base"], dtype=np.int32), c["Z"])
        assert code.m == c["m"] and code.n == c["n"]
        rows, cols = code.expand()
        if c["edges"] is not None:
            assert sorted(zip(rows.tolist(), cols.tolist())) == sorted(map(tuple, c["edges"]))
        else:
            assert code.n_edges == c["n_edges"]


def test_expansion_circulants_are_permutations():
    w = synth.workload("C2")
    code = oracle.Code(w.shifts(), w.Z)
    rows, cols = code.expand()
    Z = w.Z
    for I in range(w.Mb):
        for J in range(w.Nb):
            sel = (rows // Z == I) & (cols // Z == J)
            if w.shifts()[I, J] < 0:
                assert not sel.any()
            else:
                r = rows[sel] % Z
                cc = cols[sel] % Z
                assert sorted(r.tolist()) == list(range(Z))
                assert sorted(cc.tolist()) == list(range(Z))
                assert np.all(cc == (r + w.shifts()[I, J]) % Z)


def test_invalid_codes_rejected():
    with pytest.raises(ValueError):
        oracle.Code(np.array([[0, 5]], dtype=np.int32), 5)      # shift out of [0, Z)
    with pytest.raises(ValueError):
        oracle.Code(np.array([[0], [0]], dtype=np.int32), 4)    # Nb <= Mb


# ---------------------------------------------------------------- syndrome
def test_syndrome_linearity_and_columns():
    w = synth.workload("C1")
    code = oracle.Code(w.shifts(), w.Z)
    rows, cols = code.expand()
    rng = np.random.default_rng(2)
    nb = (code.n + 7) // 8
    zero = np.zeros(nb, dtype=np.uint8)
    assert not code.syndrome(zero).any()
    a = rng.integers(0, 256, nb, dtype=np.uint8)
    b = rng.integers(0, 256, nb, dtype=np.uint8)
    assert np.array_equal(code.syndrome(a ^ b), code.syndrome(a) ^ code.syndrome(b))
    for j in rng.integers(0, code.n, 10):
        e = np.zeros(code.n, dtype=np.uint8)
        e[j] = 1
        s = np.unpackbits(code.syndrome(np.packbits(e, bitorder="little")), bitorder="little")[: code.m]
        expect = np.zeros(code.m, dtype=np.uint8)
        expect[rows[cols == j]] = 1
        assert np.array_equal(s, expect)


# ---------------------------------------------------------------- VN processing (Alg. 2)
def test_saturation_paper_example():
    """soft value 127 (saturated), increments -50, -40, -70.  Without the guard the
    8-bit value wraps to -33; Algorithm 2 keeps 127."""
    E = 127
    Lold = 20
    for inc in (-50, -40, -70):
        x = E - Lold
        Lnew = max(-63, min(63, Lold + inc))
        E = oracle.vn_update(E, x, Lnew)
        Lold = Lnew
        assert E == 127
    assert oracle.vn_update(-127, -100, 63) == -127
    # 100 + 50 -> 127, clamped, not wrapped
    E, Lold, Lnew = 100, 10, 60            # increment L_new - L_old = +50
    assert oracle.vn_update(E, E - Lold, Lnew) == 127


def test_vn_update_exact_inside_range():
    # below the guard the update is the exact sum Eq.(9), clamped to +-127 (R4)
    for E in range(-126, 127, 7):
        for Lold in range(-63, 64, 9):
            for Lnew in range(-63, 64, 5):
                x = E - Lold
                v = oracle.vn_update(E, x, Lnew)
                exact = x + Lnew
                assert -127 <= v <= 127
                if -127 <= exact <= 127:
                    assert v == exact
                else:
                    assert v == (127 if exact > 0 else -127)


# ---------------------------------------------------------------- CN processing
def test_check_node_paper_examples():
    # degree 3, magnitudes (10,10,10) -> each output tau(10,10) = 8
    assert [abs(v) for v in oracle.check_node([10, 10, 10], 0)] == [8, 8, 8]
    # a zero magnitude zeroes every other output
    out = oracle.check_node([0, 20, -30, 40, 9], 0)
    assert out[1:] == [0, 0, 0, 0]
    # degree 2 swaps magnitudes
    assert [abs(v) for v in oracle.check_node([13, -40], 0)] == [40, 13]
    # degree 1: empty box-plus is +infinity -> MSG_max (R6)
    assert abs(oracle.check_node([5], 0)[0]) == 63


def test_check_node_degree3_is_schedule_free():
    """Degree 3: every leave-one-out output is a single tau of the two other magnitudes
    (Eq.(7) with two operands), whatever the reduction schedule."""
    rng = np.random.default_rng(3)
    for _ in range(2000):
        x = rng.integers(-190, 191, 3)
        m = [min(abs(int(v)), 63) for v in x]
        out = oracle.check_node(x, 0)
        assert [abs(v) for v in out] == [oracle.tau(m[1], m[2]), oracle.tau(m[0], m[2]), oracle.tau(m[0], m[1])]


def test_check_node_sign_and_bounds():
    """Eq.(1): output sign = target bit XOR product of the OTHER input signs (zero inputs
    count as +); |L| <= MSG_max; |o_k| <= min over the others (tau <= min)."""
    rng = np.random.default_rng(4)
    for _ in range(3000):
        d = int(rng.integers(1, 20))
        x = rng.integers(-190, 191, d)
        s = int(rng.integers(0, 2))
        out = oracle.check_node(x, s)
        neg = [int(v < 0) for v in x]
        for k in range(d):
            others = [j for j in range(d) if j != k]
            want_neg = (s + sum(neg[j] for j in others)) % 2
            mag = abs(out[k])
            assert mag <= 63
            if others:
                assert mag <= min(min(abs(int(x[j])), 63) for j in others)
            if mag:
                assert int(out[k] < 0) == want_neg


# ---------------------------------------------------------------- decoder
def _frames(name, F, f0=0):
    w = synth.workload(name)
    code = oracle.Code(w.shifts(), w.Z)
    x, y, ne = w.gen(f0, F)
    return w, code, x, y, ne


def test_zero_error_frames_converge_at_iteration_zero():
    """BASELINE north_star: zero-error frames converge at iteration 0 (R10)."""
    for name in ("C1", "C2"):
        w, code, x, y, ne = _frames(name, 16)
        syn = code.syndrome(x)
        llr = code.build_llr(w.qber, x)            # Bob's word == Alice's word
        r = code.decode(llr, syn, w.max_iter, 1)
        assert (r["iters"] == 0).all() and (r["success"] == 1).all()
        assert np.array_equal(r["bits"], x)
        assert np.array_equal(r["E"], llr)
        assert not r["L"].any()


def test_success_implies_syndrome_match():
    """P:99 / S:322: a returned success satisfies every parity check exactly."""
    for name, F in (("C1", 64), ("C2", 96)):
        w, code, x, y, ne = _frames(name, F)
        syn = code.syndrome(x)
        r = code.decode(code.build_llr(w.qber, y), syn, w.max_iter, 1)
        assert r["success"].sum() > 0
        s2 = code.syndrome(r["bits"])
        for f in range(F):
            if r["success"][f]:
                assert np.array_equal(s2[f], syn[f])
            else:
                assert r["iters"][f] == w.max_iter


def test_state_bounds_and_frozen_shortened_positions():
    """|L| <= 63 and |E| <= 127 always; shortened VNs enter at +-127 and Algorithm 2
    never lets them move."""
    w = synth.workload("C1")
    code = oracle.Code(w.shifts(), w.Z)
    x, y, ne = w.gen(0, 32)
    rng = np.random.default_rng(5)
    kind = rng.choice([0, 0, 0, 1, 2], code.n).astype(np.uint8)
    llr = code.build_llr(w.qber, y, kind, x)
    r = code.decode(llr, code.syndrome(x), 20, 0)
    assert np.abs(r["L"].astype(int)).max() <= 63
    assert np.abs(r["E"].astype(int)).max() <= 127
    sh = kind == 2
    assert np.array_equal(r["E"][:, sh], llr[:, sh])


def test_row_order_inside_a_layer_is_irrelevant():
    """F7/R13: the Z rows of one block row touch disjoint variables (each circulant is a
    permutation), so any row order inside a layer gives the same result bit for bit."""
    w, code, x, y, ne = _frames("C1", 8)
    syn = code.syndrome(x)
    llr = code.build_llr(w.qber, y)
    a = code.decode(llr, syn, 6, 0)
    b = code.decode(llr, syn, 6, 0, perm_seed=12345)
    for k in ("bits", "iters", "success", "L", "E"):
        assert np.array_equal(a[k], b[k]), k


def test_coset_equivariance():
    """Every step is odd-symmetric: flipping Bob's bits by v and Alice's syndrome by Hv
    flips E_j by (-1)^{v_j} and L_e by (-1)^{v_col(e)} exactly (early_stop = 0).  A wrong
    sign rule, a dropped syndrome bit or a mis-indexed edge breaks this."""
    for name, T in (("C1", 12), ("C2", 6)):
        w, code, x, y, ne = _frames(name, 6)
        rows, cols = code.expand()
        syn = code.syndrome(x)
        rng = np.random.default_rng(6)
        v = rng.integers(0, 2, (6, code.n)).astype(np.uint8)
        vp = np.packbits(v, axis=1, bitorder="little")
        a = code.decode(code.build_llr(w.qber, y), syn, T, 0)
        b = code.decode(code.build_llr(w.qber, y ^ vp), syn ^ code.syndrome(vp), T, 0)
        sgnE = 1 - 2 * v.astype(np.int32)
        assert np.array_equal(b["E"].astype(np.int32), sgnE * a["E"].astype(np.int32))
        sgnL = 1 - 2 * v[:, cols].astype(np.int32)
        assert np.array_equal(b["L"].astype(np.int32), sgnL * a["L"].astype(np.int32))


def test_batch_slice_determinism():
    """results depend only on the frame's own inputs."""
    w, code, x, y, ne = _frames("C2", 12)
    syn = code.syndrome(x)
    llr = code.build_llr(w.qber, y)
    full = code.decode(llr, syn, w.max_iter, 1)
    part = code.decode(llr[4:9], syn[4:9], w.max_iter, 1, nthreads=1)
    for k in ("bits", "iters", "success", "L", "E"):
        assert np.array_equal(full[k][4:9], part[k])
    # generator slice == same frames of the full batch (global frame ids)
    x2, y2, _ = w.gen(4, 5)
    assert np.array_equal(x2, x[4:9]) and np.array_equal(y2, y[4:9])


def _ml_tables(code):
    n = code.n
    words = np.arange(1 << n, dtype=np.uint32)
    bits = ((words[:, None] >> np.arange(n, dtype=np.uint32)) & 1).astype(np.uint8)
    rows, cols = code.expand()
    H = np.zeros((code.m, n), dtype=np.uint8)
    H[rows, cols] = 1
    synd = (bits.astype(np.int32) @ H.T.astype(np.int32)) & 1
    skey = synd @ (1 << np.arange(code.m))
    weight = bits.sum(1)
    return words, skey, weight


def test_brute_force_ml_bounds_frame_errors():
    """BASELINE north_star: brute-force ML decoding on tiny codes (n <= 20) bounds the frame
    error rate.  Per frame: a successful decode lies in Alice's coset, so its distance to
    Bob's word is >= the ML (minimum) distance.  Over frames: #BP-correct <= #ML-correct
    (ML with ties counted fractionally) up to sampling noise."""
    shifts = np.array([[0, 1, 3, -1], [2, -1, 4, 0]], dtype=np.int32)   # base 2x4, Z=5, n=20
    code = oracle.Code(shifts, 5)
    words, skey, weight = _ml_tables(code)
    q = 0.06
    F = 3000
    x, y, ne = synth.frames(code.n, q, 777, 0, F)
    syn = code.syndrome(x)
    r = code.decode(code.build_llr(q, y), syn, 30, 1)
    xi = np.unpackbits(x, axis=1, bitorder="little")[:, : code.n] @ (1 << np.arange(code.n))
    yi = np.unpackbits(y, axis=1, bitorder="little")[:, : code.n] @ (1 << np.arange(code.n))
    bi = np.unpackbits(r["bits"], axis=1, bitorder="little")[:, : code.n] @ (1 << np.arange(code.n))
    sk = np.unpackbits(syn, axis=1, bitorder="little")[:, : code.m] @ (1 << np.arange(code.m))
    order = np.argsort(skey, kind="stable")
    sorted_keys = skey[order]
    ml_correct = 0.0
    bp_correct = 0
    for f in range(F):
        lo, hi = np.searchsorted(sorted_keys, [sk[f], sk[f] + 1])
        coset = words[order[lo:hi]]
        dist = np.bitwise_count(coset ^ np.uint32(yi[f]))
        dmin = dist.min()
        if r["success"][f]:
            assert bin(int(bi[f]) ^ int(yi[f])).count("1") >= dmin
        dx = bin(int(xi[f]) ^ int(yi[f])).count("1")
        if dx == dmin:
            ml_correct += 1.0 / int((dist == dmin).sum())
        bp_correct += int(r["success"][f] and bi[f] == xi[f])
    assert bp_correct <= ml_correct + 3 * math.sqrt(F * 0.25)
    assert bp_correct > 0.5 * F        # the decoder does decode


def test_efficiency_closed_form():
    g = _gold("efficiency.json")
    for c in g["cases"]:
        f = oracle.efficiency(c["m"], c["n"], c["p"], c["s"], c["q"])
        assert abs(f - c["f"]) < g["tol"], c["name"]


def test_c4_rate_adaptive_recipe_hits_target_efficiency():
    for q in synth.C4_QBERS:
        w = synth.workload(f"C4@{q:g}")
        d, p, s = w.rate_adaptive_counts()
        assert d == 36965 and p + s == d
        assert abs(oracle.efficiency(w.m, w.n, p, s, q) - 1.1) < 1e-3


def test_check_node_forward_backward_schedule_golden():
    """R6 pinned on degree 4-6 rows (tests/golden/check_node_fb.json): hand traces of the
    forward/backward schedule with Algorithm 1.  Each case also records Eq.(7)'s
    literal per-edge right fold and the per-edge left fold, and differs from both, so an
    oracle that used either (or any other fold order) fails here even though every degree-3 pin
    is schedule-free."""
    g = json.load(open(os.path.join(GOLD, "check_node_fb.json")))
    assert len(g["cases"]) >= 6
    for c in g["cases"]:
        m, fb = c["mag"], c["fb"]
        assert fb != c["right_fold"] and fb != c["left_fold"]
        assert [abs(v) for v in oracle.check_node(m, 0)] == fb
        # the same magnitudes behind x = E - L of either sign and |x| above MSG_max on one edge:
        # magnitudes are min(|x|, 63) (R3) and the sign rule is Eq.(1) with s_i (R5)
        x = [(-v if k % 2 else v) for k, v in enumerate(m)]
        x = [(v + 64 if v == 63 else v) for v in x]
        out = oracle.check_node(x, 1)
        for k, v in enumerate(out):
            assert abs(v) == fb[k]
            want_neg = (1 + sum(1 for j in range(len(x)) if j != k and x[j] < 0)) % 2
            if v:
                assert int(v < 0) == want_neg
