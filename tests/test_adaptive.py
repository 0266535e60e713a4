"""Interactive rate-adaptive reconciliation (R25): the oracle's reveal
loop pinned against the accounting the paper/SPEC fix, and the CUDA path (qkd_reconcile_adaptive)
bit-exact against it."""
import numpy as np
import pytest

import oracle
import synth
from _common import assert_same


def _c4(q):
    w = synth.workload(f"C4@{q:g}")
    d, p, s = w.rate_adaptive_counts()
    return w, d, p, s, w.reveal_order()


def test_reveal_pattern_partitions_reserved_set():
    """SPEC alice_reveal: P and S stay disjoint with |P| + |S| = d; round 0 is the R19 pattern."""
    w, d, p, s, order = _c4(0.04)
    for sk in (s, s + 7, d):
        kind = oracle.reveal_pattern(w.n, order, sk)
        assert (kind == 2).sum() == sk and (kind == 1).sum() == d - sk
        assert set(np.flatnonzero(kind)) == set(order.tolist())
    assert np.array_equal(oracle.reveal_pattern(w.n, order, s), w.pos_kind())


@pytest.mark.parametrize("q", synth.C4_QBERS)
def test_adaptive_efficiency_accounting(q):
    """Round 0 is R20's f (closed form pinned in test_oracle_pins); each reveal raises the leak by
    exactly delta bits (SPEC: "leaked_bits increases by exactly k"), so f strictly increases."""
    w, d, p, s, order = _c4(q)
    oc = oracle.Code(w.shifts(), w.Z)
    f = oracle.adaptive_efficiency(oc.m, oc.n, d, s, 50, np.arange(6), q)
    assert f[0] == pytest.approx(oracle.efficiency(oc.m, oc.n, p, s, q), rel=1e-12)
    h2 = -q * np.log2(q) - (1 - q) * np.log2(1 - q)
    assert np.allclose(np.diff(f), 50 / ((oc.n - d) * h2))
    full = oracle.adaptive_efficiency(oc.m, oc.n, d, s, 50, np.array([10 ** 6]), q)[0]
    assert full == pytest.approx(oc.m / ((oc.n - d) * h2))        # everything revealed: leak = m


def _tiny():
    shifts = synth.qc_code(4, 8, 16, {2: 0.5, 3: 0.5}, 77)
    Z = 16
    order = synth.reserved_order(shifts, Z, 5)[:40].astype(np.int32)
    return shifts, Z, order


def test_reveal_rounds_invariants():
    """Zero-error frames stop at round 0; every stopped frame matches its syndrome; shortened and
    revealed positions decode to Alice's bits (their LLRs are +-127, frozen); rounds never exceed
    the reveal budget; more reveals never turn a success into a failure on these frames."""
    shifts, Z, order = _tiny()
    oc = oracle.Code(shifts, Z)
    x, y, _ = synth.frames(oc.n, 0.06, 123, 0, 40)
    y[:5] = x[:5]                                       # zero-error frames
    syn = oc.syndrome(x)
    r = oracle.reveal_rounds(oc, 0.06, y, x, syn, order, 4, 6, 6, 40)
    assert (r["rounds"][:5] == 0).all() and (r["success"][:5] == 1).all()
    ok = r["success"] == 1
    assert np.array_equal(oc.syndrome(r["bits"][ok]), syn[ok])
    assert r["rounds"].max() <= 6 and len(np.unique(r["rounds"])) > 1
    bits = np.unpackbits(r["bits"], axis=1, bitorder="little")[:, :oc.n]
    xb = np.unpackbits(x, axis=1, bitorder="little")[:, :oc.n]
    for f in range(40):
        s_k = min(4 + 6 * int(r["rounds"][f]), len(order))
        assert np.array_equal(bits[f, order[:s_k]], xb[f, order[:s_k]])
    # monotone: revealing everything up front decodes at least the frames that succeeded
    r_all = oracle.reveal_rounds(oc, 0.06, y, x, syn, order, len(order), 6, 0, 40)
    assert (r_all["success"][ok] == 1).all()


@pytest.mark.gpu
def test_adaptive_parity_tiny(gpu):
    import torch

    shifts, Z, order = _tiny()
    oc = oracle.Code(shifts, Z)
    x, y, _ = synth.frames(oc.n, 0.07, 321, 0, 61)
    syn = oc.syndrome(x)
    o = oracle.reveal_rounds(oc, 0.07, y, x, syn, order, 2, 5, 7, 40)
    code = gpu.QCCode(shifts, Z)
    g = code.reconcile_adaptive(0.07, torch.from_numpy(order).cuda(), 2, 5, 7, torch.from_numpy(y).cuda(),
                                torch.from_numpy(x).cuda(), torch.from_numpy(syn).cuda(), 40)
    g = {k: v.cpu().numpy() for k, v in g.items()}
    assert_same(g, o, keys=("bits", "iters", "success", "rounds"))
    assert len(np.unique(o["rounds"])) > 2


@pytest.mark.gpu
@pytest.mark.parametrize("q,delta", [(0.02, 400), (0.08, 800)])
def test_adaptive_parity_c4(gpu, q, delta):
    """C4 mother code (n = 81920): f = 1.1 fails at round 0; reveal rounds raise f until frames decode."""
    import torch

    w, d, p, s, order = _c4(q)
    F = 6
    x, y, _ = w.gen(0, F)
    oc = oracle.Code(w.shifts(), w.Z)
    syn = oc.syndrome(x)
    o = oracle.reveal_rounds(oc, q, y, x, syn, order, s, delta, 3, w.max_iter)
    code = gpu.QCCode(w.shifts(), w.Z, w.pos_kind())
    g = code.reconcile_adaptive(q, torch.from_numpy(order).cuda(), s, delta, 3, torch.from_numpy(y).cuda(),
                                torch.from_numpy(x).cuda(), torch.from_numpy(syn).cuda(), w.max_iter)
    g = {k: v.cpu().numpy() for k, v in g.items()}
    assert_same(g, o, keys=("bits", "iters", "success", "rounds"))


@pytest.mark.gpu
@pytest.mark.parametrize("F,q_data,rounds", [(2500, 0.07, 7), (300, 0.005, 6), (97, 0.07, 0)])
def test_adaptive_parity_device_compaction(gpu, F, q_data, rounds):
    """The round loop keeps the still-failed list on the device (no host sync): many frames (the
    1024-thread compaction takes chunks of several frames), a batch whose frames all match in round 0
    (later rounds run on an empty list), and max_rounds = 0 (a single, last round)."""
    import torch

    shifts, Z, order = _tiny()
    oc = oracle.Code(shifts, Z)
    x, y, _ = synth.frames(oc.n, q_data, 777 + F, 0, F)
    syn = oc.syndrome(x)
    o = oracle.reveal_rounds(oc, 0.07, y, x, syn, order, 2, 5, rounds, 40)
    code = gpu.QCCode(shifts, Z)
    g = code.reconcile_adaptive(0.07, torch.from_numpy(order).cuda(), 2, 5, rounds, torch.from_numpy(y).cuda(),
                                torch.from_numpy(x).cuda(), torch.from_numpy(syn).cuda(), 40)
    g = {k: v.cpu().numpy() for k, v in g.items()}
    assert_same(g, o, keys=("bits", "iters", "success", "rounds"))
