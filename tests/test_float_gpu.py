"""GPU parity of the exact floating-point BP decoder (fp32, qkd_decode_float_batch) with the fp64
oracle (R26).

Tolerance: every fp32 box-plus / sum carries a relative error of a few ulps (2^-24 ~ 6e-8) of its
magnitude, and the layered sweeps compound it roughly linearly in the sweep count T (each message is
a 1-Lipschitz function of its inputs).  Measured on B200 (scratch float_err runs, C1/C2/C3, T = 1..12):
max |fp32 - fp64| / max(1, |fp64|) = 1.1e-6 (T=1), 1.9e-6 (T=2), 4.6e-6 (T=3), 6.8e-6 (T=5), 1.3e-5
(T=12); large converged LLRs (|E| ~ 1e4) carry proportionally larger absolute errors.  The tests
use |fp32 - fp64| <= REL * T * max(1, |fp64|) with REL = 4e-6 (2-4x the measured worst case).

Full decodes: a frame's decisions can differ only if some a-posteriori value of its fp64 trajectory
comes within the tolerance of zero (a decision E < 0, or through it the syndrome test, flips).  So
every frame must match exactly (bits, iterations, success), EXCEPT frames whose fp64 trajectory has
min_j |E_j| <= MARGIN * t after some sweep t before both runs stopped -- those are checked only for
validity (success => syndrome match).  MARGIN = 1e-4 is 25x REL."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

REL = 4e-6      # per sweep, relative to max(1, |v|)
MARGIN = 1e-4   # per sweep: decisions closer to zero than this may legitimately differ


def _close(g, o, T, scale=1.0):
    tol = REL * scale * T * np.maximum(1.0, np.abs(o))
    return np.abs(g - o) <= tol


def _check_full(oc, llr_o, syn, o, g, T, flooding=False):
    """Frames where fp32 and fp64 disagree must have had a near-zero a-posteriori value on the fp64
    trajectory (recomputed sweep by sweep with early stop off) before either run stopped."""
    same = (g["iters"] == o["iters"]) & (g["success"] == o["success"]) & (g["bits"] == o["bits"]).all(axis=1)
    for f in np.flatnonzero(~same):
        stop = int(max(g["iters"][f], o["iters"][f]))
        close = abs(llr_o[f]).min() <= MARGIN
        for t in range(1, min(stop, T) + 1):
            r = oracle.decode_float(oc, llr_o[f:f + 1], syn[f:f + 1], t, 0, flooding=flooding)
            close = close or np.abs(r["E"]).min() <= MARGIN * t
        assert close, f"frame {f}: fp32 and fp64 differ with every fp64 decision margin above {MARGIN} x sweep"
    ok = g["success"] == 1
    assert np.array_equal(oc.syndrome(g["bits"][ok]), syn[ok])       # success => syndrome match
    return same.mean()


def _inputs(name, F):
    w = synth.workload(name)
    oc = oracle.Code(w.shifts(), w.Z)
    x, y, _ = w.gen(0, F)
    syn = oc.syndrome(x)
    return w, oc, x, y, syn


@pytest.mark.parametrize("name,F", [("C1", 16), ("C2", 6), ("C3", 2)])
def test_float_llr_and_few_sweeps(gpu, name, F):
    import torch

    w, oc, x, y, syn = _inputs(name, F)
    llr_o = oracle.build_llr_float(oc.n, w.qber, y)
    code = gpu.QCCode(w.shifts(), w.Z)
    llr_g = code.build_llr_float(w.qber, torch.from_numpy(y).cuda())
    assert np.allclose(llr_g.cpu().numpy(), llr_o, rtol=1e-7, atol=0)
    for T in (1, 2, 3):
        o = oracle.decode_float(oc, llr_o, syn, T, 0)
        g = code.decode_float(llr_g, torch.from_numpy(syn).cuda(), T, False, want_state=True)
        for k in ("E", "L"):
            gv = g[k].cpu().numpy()
            assert _close(gv, o[k], T).all(), (k, T, np.abs(gv - o[k]).max())


@pytest.mark.parametrize("name,F", [("C1", 64), ("C2", 48)])
def test_float_full_decodes(gpu, name, F):
    import torch

    w, oc, x, y, syn = _inputs(name, F)
    llr_o = oracle.build_llr_float(oc.n, w.qber, y)
    o = oracle.decode_float(oc, llr_o, syn, w.max_iter, 1)
    code = gpu.QCCode(w.shifts(), w.Z)
    g = code.decode_float(code.build_llr_float(w.qber, torch.from_numpy(y).cuda()), torch.from_numpy(syn).cuda(),
                          w.max_iter, True)
    g = {k: v.cpu().numpy() for k, v in g.items()}
    _check_full(oc, llr_o, syn, o, g, w.max_iter)


def test_float_zero_error_frames(gpu):
    import torch

    w, oc, x, y, syn = _inputs("C2", 5)
    code = gpu.QCCode(w.shifts(), w.Z)
    g = code.decode_float(code.build_llr_float(w.qber, torch.from_numpy(x).cuda()), torch.from_numpy(syn).cuda(),
                          w.max_iter, True)
    assert (g["iters"].cpu().numpy() == 0).all() and np.array_equal(g["bits"].cpu().numpy(), x)


@pytest.mark.parametrize("name,F", [("C1", 16), ("C2", 6)])
def test_flooding_few_sweeps(gpu, name, F):
    """Flooding schedule vs the fp64 oracle's flooding, same tolerance."""
    import torch

    w, oc, x, y, syn = _inputs(name, F)
    llr_o = oracle.build_llr_float(oc.n, w.qber, y)
    code = gpu.QCCode(w.shifts(), w.Z)
    llr_g = code.build_llr_float(w.qber, torch.from_numpy(y).cuda())
    for T in (1, 2, 3):
        o = oracle.decode_float(oc, llr_o, syn, T, 0, flooding=True)
        g = code.decode_float(llr_g, torch.from_numpy(syn).cuda(), T, False, want_state=True, flooding=True)
        for k in ("E", "L"):
            gv = g[k].cpu().numpy()
            assert _close(gv, o[k], T).all(), (k, T, np.abs(gv - o[k]).max())


def test_flooding_full_decodes(gpu):
    import torch

    w, oc, x, y, syn = _inputs("C1", 64)
    llr_o = oracle.build_llr_float(oc.n, w.qber, y)
    o = oracle.decode_float(oc, llr_o, syn, w.max_iter, 1, flooding=True)
    code = gpu.QCCode(w.shifts(), w.Z)
    g = code.decode_float(code.build_llr_float(w.qber, torch.from_numpy(y).cuda()), torch.from_numpy(syn).cuda(),
                          w.max_iter, True, flooding=True)
    g = {k: v.cpu().numpy() for k, v in g.items()}
    _check_full(oc, llr_o, syn, o, g, w.max_iter, flooding=True)


@pytest.mark.parametrize("flooding", [False, True])
def test_float_degree_21_to_32(gpu, flooding):
    """The FD = 32 instance of the float kernel (check degrees 21..32): the N3 stable-profile code
    (check degree 27-28) at QBER 1.75 %, a few sweeps against the fp64 oracle."""
    import torch

    cols = [8] * 16 + [3] * 21 + [2] * 13
    shifts = synth.girth6_shifts(synth.peg_mask(8, cols, 7), 1024, 8)
    oc = oracle.Code(shifts, 1024)
    x, y, _ = synth.frames(oc.n, 0.0175, 203, 0, 2)
    syn = oc.syndrome(x)
    llr_o = oracle.build_llr_float(oc.n, 0.0175, y)
    code = gpu.QCCode(shifts, 1024)
    llr_g = code.build_llr_float(0.0175, torch.from_numpy(y).cuda())
    for T in (1, 3):
        o = oracle.decode_float(oc, llr_o, syn, T, 0, flooding=flooding)
        g = code.decode_float(llr_g, torch.from_numpy(syn).cuda(), T, False, want_state=True, flooding=flooding)
        for k in ("E", "L"):
            gv = g[k].cpu().numpy()
            assert _close(gv, o[k], T).all(), (k, T, np.abs(gv - o[k]).max())
