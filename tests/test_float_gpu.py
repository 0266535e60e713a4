"""GPU parity of the exact floating-point BP decoder (fp32, qkd_decode_float_batch) with the fp64
oracle (R26).

Tolerance (derived, R26): each fp32 box-plus has an absolute error <= ~5e-7 (min exact,
two log1pf(expf(.)) terms <= ln 2 with <= 2 ulp each); a check-node output passes through <= 2(D-1)
box-plus evaluations, each 1-Lipschitz in its inputs, and an a-posteriori LLR sums <= 6 messages, so
after T sweeps |fp32 - fp64| stays below ~ T * 6 * 2D * 5e-7 * (growth) -- the tests use
atol = 2e-3 * T plus rtol = 1e-5 for large magnitudes.  Decisions (E < 0) and iteration counts of
full decodes are taken in fp32 on one side and fp64 on the other, so they are compared as
"identical except where the fp64 margin is within the tolerance"."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


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
            assert np.allclose(gv, o[k], rtol=1e-5, atol=2e-3 * T), (k, T, np.abs(gv - o[k]).max())


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
    same = (g["iters"] == o["iters"]) & (g["success"] == o["success"]) & (g["bits"] == o["bits"]).all(axis=1)
    assert same.mean() >= 0.95, same.mean()
    ok = (g["success"] == 1)
    assert np.array_equal(oc.syndrome(g["bits"][ok]), syn[ok])       # success => syndrome match


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
            assert np.allclose(gv, o[k], rtol=1e-5, atol=2e-3 * T), (k, T, np.abs(gv - o[k]).max())


def test_flooding_full_decodes(gpu):
    import torch

    w, oc, x, y, syn = _inputs("C1", 64)
    o = oracle.decode_float(oc, oracle.build_llr_float(oc.n, w.qber, y), syn, w.max_iter, 1, flooding=True)
    code = gpu.QCCode(w.shifts(), w.Z)
    g = code.decode_float(code.build_llr_float(w.qber, torch.from_numpy(y).cuda()), torch.from_numpy(syn).cuda(),
                          w.max_iter, True, flooding=True)
    g = {k: v.cpu().numpy() for k, v in g.items()}
    same = (g["iters"] == o["iters"]) & (g["success"] == o["success"]) & (g["bits"] == o["bits"]).all(axis=1)
    assert same.mean() >= 0.95, same.mean()


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
            assert np.allclose(gv, o[k], rtol=1e-5, atol=2e-3 * T), (k, T, np.abs(gv - o[k]).max())
