"""Shared helpers for the GPU parity tests: run the same seeded inputs through the CUDA path
(via the C ABI binding) and through the CPU oracle, and compare."""
from __future__ import annotations

import numpy as np

import oracle
import synth


def to_np(r):
    return {k: v.cpu().numpy() for k, v in r.items()}


def gpu_decode(p, shifts, Z, kind, llr_np, syn_np, T, early_stop, want_state=True, counters=None):
    import torch

    code = p.QCCode(shifts, Z, kind)
    llr = torch.from_numpy(np.ascontiguousarray(llr_np)).cuda()
    syn = torch.from_numpy(np.ascontiguousarray(syn_np)).cuda()
    r = code.decode(llr, syn, T, early_stop, want_state=want_state, counters=counters)
    torch.cuda.synchronize()
    return to_np(r), code


def oracle_decode(shifts, Z, llr_np, syn_np, T, early_stop, want_state=True):
    code = oracle.Code(shifts, Z)
    return code.decode(llr_np, syn_np, T, early_stop, want_state=want_state)


def assert_same(g, o, keys=("bits", "iters", "success", "L", "E"), frames=None):
    for k in keys:
        a = np.asarray(g[k])
        b = np.asarray(o[k])
        if frames is not None:
            a = a[frames]
        assert a.shape == b.shape, (k, a.shape, b.shape)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{k}: {len(bad)} mismatches, first at {bad[:5].tolist()} "
                                 f"gpu={a[tuple(bad[0])]} oracle={b[tuple(bad[0])]}")


def workload_inputs(name, F, f0=0):
    """Oracle-side inputs for a named workload: (w, shifts, kind, x, y, llr, syn)."""
    w = synth.workload(name)
    shifts = w.shifts()
    kind = w.pos_kind()
    x, y, _ = w.gen(f0, F)
    oc = oracle.Code(shifts, w.Z)
    syn = oc.syndrome(x)
    llr = oc.build_llr(w.qber, y, kind, x)
    return w, shifts, kind, x, y, llr, syn
