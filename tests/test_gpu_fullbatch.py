"""Full-size launches of the long-frame kernels (VERDICT r1 next#1b): at 4096 frames every
persistent slot decodes many frame groups in turn, reusing its E and message workspace, which the
small-batch parity tests never exercise.  Decode the whole configured batch in one launch and
compare >= 256 frames spread over it -- including frames of the last groups, decoded by slots'
last work items -- byte for byte against the oracle: bits, iterations, success, final L and E."""
import numpy as np
import pytest

import oracle
import synth
from _common import assert_same

pytestmark = pytest.mark.gpu

F_FULL = 4096


def _sample(F, k=256):
    """k frame ids spread over the batch: every (F/k)-th frame, plus the last 8 and frames 1-3."""
    ids = set(np.linspace(0, F - 1, k - 8).astype(int).tolist()) | set(range(F - 8, F)) | {1, 2, 3}
    return np.array(sorted(ids))


def _run(gpu, shifts, Z, kind, x, y, llr, syn, T):
    import torch

    code = gpu.QCCode(shifts, Z, kind)
    r = code.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(syn).cuda(), T, True, want_state=True)
    torch.cuda.synchronize()
    return r, code


def _compare(r, shifts, Z, llr, syn, T, ids):
    import torch

    idx = torch.from_numpy(ids).cuda()
    g = {k: r[k].index_select(0, idx).cpu().numpy() for k in ("bits", "iters", "success", "L", "E")}
    o = oracle.Code(shifts, Z).decode(llr[ids], syn[ids], T, 1, want_state=True)
    assert_same(g, o)
    return g


@pytest.mark.parametrize("q,greg", [(0.02, "1"), (0.08, "1"), (0.08, "0")])
def test_c4_full_batch(gpu, monkeypatch, q, greg):
    """BASELINE configs[3] at its configured 4096 frames (variant 7, E in global memory; QKD_NO_GREG=1:
    the generic variant 4)."""
    if greg == "0":
        monkeypatch.setenv("QKD_NO_GREG", "1")
    w = synth.workload(f"C4@{q:g}")
    shifts, kind = w.shifts(), w.pos_kind()
    x, y, _ = w.gen(0, F_FULL)
    oc = oracle.Code(shifts, w.Z)
    syn = oc.syndrome(x)
    llr = oc.build_llr(w.qber, y, kind, x)
    r, code = _run(gpu, shifts, w.Z, kind, x, y, llr, syn, w.max_iter)
    info = code.launch_info(F_FULL)
    assert info["variant"] % 10 == (7 if greg == "1" else 4)
    assert info["groups"] > 2 * info["grid"] * info["groups_per_cta"]     # slots reuse their workspace
    _compare(r, shifts, w.Z, llr, syn, w.max_iter, _sample(F_FULL))


def test_n3_100kb_full_batch(gpu):
    """The N3 stable profile at the paper's ~100 kb frame length (n = 102400, check degree 27-28:
    variant 8, 256 threads x 254 registers) on 4096 channel frames at QBER 1.75 %."""
    cols = [8] * 16 + [3] * 21 + [2] * 13
    shifts = synth.girth6_shifts(synth.peg_mask(8, cols, 7), 2048, 8)
    oc = oracle.Code(shifts, 2048)
    x, y, _ = synth.frames(oc.n, 0.0175, 211, 0, F_FULL)
    syn = oc.syndrome(x)
    llr = oc.build_llr(0.0175, y)
    r, code = _run(gpu, shifts, 2048, None, x, y, llr, syn, 50)
    info = code.launch_info(F_FULL)
    assert info["variant"] == 8 and info["groups"] > 4 * info["grid"] * info["groups_per_cta"]
    _compare(r, shifts, 2048, llr, syn, 50, _sample(F_FULL))
