#!/usr/bin/env python
"""Small decode launches of every decode-kernel variant, for compute-sanitizer.

  compute-sanitizer --tool racecheck python tools/sanitize_driver.py [--case NAME ...]

Each case builds a seeded code that selects one kernel variant (checked with launch_info), decodes a
few frames through the C ABI with early stop on and off, and compares the outputs with the oracle, so
a run that the sanitizer slows down still proves the same results.  The layered schedule's
synchronisation is what racecheck / synccheck look at: the per-slot named barrier between block rows
(PAPER.md:91-97 layered schedule, data dependencies between consecutive layers), the
double-buffered stopping flag and the per-frame refill hand-over.
  --errors : exercise the C-ABI error paths instead (memcheck: nothing may be touched on an error).
"""
from __future__ import annotations

import argparse
import os
import sys
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _code(Mb, Nb, Z, deg_row, seed):
    """Mb x Nb base matrix with deg_row non-zero blocks per block row (every column covered)."""
    rng = np.random.default_rng(seed)
    sh = -np.ones((Mb, Nb), np.int32)
    for I in range(Mb):
        cols = rng.choice(Nb, size=min(deg_row, Nb), replace=False)
        sh[I, cols] = rng.integers(0, Z, size=len(cols))
    for J in range(Nb):
        if (sh[:, J] < 0).all():
            sh[int(rng.integers(0, Mb)), J] = int(rng.integers(0, Z))
    return sh


# name -> (Mb, Nb, Z, row degree, frames, env, expected variant % 10)
CASES = {
    "v1_deg6": (4, 8, 64, 6, 9, {}, 1),                       # degree <= 8, E in smem, refill on
    "v1_norefill": (4, 8, 64, 6, 9, {"QKD_REFILL": "0"}, 1),
    "v2_deg18": (3, 24, 64, 18, 9, {}, 2),                    # degree <= 20, smem
    "v2_refill": (3, 24, 64, 18, 9, {"QKD_REFILL": "1"}, 2),
    "v3_deg40": (2, 44, 32, 40, 5, {}, 3),                    # generic, smem
    "v5_split": (3, 24, 64, 18, 9, {"QKD_SPLIT": "1"}, 5),    # lane-pair rows
    "v6_deg28": (3, 30, 64, 28, 9, {}, 6),                    # degree 21..32, smem
    "v7_long": (2, 34, 2048, 6, 5, {}, 7),                    # degree <= 8, E in global memory
    "v8_long": (2, 34, 2048, 20, 3, {}, 8),                   # degree 9..32, E in global memory
    "v4_long_generic": (2, 34, 2048, 6, 3, {"QKD_NO_GREG": "1"}, 4),
}


def run_case(name, qkd, torch):
    import oracle
    Mb, Nb, Z, D, F, env, want = CASES[name]
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        sh = _code(Mb, Nb, Z, D, zlib.crc32(name.encode()))
        n, m = Nb * Z, Mb * Z
        rng = np.random.default_rng(zlib.crc32(("in/" + name).encode()))
        base = np.where(rng.random((F, n)) < 0.04, -1, 1) * 14
        wild = rng.integers(-127, 128, size=(F, n))
        llr = np.where(rng.random((F, n)) < 0.1, wild, base).astype(np.int8)
        syn = rng.integers(0, 256, size=(F, (m + 7) // 8), dtype=np.uint8)
        code = qkd.QCCode(sh, Z)
        v = code.launch_info(F)["variant"] % 10
        assert v == want, f"{name}: variant {v}, wanted {want}"
        oc = oracle.Code(sh, Z)
        for early in (1, 0):
            r = code.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(syn).cuda(), 4, bool(early),
                            want_state=True)
            torch.cuda.synchronize()
            o = oc.decode(llr, syn, 4, early, want_state=True)
            for k in ("bits", "iters", "success", "L", "E"):
                assert np.array_equal(r[k].cpu().numpy(), o[k]), f"{name}: {k} differs from the oracle"
        print(f"{name}: variant {v}, {F} frames, oracle-exact")
    finally:
        for k, val in saved.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val


def run_errors(qkd, torch):
    """C-ABI error paths: each call must fail with its documented code and write nothing."""
    sh = _code(2, 8, 64, 6, 7)
    code = qkd.QCCode(sh, 64)
    F = 4
    llr = torch.zeros((F, 8 * 64), dtype=torch.int8, device="cuda")
    syn = torch.zeros((F, 16), dtype=torch.uint8, device="cuda")
    bad = 0
    small = torch.empty(code.workspace_bytes(F) - 4, dtype=torch.uint8, device="cuda")
    for T, ws in ((4, small), (-1, None)):                 # QKD_EDIM (workspace too small), QKD_EINVAL
        try:
            code.decode(llr, syn, T, True, workspace=ws)
        except Exception as e:   # noqa: BLE001 -- any documented error is fine, it must not write
            bad += 1
            print("error path:", type(e).__name__, str(e)[:80])
    for shifts, Z in ((np.full((1, 70), 0, np.int32), 64), (sh, 0), (np.full((2, 3), 99, np.int32), 8)):
        try:
            qkd.QCCode(shifts, Z)
        except Exception as e:   # noqa: BLE001
            bad += 1
            print("error path:", type(e).__name__, str(e)[:80])
    torch.cuda.synchronize()
    assert bad == 5, f"expected 5 rejected calls, got {bad}"
    r = code.decode(llr, syn, 4, True, want_state=True)       # the handle still works afterwards
    torch.cuda.synchronize()
    assert int(r["iters"].max()) == 0
    print("error paths ok")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", nargs="*", default=list(CASES))
    ap.add_argument("--errors", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_1903_10107_b200 as qkd
    torch.cuda.set_device(0)
    if a.errors:
        run_errors(qkd, torch)
        return
    for c in a.case:
        run_case(c, qkd, torch)


if __name__ == "__main__":
    main()
