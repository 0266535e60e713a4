#!/usr/bin/env python
"""Stable degree profiles for the C3 code family ("stable degree profiles"; F5).

  python tools/profile_search.py [--frames 1024] [--confirm 4096] [--out gpurun_out/profile_search.json]

C3 keeps n = 51200, rate 0.84 (base 8 x 50, Z = 1024, f = 1.131 at QBER 2 %), but its Q17 column-degree
profile {2: 25, 3: 20, 6: 5} violates the BP stability condition lambda_2 rho'(1) < 1/B (B = 2 sqrt(q(1-q)),
the BSC Bhattacharyya parameter): every frame fails at 1.5-2 % (profiles/r1_code_construction.md).  This
sweep keeps the base size and lifting and varies the column degrees (n2 degree-2 columns, n_hi columns of
degree d_hi, the rest degree 3), builds each code with the PEG mask + girth >= 6 shifts of
synth.peg_qc_code, and measures the frame error rate of the product decoder (T = 50, early stop) on the
same seeded BSC frames at QBER 1.5 / 1.75 / 2 %.  The best profiles are re-measured on --confirm frames.
Per profile it also prints the stability margin lambda_2 rho'(1) * B (< 1 is stable at that QBER) with
the edge-perspective lambda_2 = 2 n2 / E and rho'(1) = sum_i rho_i (i - 1) from the actual row degrees.
"""
from __future__ import annotations

import argparse
import itertools
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_10107_b200 as qkd  # noqa: E402
import synth  # noqa: E402

MB, NB, Z = 8, 50, 1024
QBERS = (0.015, 0.0175, 0.02)


def set_z(z: int) -> None:
    global Z
    Z = z


def h2(q):
    return -q * math.log2(q) - (1 - q) * math.log2(1 - q)


def stability(shifts: np.ndarray, q: float) -> float:
    mask = shifts >= 0
    E = int(mask.sum())
    n2 = int((mask.sum(axis=0) == 2).sum())
    lam2 = 2 * n2 / E
    rd = mask.sum(axis=1)
    rho1 = float(sum(d * (d - 1) for d in rd) / E)          # sum_i rho_i (i - 1), rho_i = edge fraction
    return lam2 * rho1 * 2 * math.sqrt(q * (1 - q))


def build(n2: int, d_hi: int, n_hi: int, seed: int) -> np.ndarray:
    cols = [d_hi] * n_hi + [3] * (NB - n2 - n_hi) + [2] * n2
    return synth.girth6_shifts(synth.peg_mask(MB, cols, seed), Z, seed + 1)


def measure(shifts: np.ndarray, F: int, frames: dict) -> dict:
    code = qkd.QCCode(shifts, Z)
    out = {}
    for q in QBERS:
        xs, ys = frames[(q, F)]
        syn = code.syndrome(xs)
        r = code.decode(code.build_llr(q, ys), syn, 50, True)
        err = code.score(r["bits"], xs, r["success"], want_errors=True).cpu().numpy()
        ok = (r["success"].cpu().numpy() == 1) & (err == 0)
        out[q] = dict(fer=float(1 - ok.mean()), mean_iters=float(r["iters"].float().mean().item()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=1024)
    ap.add_argument("--confirm", type=int, default=4096)
    ap.add_argument("--top", type=int, default=4)
    ap.add_argument("--out", default=None)
    ap.add_argument("--z", type=int, default=Z, help="lifting size (1024: n = 51200; 2048: the paper's ~100 kb)")
    ap.add_argument("--only", default=None, help="n2,d_hi,n_hi: measure one profile on --confirm frames")
    a = ap.parse_args()
    if a.z != Z:
        set_z(a.z)
    if a.only:
        n2, d_hi, n_hi = (int(v) for v in a.only.split(","))
        frames = {}
        for q in QBERS:
            x, y, _ = synth.frames(NB * Z, q, 203, 0, a.confirm)
            frames[(q, a.confirm)] = (torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        sh = build(n2, d_hi, n_hi, 7)
        res = measure(sh, a.confirm, frames)
        print(json.dumps(dict(n=NB * Z, n2=n2, d_hi=d_hi, n_hi=n_hi, frames=a.confirm,
                              variant=qkd.QCCode(sh, Z).launch_info(a.confirm)["variant"],
                              **{f"fer_{q:g}": res[q]["fer"] for q in QBERS},
                              **{f"iters_{q:g}": res[q]["mean_iters"] for q in QBERS})), flush=True)
        return
    frames = {}
    for q in QBERS:
        for F in (a.frames, a.confirm):
            x, y, _ = synth.frames(NB * Z, q, 203, 0, F)
            frames[(q, F)] = (torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    rows = []
    grid = [(25, 6, 5)] + list(itertools.product((0, 4, 7, 10, 13, 16, 20), (4, 5, 6, 8), (3, 5, 8, 12)))
    grid += list(itertools.product((0, 4, 7, 10, 13), (6, 7, 8), (16, 20, 25, 30, 35)))
    for n2, d_hi, n_hi in grid:
        if n2 + n_hi > NB:
            continue
        try:
            sh = build(n2, d_hi, n_hi, 7)
        except Exception as e:   # girth-6 placement impossible for this mask
            print(json.dumps(dict(n2=n2, d_hi=d_hi, n_hi=n_hi, error=str(e))), flush=True)
            continue
        res = measure(sh, a.frames, frames)
        mask = sh >= 0
        row = dict(n2=n2, d_hi=d_hi, n_hi=n_hi, n3=NB - n2 - n_hi, base_edges=int(mask.sum()),
                   row_degrees=sorted(set(mask.sum(axis=1).tolist())),
                   stability_2pct=stability(sh, 0.02), frames=a.frames,
                   **{f"fer_{q:g}": res[q]["fer"] for q in QBERS},
                   **{f"iters_{q:g}": res[q]["mean_iters"] for q in QBERS})
        rows.append(row)
        print(json.dumps(row), flush=True)
    key = lambda r: tuple(r[f"fer_{q:g}"] for q in reversed(QBERS))   # noqa: E731  best at 2 %, then 1.75 %, ...
    best = sorted(rows, key=key)[: a.top]
    confirmed = []
    for r in best:
        sh = build(r["n2"], r["d_hi"], r["n_hi"], 7)
        res = measure(sh, a.confirm, frames)
        c = dict(n2=r["n2"], d_hi=r["d_hi"], n_hi=r["n_hi"], frames=a.confirm, base_edges=r["base_edges"],
                 row_degrees=r["row_degrees"], stability_2pct=r["stability_2pct"],
                 **{f"fer_{q:g}": res[q]["fer"] for q in QBERS},
                 **{f"iters_{q:g}": res[q]["mean_iters"] for q in QBERS},
                 **{f"f_{q:g}": MB * Z / (NB * Z * h2(q)) for q in QBERS})
        confirmed.append(c)
        print("confirm", json.dumps(c), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(dict(config=f"base {MB}x{NB}, Z={Z}, n={NB * Z}, rate {1 - MB / NB:.2f}, T=50, "
                                  "PEG + girth>=6, frames seed 203 (C3's)", sweep=rows, confirmed=confirmed),
                      fh, indent=1)


if __name__ == "__main__":
    main()
