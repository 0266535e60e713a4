#!/usr/bin/env python
"""Quantized (improved RCBP + saturation, the product path) vs exact floating-point BP (layered, and
flooding: SURVEY §8(f) N4) on the same
frames ("maintain the high efficiency as the floating-point version").

  python tools/float_vs_quant.py [--frames 4096] [--out gpurun_out/float_vs_quant.json]

For each (code, QBER) point: frame error rate (syndrome not matched, or matched with payload errors),
mean iterations, and decode time of both decoders on identical BSC frames.  Codes: BASELINE configs[0]
(C1) and configs[1] (C2) at and around their QBERs, and the C4 mother code unpunctured at 6 % and 8 %
(SURVEY §8(d) diagnostic points, f = 1.527 / 1.243), plus the best stable rate-0.84 profile of N3
(profiles/r1_degree_profiles.md) at 1.5 / 1.75 / 2 % (f = 1.42 / 1.26 / 1.13).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_10107_b200 as qkd  # noqa: E402
import synth  # noqa: E402

POINTS = [("C1", 0.04), ("C1", 0.05), ("C1", 0.06), ("C2", 0.06), ("C2", 0.07), ("C2", 0.08), ("C2", 0.09),
          ("C4mother", 0.06), ("C4mother", 0.08), ("N3best", 0.015), ("N3best", 0.0175), ("N3best", 0.02)]


class _N3Best:
    """The best stable rate-0.84 profile of profiles/r1_degree_profiles.md (n = 51200, check degree 27-28)."""
    Z, n, max_iter = 1024, 51200, 50

    def __init__(self, q):
        self.qber = q
        cols = [8] * 16 + [3] * 21 + [2] * 13
        self._sh = synth.girth6_shifts(synth.peg_mask(8, cols, 7), 1024, 8)

    def shifts(self):
        return self._sh

    def gen(self, f0, F):
        return synth.frames(self.n, self.qber, 203, f0, F)


def workload(name, q):
    if name == "N3best":
        return _N3Best(q)
    if name == "C4mother":
        w = synth.workload("C4@0.06")
        w.rate_adaptive = False          # unpunctured mother code (diagnostic point)
    else:
        w = synth.workload(name)
    w.qber = q
    return w


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for name, q in POINTS:
        w = workload(name, q)
        F = a.frames if w.n <= 8192 else a.frames // 4
        code = qkd.QCCode(w.shifts(), w.Z)
        x, y, _ = w.gen(0, F)
        xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        syn = code.syndrome(xs)
        res = {}
        for kind in ("quantized", "float", "float_flooding"):
            if kind == "quantized":
                llr = code.build_llr(q, ys)
                run = lambda: code.decode(llr, syn, w.max_iter, True)          # noqa: E731
            else:
                llr = code.build_llr_float(q, ys)
                fl = kind == "float_flooding"
                run = lambda: code.decode_float(llr, syn, w.max_iter, True, flooding=fl)    # noqa: E731
            run()
            torch.cuda.synchronize()
            r, ms = timed(run)
            err = code.score(r["bits"], xs, r["success"], want_errors=True).cpu().numpy()
            succ = r["success"].cpu().numpy().astype(bool)
            it = r["iters"].cpu().numpy()
            res[kind] = dict(fer=float(1 - (succ & (err == 0)).mean()), undetected=int((succ & (err > 0)).sum()),
                             mean_iters=float(it.mean()), ms=ms,
                             mbps_processed=float(F * w.n / (ms * 1e-3) / 1e6))
        both = dict(code=name, qber=q, n=w.n, frames=F, **{f"{k}_{m}": v for k, d in res.items() for m, v in d.items()})
        rows.append(both)
        print(json.dumps(both), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
