#!/usr/bin/env python
"""Frame error rate of the product decoder on two constructions of the same degree profile (SURVEY
§8(f) N3): BASELINE's rule (Q17: uniform seeded shifts, no girth filter) vs a PEG base mask with
girth >= 6 shifts (synth.peg_qc_code).

  python tools/code_construction_sweep.py [--frames 4096] [--out gpurun_out/code_construction.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1903_10107_b200 as qkd  # noqa: E402
import synth  # noqa: E402

PROFILES = {   # name: (Mb, Nb, Z, degree fractions, QBERs, max iterations)
    "C1 (3,6)-regular": (6, 12, 64, {3: 1.0}, (0.05, 0.06, 0.07), 30),
    "C2 irregular R=1/2": (16, 32, 256, {2: 0.45, 3: 0.35, 8: 0.20}, (0.08, 0.085, 0.09), 50),
    "C3 irregular R=0.84": (8, 50, 1024, {2: 0.5, 3: 0.4, 6: 0.1}, (0.01, 0.015, 0.02), 50),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for name, (Mb, Nb, Z, fr, qbers, T) in PROFILES.items():
        codes = {"Q17 rule": synth.qc_code(Mb, Nb, Z, fr, 7), "PEG + girth>=6": synth.peg_qc_code(Mb, Nb, Z, fr, 7)}
        for q in qbers:
            x, y, _ = synth.frames(Nb * Z, q, 303, 0, a.frames)
            row = dict(profile=name, n=Nb * Z, qber=q, frames=a.frames)
            for cname, sh in codes.items():
                code = qkd.QCCode(sh, Z)
                xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
                syn = code.syndrome(xs)
                r = code.decode(code.build_llr(q, ys), syn, T, True)
                err = code.score(r["bits"], xs, r["success"], want_errors=True).cpu().numpy()
                ok = (r["success"].cpu().numpy() == 1) & (err == 0)
                row[f"{cname} FER"] = float(1 - ok.mean())
                row[f"{cname} mean iters"] = float(r["iters"].float().mean().item())
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
