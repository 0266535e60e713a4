#!/usr/bin/env python
"""Codes from density-evolution profiles (tools/de_search.py), decoded by the product on the GPU:
frame error rate against QBER.

  python tools/de_codes.py --profile "16,100,512;2:10,3:66,12:24" [--profile ...] \
      [--qbers 0.015,0.016,...] [--frames 4096] [--out gpurun_out/de_codes.json]

Each profile "Mb,Nb,Z;d:count,..." is built as synth.peg_qc_code builds codes (PEG base mask,
P:155 / Hu et al., then girth >= 6 circulant shifts), seed 7; frames are the seeded BSC frames of
synth.frames (C3's data seed 203, so the rate-0.84 codes see the same channel draws at every QBER);
the decoder is the product (T = 50, early stop, int8 LLRs at the frame's QBER).  f = (Mb / Nb) / h(q)
(R20, no puncturing).  --float adds exact floating-point BP (N1) on the same frames: the BP
waterfall of the profile, against which the quantized decoder's loss is read.  Parity of such codes
against the oracle: tests/test_gpu_parity.py.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_10107_b200 as qkd  # noqa: E402
import synth  # noqa: E402


def h2(q):
    return -q * math.log2(q) - (1 - q) * math.log2(1 - q)


def build(Mb: int, Nb: int, Z: int, counts: dict[int, int], seed: int = 7) -> np.ndarray:
    cols = [d for d in sorted(counts, reverse=True) for _ in range(counts[d])]
    assert len(cols) == Nb, "column counts must sum to Nb"
    return synth.girth6_shifts(synth.peg_mask(Mb, cols, seed), Z, seed + 1)


def parse(spec: str):
    dims, cnt = spec.split(";")
    Mb, Nb, Z = (int(v) for v in dims.split(","))
    return Mb, Nb, Z, {int(a): int(b) for a, b in (x.split(":") for x in cnt.split(","))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", action="append", required=True)
    ap.add_argument("--qbers", default="0.015,0.016,0.017,0.018,0.019,0.02,0.021")
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--T", type=int, default=50)
    ap.add_argument("--float", action="store_true", help="also exact floating-point BP (N1, qkd_decode_float_batch)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for spec in a.profile:
        Mb, Nb, Z, counts = parse(spec)
        t0 = time.time()
        sh = build(Mb, Nb, Z, counts)
        code = qkd.QCCode(sh, Z)
        n = Nb * Z
        rd = (sh >= 0).sum(axis=1)
        for q in (float(v) for v in a.qbers.split(",")):
            x, y, _ = synth.frames(n, q, 203, 0, a.frames)
            xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
            syn = code.syndrome(xs)
            llr = code.build_llr(q, ys)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = code.decode(llr, syn, a.T, True)
            e1.record()
            torch.cuda.synchronize()
            err = code.score(r["bits"], xs, r["success"], want_errors=True).cpu().numpy()
            succ = r["success"].cpu().numpy() == 1
            ok = succ & (err == 0)
            row = dict(profile=spec, n=n, rate=1 - Mb / Nb, row_degrees=[int(rd.min()), int(rd.max())],
                       variant=code.launch_info(a.frames)["variant"], qber=q, f=(Mb / Nb) / h2(q),
                       frames=a.frames, fer=float(1 - ok.mean()), undetected=int((succ & (err > 0)).sum()),
                       mean_iters=float(r["iters"].float().mean().item()), decode_ms=e0.elapsed_time(e1),
                       build_s=round(time.time() - t0, 1))
            if a.float:
                lf = code.build_llr_float(q, ys)
                rf = code.decode_float(lf, syn, a.T, True)
                torch.cuda.synchronize()
                ef = code.score(rf["bits"], xs, rf["success"], want_errors=True).cpu().numpy()
                sf = rf["success"].cpu().numpy() == 1
                row.update(fer_float=float(1 - (sf & (ef == 0)).mean()),
                           mean_iters_float=float(rf["iters"].float().mean().item()))
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
