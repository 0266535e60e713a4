#!/usr/bin/env python
"""Interactive rate-adaptive reconciliation on the C4 mother code (DESIGN R25).

  python tools/adaptive_sweep.py [--frames 4096] [--df 0.02] [--rounds 25] [--out gpurun_out/adaptive.json]

For each QBER of BASELINE configs[3] (1, 2, 4, 6, 8 %): frames start at the R19 pattern (f = 1.1);
every frame that fails has the next delta = ceil(df (n - d) h2(q)) punctured positions revealed
(shortened) and is decoded again from scratch, up to --rounds reveals (qkd_reconcile_adaptive).
Reports per QBER: frame error rate after the rounds, mean efficiency f of the reconciled frames,
mean reveal rounds, the wall time of the whole interactive reconciliation (CUDA events; since
round 2 the rounds are enqueued without host synchronisation) and the corrected-key Mbps = reconciled payload bits / time.
"""
from __future__ import annotations

import argparse
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


def h2(q):
    return -q * math.log2(q) - (1 - q) * math.log2(1 - q)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--df", type=float, default=0.02)
    ap.add_argument("--rounds", type=int, default=25)
    ap.add_argument("--qbers", default=",".join(f"{q:g}" for q in synth.C4_QBERS))
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for q in [float(v) for v in a.qbers.split(",")]:
        w = synth.workload(f"C4@{q:g}")
        d, p, s = w.rate_adaptive_counts()
        order = torch.from_numpy(w.reveal_order()).cuda()
        code = qkd.QCCode(w.shifts(), w.Z, w.pos_kind())
        x, y, _ = w.gen(0, a.frames)
        xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        syn = code.syndrome(xs)
        delta = int(math.ceil(a.df * (w.n - d) * h2(q)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        code.reconcile_adaptive(q, order, s, delta, a.rounds, ys[:8], xs[:8], syn[:8], w.max_iter)   # warm-up
        torch.cuda.synchronize()
        e0.record()
        r = code.reconcile_adaptive(q, order, s, delta, a.rounds, ys, xs, syn, w.max_iter)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        errs = code.score(r["bits"], xs, r["success"], want_errors=True)
        succ = r["success"].cpu().numpy().astype(bool)
        rounds = r["rounds"].cpu().numpy()
        nerr = errs["errors"].cpu().numpy() if isinstance(errs, dict) else errs.cpu().numpy()
        good = succ & (nerr == 0)
        s_k = np.minimum(s + rounds.astype(np.int64) * delta, d)
        f = (code.m - d + s_k) / ((w.n - d) * h2(q))
        payload = w.n - d
        row = dict(qber=q, frames=a.frames, delta=delta, max_rounds=a.rounds,
                   f_round0=float((code.m - d + s) / ((w.n - d) * h2(q))),
                   fer_round0=float(1 - (good & (rounds == 0)).mean()),
                   fer=float(1 - good.mean()), undetected=int((succ & (nerr > 0)).sum()),
                   mean_f_reconciled=float(f[good].mean()) if good.any() else None,
                   mean_rounds=float(rounds.mean()), ms=ms,
                   corrected_key_mbps=float(good.sum() * payload / (ms * 1e-3) / 1e6))
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(dict(config="C4 mother code 20x40 Z=2048 (n=81920), reserved d=36965, R19/R25", rows=rows),
                      fh, indent=1)


if __name__ == "__main__":
    main()
