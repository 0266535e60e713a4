#!/usr/bin/env python
"""Time (and, under ncu, profile) one decode workload in isolation.

  python tools/prof_decode.py [--workload C5a] [--frames 4736] [--reps 5]

Prints one JSON line per workload: mean/min decode ms over --reps launches (CUDA events on the
launching stream), algorithmic GB/s (per-frame iterations x 2|E| + once-bytes) and
the launch plan.  Under ncu use --reps 1.  (Parity of an A/B build: QKD_LIB=<lib> pytest tests -m gpu;
tools never run the oracle.)
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--frames", type=int, default=4736)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--max-iter", type=int, default=None)
    ap.add_argument("--early-stop", type=int, default=1, help="0: no per-iteration syndrome check (all T sweeps)")
    a = ap.parse_args()
    for name in a.workload.split(","):
        w = synth.workload(name)
        T = a.max_iter if a.max_iter is not None else w.max_iter
        code = qkd.QCCode(w.shifts(), w.Z, w.pos_kind())
        x, y, _ = w.gen(0, a.frames)
        xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        syn = code.syndrome(xs)
        llr = code.build_llr(w.qber, ys, xs if w.pos_kind() is not None else None)
        ws = torch.empty(code.workspace_bytes(a.frames), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream()
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = code.decode(llr, syn, T, bool(a.early_stop), workspace=ws)
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        iters = r["iters"].cpu().numpy().astype(np.int64)
        n_edges = code.n_edges
        once = code.n + code.mb8 + code.nb8 + 5
        alg = float(iters.sum() * 2 * n_edges + a.frames * once)
        t = min(times)
        out = dict(workload=name, frames=a.frames, T=T, early_stop=a.early_stop, ms_mean=sum(times) / len(times), ms_min=t,
                   alg_GBps=alg / (t * 1e-3) / 1e9, mean_iters=float(iters.mean()),
                   success=float(r["success"].float().mean().item()), launch=code.launch_info(a.frames))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
