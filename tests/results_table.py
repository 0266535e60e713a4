#!/usr/bin/env python
"""BASELINE.md §4 results table: every BASELINE config at its configured batch on one B200.

  python tests/results_table.py [--out gpurun_out/results_table.json] [--reps 5] [--check 64]
                                [--oracle-seconds 3]

Lives under tests/ because it runs the oracle (bit-exactness of spread frames, oracle Mbps): only
test infrastructure may execute oracle/ (DESIGN §4).

Per workload (C1 64 frames, C2 1024, C3 4096, C4 at each QBER 4096, C5a/C5b 65536):
  * the whole hot path (syndrome a3, LLR a2, decode a4-a8, score a9) timed with CUDA events on the
    launching stream, inputs resident in HBM (min and median of --reps steps), plus the decode alone;
  * FER, mean iterations, f (R20: (m - p) / ((n - p - s) h(q))), processed-key Mbps (frames x payload
    bits / step time), corrected-key Mbps (frames decoded to Alice's key x payload bits / step time);
  * HBM roofline fraction of the decode (SURVEY §8(d) algorithmic bytes / decode time / measured peak);
  * bit-exactness: --check frames spread over the batch (first, last, and evenly between) compared with
    the oracle in bits, iterations and success;
  * the oracle's own Mbps on a bounded sample (1 thread and all host cores; test infrastructure,
    like bench.py's cpu_baseline leg).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_10107_b200 as qkd  # noqa: E402
import synth  # noqa: E402

NAMES = ["C1", "C2", "C3"] + [f"C4@{q:g}" for q in synth.C4_QBERS] + ["C5a", "C5b"]


def efficiency(w):
    d, p, s = w.rate_adaptive_counts()
    q = w.qber
    h2 = -q * math.log2(q) - (1 - q) * math.log2(1 - q)
    return (w.m - p) / ((w.n - p - s) * h2)


def payload(w):
    d, p, s = w.rate_adaptive_counts()
    return w.n - p - s


def hbm_peak():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        return float(json.load(f)["hbm_gbs"])


def run(name, reps, check, oracle_s, peak):
    w = synth.workload(name)
    F = w.frames
    kind = w.pos_kind()
    code = qkd.QCCode(w.shifts(), w.Z, kind)
    x, y, _ = w.gen(0, F, os.cpu_count())
    xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    known = xs if kind is not None else None
    syn = torch.empty((F, code.mb8), dtype=torch.uint8, device="cuda")
    llr = torch.empty((F, code.n), dtype=torch.int8, device="cuda")
    ws = torch.empty(code.workspace_bytes(F), dtype=torch.uint8, device="cuda")
    out = dict(bits=torch.empty((F, code.nb8), dtype=torch.uint8, device="cuda"),
               iters=torch.empty(F, dtype=torch.int32, device="cuda"),
               success=torch.empty(F, dtype=torch.uint8, device="cuda"))
    cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    step_ms, dec_ms = [], []
    for i in range(reps + 2):
        cnt.zero_()
        a, b, c, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        torch.cuda.synchronize()
        a.record(st)
        code.syndrome(xs, out=syn)
        code.build_llr(w.qber, ys, known, out=llr)
        b.record(st)
        code.decode(llr, syn, w.max_iter, True, counters=cnt, workspace=ws, out=out)
        c.record(st)
        code.score(out["bits"], xs, out["success"], counters=cnt)
        d.record(st)
        torch.cuda.synchronize()
        if i >= 2:                                       # two warm-up steps
            step_ms.append(a.elapsed_time(d))
            dec_ms.append(b.elapsed_time(c))
    c5 = cnt.cpu().numpy()
    iters = out["iters"].cpu().numpy().astype(np.int64)
    once = code.n + code.mb8 + code.nb8 + 5
    alg = float(iters.sum() * 2 * code.n_edges + F * once)
    corrected = int(c5[1] - c5[3])
    t_step = min(step_ms) * 1e-3
    row = dict(workload=name, frames=F, qber=w.qber, T=w.max_iter, n=code.n, payload_bits=payload(w),
               f=round(efficiency(w), 4), FER=1.0 - corrected / F, successes=int(c5[1]),
               undetected=int(c5[3]), mean_iters=float(iters.mean()),
               step_ms_min=min(step_ms), step_ms_median=statistics.median(step_ms),
               decode_ms_min=min(dec_ms), decode_share=min(dec_ms) / min(step_ms),
               processed_mbps=F * payload(w) / t_step / 1e6,
               corrected_mbps=corrected * payload(w) / t_step / 1e6,
               decode_alg_GBps=alg / (min(dec_ms) * 1e-3) / 1e9,
               hbm_frac=alg / (min(dec_ms) * 1e-3) / 1e9 / peak,
               launch=code.launch_info(F))
    if check:
        import oracle
        idx = np.unique(np.concatenate([[0, F - 1], np.linspace(0, F - 1, min(check, F)).astype(np.int64)]))
        oc = oracle.Code(w.shifts(), w.Z)
        xo, yo = x[idx], y[idx]
        o = oc.decode(oc.build_llr(w.qber, yo, kind, xo if kind is not None else None), oc.syndrome(xo),
                      w.max_iter, 1, want_state=False, nthreads=os.cpu_count())
        ok = all(np.array_equal(out[k].cpu().numpy()[idx], o[k]) for k in ("bits", "iters", "success"))
        row["bit_exact"] = f"{len(idx)} spread frames {'bit-exact' if ok else 'MISMATCH'}"
    if oracle_s > 0:
        import oracle
        oc = oracle.Code(w.shifts(), w.Z)
        per_frame = float(np.mean(iters)) * code.n_edges * 3.5e-8 + 1e-5       # rough, to size the sample
        for label, nth in (("1T", 1), ("all", os.cpu_count())):
            k = int(max(nth, min(F, round(oracle_s * nth / per_frame))))
            xo, yo = x[:k], y[:k]
            t0 = time.perf_counter()
            llo = oc.build_llr(w.qber, yo, kind, xo if kind is not None else None)
            so = oc.syndrome(xo)
            o = oc.decode(llo, so, w.max_iter, 1, want_state=False, nthreads=nth)
            dt = time.perf_counter() - t0
            row[f"oracle_mbps_{label}"] = k * payload(w) / dt / 1e6
            row[f"oracle_sample_{label}"] = k
        row["oracle_cores"] = os.cpu_count()
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default=",".join(NAMES))
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "results_table.json"))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", type=int, default=64)
    ap.add_argument("--oracle-seconds", type=float, default=3.0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    peak = hbm_peak()
    rows = []
    for name in a.workloads.split(","):
        r = run(name, a.reps, a.check, a.oracle_seconds, peak)
        print(json.dumps(r), flush=True)
        rows.append(r)
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(dict(peak_GBps=peak, gpu=torch.cuda.get_device_name(0), rows=rows), open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
