#!/usr/bin/env python
"""Density evolution of the product's quantized decoder and a degree-profile search.

PAPER.md:155: "The check and variable node degree distributions are both irregular and optimized using
the Density Evolution (DE) algorithm".  The paper's profiles are not published, so this tool runs DE on
the decoder the product actually implements -- int8 channel LLRs of magnitude round(4 ln((1-q)/q)),
check-to-variable messages in [-63, 63] combined by Algorithm 1's tau along the forward /
backward schedule of DESIGN R6, variable-to-check messages min(|x|, 63) with x = E - L_ij --
over the ensemble of a QC base matrix's degree profile, and searches integer column-degree counts of
an Mb x Nb base matrix (rate 1 - Mb/Nb fixed) for the highest DE threshold.

Exactness notes (the approximations DE makes, stated):
  * flooding DE stands in for the layered schedule (same fixed points; layered converges ~2x faster, so
    the T-iteration layered decoder is compared with 2T flooding DE iterations);
  * the int8 clamp of E at +-127 does not change min(|x|, 63) (|L| <= 63), so the variable-to-check
    message is exactly clamp(LLR + sum of the other incoming L, -63, 63); Algorithm 2's guard (a
    saturated E is never updated) is not modelled;
  * "converged" = the variable-to-check error probability falls below 1e-6 (the quantized decoder has
    a floor: chains of tau shrink even perfect messages by up to 2 per combination, so the error
    probability settles near 1e-7 instead of 0; at n = 51200 that is < 0.05 bit errors per frame);
  * the all-zero error pattern is assumed (the syndrome decoder is symmetric in the coset: BSC
    symmetry), and the edges of a degree-D row sit at every position of the F/B fold with equal
    probability (the PEG mask orders a row's columns arbitrarily).

  python tools/de_search.py threshold --counts 2:13,3:21,8:16 --mb 8
  python tools/de_search.py search --mb 8 --nb 50 --degrees 2,3,4,5,6,7,8 --start 2:13,3:21,8:16
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

MSG = 63                         # MSG_max: check messages in [-63, 63]
NV = 2 * MSG + 1                 # values -63..63, index v + 63


def tau(p: int, q: int) -> int:
    """Algorithm 1, restated."""
    a, b = min(p, MSG), min(q, MSG)
    g, l = max(a, b), min(a, b)
    d = g - l
    if l > 2:
        return l - (d < 2) - (d < 6)
    return max(l - (d < 4), 0)


def combine_index() -> np.ndarray:
    """out[a, b] = index of sign(a) sign(b) tau(|a|, |b|) for a, b in -63..63 (a zero magnitude gives
    a zero output, whose sign is immaterial)."""
    v = np.arange(-MSG, MSG + 1)
    T = np.array([[tau(i, j) for j in range(MSG + 1)] for i in range(MSG + 1)])
    mag = T[np.abs(v)[:, None], np.abs(v)[None, :]]
    sgn = np.where(v > 0, 1, -1)
    out = sgn[:, None] * sgn[None, :] * mag
    return (out + MSG).ravel()


OUT = combine_index()


def cnode(Pa: np.ndarray, Pb: np.ndarray) -> np.ndarray:
    """Distribution of the pairwise check combination of two independent messages."""
    return np.bincount(OUT, weights=np.outer(Pa, Pb).ravel(), minlength=NV)


def check_out(P: np.ndarray, D: int) -> np.ndarray:
    """Check-to-variable distribution of a degree-D row with i.i.d. inputs P, averaged over the D
    positions of the F/B leave-one-out (R6: F_k = tau(F_{k-1}, m_k), B_k = tau(m_k, B_{k+1}),
    o_k = tau(F_{k-1}, B_{k+1}); with i.i.d. inputs dist(B_k) = dist(F_{D-1-k}))."""
    if D == 1:
        out = np.zeros(NV); out[MSG + MSG] = 1.0          # empty box-plus -> +MSG_max (R6)
        return out
    F = [P]
    for _ in range(1, D - 1):
        F.append(cnode(F[-1], P))                           # F_0 .. F_{D-2}
    acc = F[D - 2] * 2.0                                    # o_0 = B_1 ~ F_{D-2}, o_{D-1} = F_{D-2}
    for k in range(1, D - 1):
        acc += cnode(F[k - 1], F[D - 2 - k])                # o_k = tau(F_{k-1}, B_{k+1}), B_{k+1} ~ F_{D-2-k}
    return acc / D


def var_out(Q: np.ndarray, dv: int, Lq: int, q: float) -> np.ndarray:
    """Variable-to-check distribution of a degree-dv column: clamp(LLR + sum of dv-1 messages, +-63)."""
    s = np.array([1.0])
    for _ in range(dv - 1):
        s = np.convolve(s, Q)
    off = (dv - 1) * MSG                                    # s[i] is the value i - off
    vals = np.arange(len(s)) - off
    out = np.zeros(NV)
    for llr, w in ((Lq, 1.0 - q), (-Lq, q)):
        x = np.clip(vals + llr, -MSG, MSG) + MSG
        out += w * np.bincount(x, weights=s, minlength=NV)
    return out


def profile(counts: dict[int, int], Mb: int):
    """Edge-perspective (lambda, rho) of a base matrix with `counts` columns of each degree and rows
    as uniform as possible (PEG balances check degrees)."""
    E = sum(d * n for d, n in counts.items())
    lam = {d: d * n / E for d, n in counts.items() if n}
    lo, r = divmod(E, Mb)
    rows = {lo: Mb - r} if r == 0 else {lo: Mb - r, lo + 1: r}
    rho = {D: D * m / E for D, m in rows.items() if m}
    return lam, rho, E


def run_de(counts: dict[int, int], Mb: int, q: float, iters: int, tol: float = 1e-6):
    """Returns (converged, iterations, final bit error probability of the variable-to-check messages)."""
    lam, rho, E = profile(counts, Mb)
    Lq = min(127, int(math.floor(4.0 * math.log((1 - q) / q) + 0.5)))
    Q = np.zeros(NV); Q[MSG] = 1.0                          # first iteration: L = 0
    pe = 1.0
    for t in range(iters):
        P = sum(w * var_out(Q, d, Lq, q) for d, w in lam.items())
        P /= P.sum()                                        # rounding drift grows ~D dv per iteration
        pe = P[:MSG].sum() + 0.5 * P[MSG]
        if pe < tol:
            return True, t, pe
        Q = sum(w * check_out(P, D) for D, w in rho.items())
        Q /= Q.sum()
    return False, iters, pe


def threshold(counts, Mb, iters, lo=0.010, hi=0.030, steps=9):
    """Largest QBER (bisection on [lo, hi]) at which DE converges within `iters` iterations."""
    ok, _, _ = run_de(counts, Mb, lo, iters)
    if not ok:
        return lo
    for _ in range(steps):
        mid = 0.5 * (lo + hi)
        if run_de(counts, Mb, mid, iters)[0]:
            lo = mid
        else:
            hi = mid
    return lo


def parse_counts(s: str) -> dict[int, int]:
    return {int(a): int(b) for a, b in (x.split(":") for x in s.split(","))}


def fmt(c):
    return ",".join(f"{d}:{n}" for d, n in sorted(c.items()) if n)


def search(Mb, Nb, degrees, start, iters, budget_s, log):
    """Greedy local search over integer column-degree counts (sum Nb): move one column from degree a
    to degree b, keep the move that raises the threshold most; stop at a local optimum."""
    cur = {d: start.get(d, 0) for d in degrees}
    assert sum(cur.values()) == Nb, "start counts must sum to Nb"
    best = threshold(cur, Mb, iters)
    log({"counts": fmt(cur), "threshold": best, "step": "start"})
    t0 = time.time()
    seen = {fmt(cur)}
    while time.time() - t0 < budget_s:
        cands = []
        for a in degrees:
            for b in degrees:
                if a == b or cur[a] == 0:
                    continue
                for k in (1, 2):
                    if cur[a] < k:
                        continue
                    c = dict(cur); c[a] -= k; c[b] += k
                    if c.get(2, 0) > 2 * Mb + 4:                 # degree-2 columns beyond a few cycles' worth
                        continue
                    key = fmt(c)
                    if key in seen:
                        continue
                    seen.add(key)
                    cands.append(c)
        scored = []
        for c in cands:
            th = threshold(c, Mb, iters, lo=max(0.01, best - 0.002))
            scored.append((th, c))
            log({"counts": fmt(c), "threshold": th})
            if time.time() - t0 > budget_s:
                break
        if not scored:
            break
        th, c = max(scored, key=lambda x: x[0])
        if th <= best:
            break
        best, cur = th, c
        log({"counts": fmt(cur), "threshold": best, "step": "accept"})
    return cur, best


def _grid_one(args):
    c, Mb, iters = args
    return fmt(c), threshold(c, Mb, iters)


def grid(Mb, Nb, two, his, nhis, fours, iters, procs, log):
    """Threshold of every profile {2: n2, 3: rest, 4: n4, hi: n_hi} of the grid (process pool)."""
    from multiprocessing import Pool
    jobs = []
    for n2 in two:
        for hi in his:
            for nh in nhis:
                for n4 in fours:
                    n3 = Nb - n2 - nh - n4
                    if n3 < 0:
                        continue
                    c = {2: n2, 3: n3, 4: n4, hi: nh}
                    jobs.append(({k: v for k, v in c.items() if v}, Mb, iters))
    best = (0.0, None)
    with Pool(procs) as pool:
        for key, th in pool.imap_unordered(_grid_one, jobs):
            log({"counts": key, "threshold": th})
            best = max(best, (th, key))
    return best


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    a1 = sub.add_parser("threshold")
    a1.add_argument("--counts", required=True)
    a1.add_argument("--mb", type=int, default=8)
    a1.add_argument("--iters", type=int, default=100)
    a2 = sub.add_parser("search")
    a2.add_argument("--mb", type=int, default=8)
    a2.add_argument("--nb", type=int, default=50)
    a2.add_argument("--degrees", default="2,3,4,5,6,7,8")
    a2.add_argument("--start", default="2:13,3:21,8:16")
    a2.add_argument("--iters", type=int, default=100)
    a2.add_argument("--budget", type=float, default=1800)
    a2.add_argument("--out", default=None)
    a3 = sub.add_parser("grid")
    a3.add_argument("--mb", type=int, default=16)
    a3.add_argument("--nb", type=int, default=100)
    a3.add_argument("--two", default="12,14,16,18,20,22,24")
    a3.add_argument("--hi", default="10,12,14,16")
    a3.add_argument("--nhi", default="4,6,8,10,12,14,16,18,20")
    a3.add_argument("--four", default="0")
    a3.add_argument("--iters", type=int, default=100)
    a3.add_argument("--procs", type=int, default=os.cpu_count())
    a3.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.cmd == "grid":
        out = open(a.out, "a") if a.out else None

        def glog(d):
            print(json.dumps(d), flush=True)
            if out:
                out.write(json.dumps(d) + "\n"); out.flush()
        ints = lambda s: [int(x) for x in s.split(",")]   # noqa: E731
        th, key = grid(a.mb, a.nb, ints(a.two), ints(a.hi), ints(a.nhi), ints(a.four), a.iters, a.procs, glog)
        glog({"best": key, "threshold": th})
        return
    if a.cmd == "threshold":
        c = parse_counts(a.counts)
        t0 = time.time()
        th = threshold(c, a.mb, a.iters)
        lam, rho, E = profile(c, a.mb)
        print(json.dumps({"counts": fmt(c), "Mb": a.mb, "edges": E, "rho": rho, "threshold": th,
                          "f_at_threshold": (a.mb / sum(c.values())) / (-th * math.log2(th) - (1 - th) * math.log2(1 - th)),
                          "seconds": round(time.time() - t0, 1)}))
        return
    out = open(a.out, "a") if a.out else None

    def log(d):
        print(json.dumps(d), flush=True)
        if out:
            out.write(json.dumps(d) + "\n"); out.flush()
    degs = [int(x) for x in a.degrees.split(",")]
    cur, best = search(a.mb, a.nb, degs, parse_counts(a.start), a.iters, a.budget, log)
    log({"final": fmt(cur), "threshold": best})


if __name__ == "__main__":
    main()
