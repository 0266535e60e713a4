"""Seeded synthetic workloads (inputs only) for the QKD LDPC decoder.

This module is the ONE piece shared by the oracle tests and the CUDA path's
tests/bench.  It contains no decoder arithmetic: it
builds QC base matrices, rate-adaptive position patterns and BSC frames, exactly
as SURVEY.md §8(c) Q17/Q18/Q19 and BASELINE.json `configs` describe.  Alice's
syndrome and Bob's LLRs are computed by each side itself.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            import _build  # repo root

            _build.build_synth()
        lib = ctypes.CDLL(_LIB_PATH)
        i32p = ctypes.POINTER(ctypes.c_int32)
        lib.synth_qc_code.argtypes = [ctypes.c_int32] * 4 + [i32p, i32p, ctypes.c_uint64, i32p]
        lib.synth_degree_counts.argtypes = [ctypes.c_int32, ctypes.c_int32, i32p, i32p, i32p]
        lib.synth_reserved_order.argtypes = [i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)]
        lib.synth_frames.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_int32]
        lib.synth_mix64.argtypes = [ctypes.c_uint64]
        lib.synth_mix64.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def _i32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def degree_counts(Nb: int, fracs: dict[int, float]) -> dict[int, int]:
    """Largest-remainder column-degree counts (Q17 step 1; ties to the lower degree)."""
    degs = np.array(sorted(fracs), dtype=np.int32)
    fe4 = np.array([int(round(fracs[d] * 10000)) for d in degs], dtype=np.int32)
    out = np.zeros(len(degs), dtype=np.int32)
    rc = _load().synth_degree_counts(Nb, len(degs), _i32(degs), _i32(fe4), _i32(out))
    if rc:
        raise ValueError("bad degree distribution")
    return {int(d): int(c) for d, c in zip(degs, out)}


def qc_code(Mb: int, Nb: int, Z: int, fracs: dict[int, float], seed: int) -> np.ndarray:
    """Seeded QC base matrix (Mb, Nb) int32, -1 = zero block (Q17)."""
    degs = np.array(sorted(fracs), dtype=np.int32)
    fe4 = np.array([int(round(fracs[d] * 10000)) for d in degs], dtype=np.int32)
    out = np.empty(Mb * Nb, dtype=np.int32)
    rc = _load().synth_qc_code(Mb, Nb, Z, len(degs), _i32(degs), _i32(fe4), seed, _i32(out))
    if rc:
        raise ValueError("synth_qc_code failed")
    return out.reshape(Mb, Nb)


def reserved_order(shifts: np.ndarray, Z: int, seed: int) -> np.ndarray:
    """All n variables by (column weight asc, seeded key) -- P:157 puncturing rule."""
    Mb, Nb = shifts.shape
    s = np.ascontiguousarray(shifts, dtype=np.int32).ravel()
    out = np.empty(Nb * Z, dtype=np.int64)
    rc = _load().synth_reserved_order(_i32(s), Mb, Nb, Z, seed,
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc:
        raise ValueError("synth_reserved_order failed")
    return out


def bsc_threshold(qber: float) -> int:
    """floor(q * 2^64) computed exactly from the decimal value of q."""
    return int(Fraction(repr(qber)) * (1 << 64))


def frames(n: int, qber: float, seed: int, f0: int, F: int, nthreads: int | None = None,
           want_y: bool = True, out_x: np.ndarray | None = None, out_y: np.ndarray | None = None):
    """BSC frames [f0, f0+F): returns (x, y, nerr); x, y are uint8 [F][ceil(n/8)] LSB-first."""
    nb = (n + 7) // 8
    x = out_x if out_x is not None else np.empty((F, nb), dtype=np.uint8)
    y = (out_y if out_y is not None else np.empty((F, nb), dtype=np.uint8)) if want_y else None
    nerr = np.empty(F, dtype=np.int32)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    assert x.flags.c_contiguous and x.shape == (F, nb)
    rc = _load().synth_frames(n, bsc_threshold(qber), seed, f0, F, x.ctypes.data,
                              y.ctypes.data if y is not None else None, nerr.ctypes.data, nthreads)
    if rc:
        raise ValueError("synth_frames failed")
    return x, y, nerr


def h2(q: float) -> float:
    return -q * math.log2(q) - (1 - q) * math.log2(1 - q)


# ---------------------------------------------------------------------------
# Workloads: BASELINE.json configs[0..4] with the seeds of SURVEY.md §8(d).
# ---------------------------------------------------------------------------
@dataclass
class Workload:
    name: str
    Mb: int
    Nb: int
    Z: int
    fracs: dict
    code_seed: int
    qber: float
    data_seed: int
    frames: int
    max_iter: int
    early_stop: int = 1
    rate_adaptive: bool = False   # C4: puncture/shorten for f = 1.1 (Q19)
    f_target: float = 1.1
    order_seed: int = 0
    _shifts: np.ndarray | None = field(default=None, repr=False)

    @property
    def n(self):
        return self.Nb * self.Z

    @property
    def m(self):
        return self.Mb * self.Z

    def shifts(self) -> np.ndarray:
        if self._shifts is None:
            self._shifts = qc_code(self.Mb, self.Nb, self.Z, self.fracs, self.code_seed)
        return self._shifts

    def rate_adaptive_counts(self) -> tuple[int, int, int]:
        """(reserved d, punctured p, shortened s) per Q19; (0,0,0) when not rate adaptive."""
        if not self.rate_adaptive:
            return 0, 0, 0
        n, m, f = self.n, self.m, self.f_target
        hq1 = h2(0.01)
        d = int(round((m - f * hq1 * n) / (1 - f * hq1)))
        p = int(round(m - f * h2(self.qber) * (n - d)))
        p = max(0, min(p, d))
        return d, p, d - p

    def pos_kind(self) -> np.ndarray | None:
        """uint8[n]: 0 payload, 1 punctured (LLR 0), 2 shortened (LLR +-127)."""
        if not self.rate_adaptive:
            return None
        d, p, s = self.rate_adaptive_counts()
        order = reserved_order(self.shifts(), self.Z, self.order_seed)
        kind = np.zeros(self.n, dtype=np.uint8)
        kind[order[:s]] = 2          # "shortened bits are selected in turn from the puncturing bits"
        kind[order[s:d]] = 1
        return kind

    def reveal_order(self) -> np.ndarray:
        """int32 [d]: the reserved positions in reveal order (shortened first, then punctured);
        interactive rounds shorten them in this order (DESIGN R25)."""
        d, p, s = self.rate_adaptive_counts()
        return reserved_order(self.shifts(), self.Z, self.order_seed)[:d].astype(np.int32)

    def gen(self, f0: int = 0, F: int | None = None, nthreads: int | None = None):
        F = self.frames if F is None else F
        return frames(self.n, self.qber, self.data_seed, f0, F, nthreads)


def _c1():
    return Workload("C1", 6, 12, 64, {3: 1.0}, 101, 0.05, 201, 64, 30)


def _c2():
    return Workload("C2", 16, 32, 256, {2: 0.45, 3: 0.35, 8: 0.20}, 102, 0.08, 202, 1024, 50)


def _c3():
    return Workload("C3", 8, 50, 1024, {2: 0.5, 3: 0.4, 6: 0.1}, 103, 0.02, 203, 4096, 50)


def _c4(qber: float, k: int):
    return Workload(f"C4@{qber:g}", 20, 40, 2048, {2: 0.45, 3: 0.35, 10: 0.20}, 104, qber, 204 + k,
                    4096, 60, rate_adaptive=True, order_seed=1104)


C4_QBERS = (0.01, 0.02, 0.04, 0.06, 0.08)


def workload(name: str) -> Workload:
    """C1, C2, C3, C4@<q> (q in 0.01..0.08), C5a (C3 code, 65536 frames), C5b (C2 code, 65536)."""
    if name == "C1":
        return _c1()
    if name == "C2":
        return _c2()
    if name == "C3":
        return _c3()
    if name.startswith("C4@"):
        q = float(name[3:])
        k = [round(v, 6) for v in C4_QBERS].index(round(q, 6))
        return _c4(q, k)
    if name == "C5a":
        w = _c3(); w.name = "C5a"; w.frames = 65536; return w
    if name == "C5b":
        w = _c2(); w.name = "C5b"; w.frames = 65536; return w
    raise KeyError(name)


ALL_PARITY_WORKLOADS = ["C1", "C2", "C3"] + [f"C4@{q:g}" for q in C4_QBERS] + ["C5a", "C5b"]


# ---------------------------------------------------------------------------
# Code construction: PEG base masks and girth >= 6 circulant shifts.
# P:155 "the girth of a LDPC code is at least 6 ... masking matrices are constructed by using
# standard PEG algorithm"; SPEC code-model peg_mask / girth_of / seeded shift retry.
# These build alternative codes; BASELINE's configs keep the Q17 rule (qc_code).
# ---------------------------------------------------------------------------
def peg_mask(Mb: int, col_degrees, seed: int = 0) -> np.ndarray:
    """Progressive edge growth on the base graph (Hu, Eleftheriou, Arnold): columns in non-decreasing
    degree order; each new edge of a column goes to a check outside its current BFS neighbourhood if
    one exists, else to a check at the largest BFS depth; ties by lowest check degree, then by a
    seeded order.  Returns a bool mask [Mb][Nb] (column J gets col_degrees[J] distinct checks)."""
    Nb = len(col_degrees)
    rng = np.random.default_rng(seed)
    tie = rng.permutation(Mb)                       # seeded tie order among equal-degree checks
    mask = np.zeros((Mb, Nb), dtype=bool)
    cdeg = np.zeros(Mb, dtype=np.int64)
    for J in sorted(range(Nb), key=lambda j: (col_degrees[j], j)):
        for e in range(int(col_degrees[J])):
            if e == 0:
                cand = np.arange(Mb)
            else:
                # BFS from variable J over the current Tanner graph (checks <-> variables)
                depth = np.full(Mb, -1)
                frontier_c = list(np.flatnonzero(mask[:, J]))
                for c in frontier_c:
                    depth[c] = 0
                seen_v = {J}
                d = 0
                while frontier_c:
                    nxt_v = {v for c in frontier_c for v in np.flatnonzero(mask[c]) if v not in seen_v}
                    seen_v |= nxt_v
                    d += 1
                    nxt_c = [c for v in nxt_v for c in np.flatnonzero(mask[:, v]) if depth[c] < 0]
                    nxt_c = sorted(set(nxt_c))
                    for c in nxt_c:
                        depth[c] = d
                    frontier_c = nxt_c
                free = np.flatnonzero((depth < 0) & ~mask[:, J])
                cand = free if len(free) else np.flatnonzero((depth == depth.max()) & ~mask[:, J])
            best = min(cand, key=lambda c: (cdeg[c], tie[c]))
            mask[best, J] = True
            cdeg[best] += 1
    return mask


def _creates_4cycle(sh: np.ndarray, Z: int, I: int, J: int, s: int) -> bool:
    """Would shift s at (I, J) close a 4-cycle with already assigned entries?  A cycle through rows
    I, I2 and columns J, J2 exists iff s(I,J) - s(I,J2) + s(I2,J2) - s(I2,J) = 0 mod Z."""
    Mb, Nb = sh.shape
    for J2 in range(Nb):
        if J2 == J or sh[I, J2] < 0:
            continue
        for I2 in range(Mb):
            if I2 == I or sh[I2, J] < 0 or sh[I2, J2] < 0:
                continue
            if (s - sh[I, J2] + sh[I2, J2] - sh[I2, J]) % Z == 0:
                return True
    return False


def girth6_shifts(mask: np.ndarray, Z: int, seed: int = 0, tries: int = 1000) -> np.ndarray:
    """Seeded uniform shifts in row-major order over the mask, each redrawn until it closes no 4-cycle
    with the entries already placed ("rejected and retried if girth < 6").  Raises if an
    entry cannot be placed in `tries` draws (Z too small for the mask)."""
    rng = np.random.default_rng(seed)
    sh = np.full(mask.shape, -1, dtype=np.int32)
    for I, J in zip(*np.nonzero(mask)):
        for _ in range(tries):
            s = int(rng.integers(0, Z))
            if not _creates_4cycle(sh, Z, I, J, s):
                sh[I, J] = s
                break
        else:
            raise ValueError(f"no 4-cycle-free shift for block ({I},{J}) with Z={Z}")
    return sh


def peg_qc_code(Mb: int, Nb: int, Z: int, fracs: dict[int, float], seed: int) -> np.ndarray:
    """Q17 degree counts (degree_counts), PEG mask, girth >= 6 shifts."""
    cnt = degree_counts(Nb, fracs)
    cols = [d for d in sorted(cnt, reverse=True) for _ in range(cnt[d])]
    return girth6_shifts(peg_mask(Mb, cols, seed), Z, seed + 1)
