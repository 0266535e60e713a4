"""ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper over oracle/liboracle.so, the plain scalar C oracle of the quantized
layered RCBP decoder (arXiv:1903.10107, §2-§3).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package.  It shares no code with paper_1903_10107_b200 (the CUDA product) and never
imports it; the product never imports this.

Parity status per function:
  tau, check_node, vn_update, decode, syndrome, llr_magnitude, build_llr, expand,
  efficiency -- pinned by tests/test_oracle_pins.py (paper examples, closed forms,
  invariants, brute-force ML on tiny codes, coset equivariance).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            import _build

            _build.build_oracle()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_code_create.argtypes = [_i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.orc_code_create.restype = _vp
        L.orc_code_destroy.argtypes = [_vp]
        for f in ("orc_code_n", "orc_code_m", "orc_code_edges"):
            getattr(L, f).argtypes = [_vp]
            getattr(L, f).restype = ctypes.c_int64
        L.orc_expand.argtypes = [_vp, _vp, _vp]
        L.orc_llr_magnitude.argtypes = [ctypes.c_double]
        L.orc_llr_magnitude.restype = ctypes.c_int
        L.orc_build_llr.argtypes = [ctypes.c_int64, ctypes.c_int, _vp, _vp, _vp, _vp]
        L.orc_syndrome.argtypes = [_vp, _vp, _vp]
        L.orc_tau.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_tau.restype = ctypes.c_int
        L.orc_check_node.argtypes = [ctypes.c_int, _vp, ctypes.c_int, _vp]
        L.orc_vn_update.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_vn_update.restype = ctypes.c_int
        L.orc_decode.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                 _vp, _vp, _vp, _vp, _vp]
        L.orc_decode_batch.argtypes = [_vp, ctypes.c_int64, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                       _vp, _vp, _vp, _vp, _vp, ctypes.c_int]
        L.orc_efficiency.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_double]
        L.orc_efficiency.restype = ctypes.c_double
        for f in ("orc_beta", "orc_beta_eq6"):
            getattr(L, f).argtypes = [ctypes.c_double, ctypes.c_double]
            getattr(L, f).restype = ctypes.c_double
        L.orc_check_node_float.argtypes = [ctypes.c_int, _vp, ctypes.c_int, _vp]
        L.orc_build_llr_float.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _vp]
        L.orc_decode_float_batch.argtypes = [_vp, ctypes.c_int64, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                             _vp, _vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def tau(p: int, q: int) -> int:
    """Algorithm 1."""
    return _load().orc_tau(int(p), int(q))


def llr_magnitude(q: float) -> int:
    """min(127, round(4 ln((1-q)/q))); -1 outside (0, 0.5)."""
    return _load().orc_llr_magnitude(float(q))


def check_node(x, s_i: int) -> list[int]:
    """One check row: exact inputs x_k = E - L_old -> new messages L_k (Eq.(1), Alg. 1, F/B)."""
    xa = np.ascontiguousarray(x, dtype=np.int32)
    out = np.zeros(len(xa), dtype=np.int32)
    _load().orc_check_node(len(xa), _p(xa), int(s_i), _p(out))
    return out.tolist()


def vn_update(E_before: int, x: int, Lnew: int) -> int:
    """Algorithm 2 + Eq.(9) with saturation."""
    return _load().orc_vn_update(int(E_before), int(x), int(Lnew))


def efficiency(m: int, n: int, p: int, s: int, q: float) -> float:
    return _load().orc_efficiency(int(m), int(n), int(p), int(s), float(q))


class Code:
    """Expanded QC code (oracle's own expansion of the base matrix)."""

    def __init__(self, shifts: np.ndarray, Z: int):
        shifts = np.ascontiguousarray(shifts, dtype=np.int32)
        self.Mb, self.Nb = shifts.shape
        self.Z = int(Z)
        self._h = _load().orc_code_create(shifts.ctypes.data_as(_i32p), self.Mb, self.Nb, self.Z)
        if not self._h:
            raise ValueError("invalid base matrix")
        L = _load()
        self.n = L.orc_code_n(self._h)
        self.m = L.orc_code_m(self._h)
        self.n_edges = L.orc_code_edges(self._h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_code_destroy(self._h)
            self._h = None

    def expand(self):
        rows = np.empty(self.n_edges, dtype=np.int64)
        cols = np.empty(self.n_edges, dtype=np.int64)
        _load().orc_expand(self._h, _p(rows), _p(cols))
        return rows, cols

    def syndrome(self, bits: np.ndarray) -> np.ndarray:
        """bits: uint8 [F][ceil(n/8)] or [ceil(n/8)] -> syndrome bytes, LSB-first."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        flat = b.reshape(-1, (self.n + 7) // 8)
        out = np.zeros((flat.shape[0], (self.m + 7) // 8), dtype=np.uint8)
        for f in range(flat.shape[0]):
            _load().orc_syndrome(self._h, _p(flat[f]), _p(out[f]))
        return out.reshape(b.shape[:-1] + (out.shape[1],))

    def build_llr(self, qber: float, y_bits: np.ndarray, kind: np.ndarray | None = None,
                  known_bits: np.ndarray | None = None) -> np.ndarray:
        Lq = llr_magnitude(qber)
        if Lq < 0:
            raise ValueError("qber outside (0, 0.5)")
        y = np.ascontiguousarray(y_bits, dtype=np.uint8).reshape(-1, (self.n + 7) // 8)
        kn = None if known_bits is None else np.ascontiguousarray(known_bits, dtype=np.uint8).reshape(y.shape)
        kd = None if kind is None else np.ascontiguousarray(kind, dtype=np.uint8)
        out = np.empty((y.shape[0], self.n), dtype=np.int8)
        for f in range(y.shape[0]):
            _load().orc_build_llr(self.n, Lq, _p(y[f]), _p(kd), None if kn is None else _p(kn[f]), _p(out[f]))
        return out

    def decode(self, llr: np.ndarray, syn: np.ndarray, max_iter: int, early_stop: int = 1,
               want_state: bool = True, nthreads: int | None = None, perm_seed: int = 0):
        """Batch decode. llr int8 [F][n], syn uint8 [F][ceil(m/8)].
        Returns dict(bits, iters, success, L, E)."""
        llr = np.ascontiguousarray(llr, dtype=np.int8).reshape(-1, self.n)
        F = llr.shape[0]
        syn = np.ascontiguousarray(syn, dtype=np.uint8).reshape(F, (self.m + 7) // 8)
        bits = np.zeros((F, (self.n + 7) // 8), dtype=np.uint8)
        iters = np.zeros(F, dtype=np.int32)
        succ = np.zeros(F, dtype=np.uint8)
        Lo = np.zeros((F, self.n_edges), dtype=np.int8) if want_state else None
        Eo = np.zeros((F, self.n), dtype=np.int8) if want_state else None
        L = _load()
        if perm_seed:
            for f in range(F):
                L.orc_decode(self._h, _p(llr[f]), _p(syn[f]), max_iter, early_stop, perm_seed + f,
                             _p(bits[f]), _p(iters[f:]), _p(succ[f:]),
                             None if Lo is None else _p(Lo[f]), None if Eo is None else _p(Eo[f]))
        else:
            if nthreads is None:
                nthreads = os.cpu_count() or 1
            L.orc_decode_batch(self._h, F, _p(llr), _p(syn), max_iter, early_stop, _p(bits), _p(iters),
                               _p(succ), _p(Lo), _p(Eo), min(nthreads, max(F, 1)))
        return dict(bits=bits, iters=iters, success=succ, L=Lo, E=Eo)


# ---------------------------------------------------------------------------------------
# Exact floating-point layered BP (R26), fp64.
# ---------------------------------------------------------------------------------------
LLR_KNOWN = 1000.0   # R26: finite stand-in for +-infinity (shortened bits, degree-1 checks)


def beta(a: float, b: float) -> float:
    """Eq.(6) box-plus of two magnitudes, stable form (R26)."""
    return _load().orc_beta(a, b)


def beta_eq6(a: float, b: float) -> float:
    """Eq.(6) written literally: 2 atanh(tanh(a/2) tanh(b/2))."""
    return _load().orc_beta_eq6(a, b)


def check_node_float(x, s_i: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _load().orc_check_node_float(len(x), _p(x), int(s_i), _p(out))
    return out


def build_llr_float(n: int, qber: float, y_bits: np.ndarray, kind=None, known_bits=None) -> np.ndarray:
    y = np.ascontiguousarray(y_bits, dtype=np.uint8).reshape(-1, (n + 7) // 8)
    kd = None if kind is None else np.ascontiguousarray(kind, dtype=np.uint8)
    kn = None if known_bits is None else np.ascontiguousarray(known_bits, dtype=np.uint8).reshape(y.shape)
    out = np.empty((y.shape[0], n), dtype=np.float64)
    for f in range(y.shape[0]):
        _load().orc_build_llr_float(n, qber, LLR_KNOWN, _p(y[f]), _p(kd), None if kn is None else _p(kn[f]),
                                    _p(out[f]))
    return out


def decode_float(code: "Code", llr: np.ndarray, syn: np.ndarray, max_iter: int, early_stop: int = 1,
                 want_state: bool = True, nthreads: int | None = None, flooding: bool = False) -> dict:
    """Batch fp64 BP decode (layered, or the flooding schedule of N4); same outputs as Code.decode
    with float L and E."""
    llr = np.ascontiguousarray(llr, dtype=np.float64).reshape(-1, code.n)
    F = llr.shape[0]
    syn = np.ascontiguousarray(syn, dtype=np.uint8).reshape(F, (code.m + 7) // 8)
    bits = np.zeros((F, (code.n + 7) // 8), dtype=np.uint8)
    iters = np.zeros(F, dtype=np.int32)
    succ = np.zeros(F, dtype=np.uint8)
    Lo = np.zeros((F, code.n_edges), dtype=np.float64) if want_state else None
    Eo = np.zeros((F, code.n), dtype=np.float64) if want_state else None
    nthreads = nthreads or os.cpu_count() or 1
    _load().orc_decode_float_batch(code._h, F, _p(llr), _p(syn), max_iter, early_stop, _p(bits), _p(iters),
                                   _p(succ), _p(Lo), _p(Eo), min(nthreads, max(F, 1)), int(bool(flooding)))
    return dict(bits=bits, iters=iters, success=succ, L=Lo, E=Eo)


# ---------------------------------------------------------------------------------------
# Interactive rate-adaptive reconciliation (R25), step by step.
# ---------------------------------------------------------------------------------------
def reveal_pattern(n: int, order: np.ndarray, s: int) -> np.ndarray:
    """pos_kind after revealing: order[:s] shortened (2), order[s:] punctured (1), rest payload (0).
    P:157 "the shortened bits are selected in turn from the puncturing bits"."""
    kind = np.zeros(n, dtype=np.uint8)
    order = np.asarray(order, dtype=np.int64)
    kind[order[s:]] = 1
    kind[order[:s]] = 2
    return kind


def reveal_rounds(code: "Code", qber: float, y: np.ndarray, x: np.ndarray, syn: np.ndarray, order: np.ndarray,
                  s0: int, delta: int, max_rounds: int, max_iter: int, nthreads: int | None = None) -> dict:
    """Bob decodes every frame with s0 shortened positions (SPEC bob_attempt); each frame
    that fails asks Alice to reveal the next `delta` punctured positions in reveal order (SPEC
    alice_reveal) and decodes again from scratch, until it matches its syndrome, the
    punctured positions run out, or max_rounds reveals were made ("multi-interaction").
    Returns per frame: bits, iters, success of the round it stopped at, rounds = that round index.
    Frames are independent: a plain loop over rounds, each decoding the frames still failing."""
    F = y.shape[0]
    d = len(order)
    nb8 = (code.n + 7) // 8
    out = dict(bits=np.zeros((F, nb8), np.uint8), iters=np.zeros(F, np.int32), rounds=np.zeros(F, np.int32),
               success=np.zeros(F, np.uint8))
    active = list(range(F))
    s_prev = -1
    for k in range(max_rounds + 1):
        if not active:
            break
        s = min(s0 + k * delta, d)
        if s == s_prev:
            break
        s_prev = s
        last = k == max_rounds or s == d
        kind = reveal_pattern(code.n, order, s)
        a = np.array(active)
        llr = code.build_llr(qber, y[a], kind, x[a])
        r = code.decode(llr, syn[a], max_iter, 1, want_state=False, nthreads=nthreads)
        still = []
        for i, f in enumerate(active):
            if r["success"][i] or last:
                out["bits"][f] = r["bits"][i]
                out["iters"][f] = r["iters"][i]
                out["success"][f] = r["success"][i]
                out["rounds"][f] = k
            if not r["success"][i]:
                still.append(f)
        if last:
            break
        active = still
    return out


def adaptive_efficiency(m: int, n: int, d: int, s0: int, delta: int, rounds: np.ndarray, qber: float) -> np.ndarray:
    """Per-frame efficiency after `rounds` reveals: R20 with p = d - s_k, s = s_k, i.e.
    f = (m - d + s_k) / ((n - d) h2(q)); each reveal round raises the leak by delta bits (SPEC
    alice_reveal: "leaked_bits increases by exactly k")."""
    s_k = np.minimum(s0 + np.asarray(rounds, dtype=np.int64) * delta, d)
    h2 = -qber * np.log2(qber) - (1 - qber) * np.log2(1 - qber)
    return (m - d + s_k) / ((n - d) * h2)
