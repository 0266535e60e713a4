"""B200-native (sm_100a) batched quantized LDPC syndrome decoder for QKD reconciliation,
after arXiv:1903.10107 (§3: 8-bit quantization, improved RCBP check nodes,
saturation-oriented variable nodes, layered schedule with early termination).

This module is a thin ctypes binding over libqkdldpc.so (include/qkd_ldpc.h): argument
marshalling only.  Every step of the decoding path runs in the library's CUDA kernels; there
is no CPU fallback -- importing works without a GPU, but every call needs the built library
and a CUDA device and raises otherwise.  PyTorch is used for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QKD_LIB") or os.path.join(_HERE, "libqkdldpc.so")  # QKD_LIB: an alternative in-tree build (A/B timing)
_lib = None

QKD_OK = 0
N_COUNTERS = 5   # [frames, successes, frames with bit errors, undetected errors, sum of iterations]


class QkdError(RuntimeError):
    pass


def lib():
    """Load libqkdldpc.so (raises if it was not built -- run __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise QkdError(f"{LIB_PATH} missing: the CUDA extension is not built (python _build.py)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.qkd_code_create.argtypes = [vp, i32, i32, i32, vp, ctypes.POINTER(vp)]
        L.qkd_code_destroy.argtypes = [vp]
        L.qkd_code_destroy.restype = None
        L.qkd_code_info.argtypes = [vp, vp, vp, vp, vp]
        L.qkd_llr_magnitude.argtypes = [dbl]
        L.qkd_syndrome.argtypes = [vp, i64, vp, vp, vp]
        L.qkd_build_llr.argtypes = [vp, dbl, i64, vp, vp, vp, vp]
        L.qkd_workspace_bytes.argtypes = [vp, i64]
        L.qkd_workspace_bytes.restype = ctypes.c_size_t
        L.qkd_decode_batch.argtypes = [vp, i64, vp, vp, i32, i32, vp, ctypes.c_size_t, vp, vp, vp, vp, vp,
                                       vp, vp]
        L.qkd_score_batch.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
        L.qkd_reconcile_device_bytes.argtypes = [vp, i64]
        L.qkd_reconcile_device_bytes.restype = ctypes.c_size_t
        L.qkd_reconcile_host.argtypes = [vp, dbl, i64, vp, vp, vp, i32, i32, vp, ctypes.c_size_t, vp, vp,
                                         vp, vp]
        L.qkd_launch_info.argtypes = [vp, i64, vp]
        L.qkd_build_llr_float.argtypes = [vp, dbl, i64, vp, vp, vp, vp]
        L.qkd_float_workspace_bytes.argtypes = [vp, i64]
        L.qkd_float_workspace_bytes.restype = ctypes.c_size_t
        L.qkd_decode_float_batch.argtypes = [vp, i64, vp, vp, i32, i32, i32, vp, ctypes.c_size_t, vp, vp, vp, vp,
                                             vp, vp]
        L.qkd_adaptive_work_bytes.argtypes = [vp, i64]
        L.qkd_adaptive_work_bytes.restype = ctypes.c_size_t
        L.qkd_reconcile_adaptive.argtypes = [vp, dbl, i64, vp, i64, i64, i64, i32, vp, vp, vp, i32, vp,
                                             ctypes.c_size_t, vp, vp, vp, vp, vp]
        L.qkd_tau_table.argtypes = [vp, vp]
        L.qkd_last_error.argtypes = []
        L.qkd_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != QKD_OK:
        raise QkdError(f"qkd error {rc}: {lib().qkd_last_error().decode()}")


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise QkdError("no CUDA device: the decoder has no CPU path")
    return torch


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need(t, dtype, shape, name):
    torch = _torch()
    if t.device.type != "cuda" or t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise QkdError(f"{name}: expected contiguous cuda {dtype} {tuple(shape)}, got {t.device} {t.dtype} "
                       f"{tuple(t.shape)}")
    return t


def llr_magnitude(qber: float) -> int:
    """min(127, round(4 ln((1-q)/q))) -- quantized BSC channel LLR magnitude."""
    v = lib().qkd_llr_magnitude(float(qber))
    _check(min(v, 0))
    return v


def tau_table(stream=None):
    """64x64 uint8 table of tau(p, q) computed by the kernels' packed arithmetic (self-test)."""
    torch = _torch()
    out = torch.empty((64, 64), dtype=torch.uint8, device="cuda")
    _check(lib().qkd_tau_table(_ptr(out), _stream(stream)))
    return out


class QCCode:
    """QC-LDPC code on the current CUDA device (qkd_code_create)."""

    def __init__(self, shifts, Z: int, pos_kind=None):
        sh = np.ascontiguousarray(np.asarray(shifts), dtype=np.int32)
        if sh.ndim != 2:
            raise QkdError("shifts must be a 2-D base matrix")
        self.Mb, self.Nb = sh.shape
        self.Z = int(Z)
        kind = None
        if pos_kind is not None:
            kind = np.ascontiguousarray(np.asarray(pos_kind), dtype=np.uint8)
            if kind.shape != (self.Nb * self.Z,):
                raise QkdError("pos_kind must have n = Nb*Z entries")
        self._kind = kind
        h = ctypes.c_void_p()
        _check(lib().qkd_code_create(sh.ctypes.data, self.Mb, self.Nb, self.Z,
                                     None if kind is None else kind.ctypes.data, ctypes.byref(h)))
        self._h = h
        n, m, e, d = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        _check(lib().qkd_code_info(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(e), ctypes.byref(d)))
        self.n, self.m, self.n_edges, self.max_row_deg = n.value, m.value, e.value, d.value
        self.nb8 = (self.n + 7) // 8
        self.mb8 = (self.m + 7) // 8

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib is not None:
            _lib.qkd_code_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- Alice -------------------------------------------------------------------------
    def syndrome(self, bits, out=None, stream=None):
        torch = _torch()
        F = bits.shape[0]
        _need(bits, torch.uint8, (F, self.nb8), "bits")
        out = out if out is not None else torch.empty((F, self.mb8), dtype=torch.uint8, device=bits.device)
        _check(lib().qkd_syndrome(self._h, F, _ptr(bits), _ptr(out), _stream(stream)))
        return out

    # -- Bob ---------------------------------------------------------------------------
    def build_llr(self, qber, bob_bits, known_bits=None, out=None, stream=None):
        torch = _torch()
        F = bob_bits.shape[0]
        _need(bob_bits, torch.uint8, (F, self.nb8), "bob_bits")
        if known_bits is not None:
            _need(known_bits, torch.uint8, (F, self.nb8), "known_bits")
        out = out if out is not None else torch.empty((F, self.n), dtype=torch.int8, device=bob_bits.device)
        _check(lib().qkd_build_llr(self._h, float(qber), F, _ptr(bob_bits), _ptr(known_bits), _ptr(out),
                                   _stream(stream)))
        return out

    def workspace_bytes(self, n_frames: int) -> int:
        v = lib().qkd_workspace_bytes(self._h, int(n_frames))
        if v == 0:
            _check(-4)
        return v

    def launch_info(self, n_frames: int) -> dict:
        info = (ctypes.c_int32 * 8)()
        _check(lib().qkd_launch_info(self._h, int(n_frames), info))
        keys = ("variant", "threads_per_group", "groups_per_cta", "grid", "smem_bytes", "frames_per_group",
                "groups")
        return {k: int(info[i]) for i, k in enumerate(keys)}

    def decode(self, llr, syn, max_iter: int, early_stop: bool = True, want_state: bool = False,
               counters=None, workspace=None, out=None, stream=None):
        """Returns dict(bits, iters, success[, L, E]) as cuda tensors (asynchronous)."""
        torch = _torch()
        F = llr.shape[0]
        _need(llr, torch.int8, (F, self.n), "llr")
        _need(syn, torch.uint8, (F, self.mb8), "syn")
        dev = llr.device
        o = out or {}
        bits = o.get("bits", None)
        bits = bits if bits is not None else torch.empty((F, self.nb8), dtype=torch.uint8, device=dev)
        iters = o.get("iters", None)
        iters = iters if iters is not None else torch.empty(F, dtype=torch.int32, device=dev)
        succ = o.get("success", None)
        succ = succ if succ is not None else torch.empty(F, dtype=torch.uint8, device=dev)
        Lo = Eo = None
        if want_state:
            Lo = torch.empty((F, self.n_edges), dtype=torch.int8, device=dev)
            Eo = torch.empty((F, self.n), dtype=torch.int8, device=dev)
        if workspace is None:
            workspace = torch.empty(self.workspace_bytes(F), dtype=torch.uint8, device=dev)
        if counters is not None:
            _need(counters, torch.int64, (N_COUNTERS,), "counters")
        _check(lib().qkd_decode_batch(self._h, F, _ptr(llr), _ptr(syn), int(max_iter), int(bool(early_stop)),
                                      _ptr(workspace), workspace.numel(), _ptr(bits), _ptr(iters), _ptr(succ),
                                      _ptr(Lo), _ptr(Eo), _ptr(counters), _stream(stream)))
        r = dict(bits=bits, iters=iters, success=succ)
        if want_state:
            r["L"], r["E"] = Lo, Eo
        return r

    # -- exact floating-point BP (DESIGN R26) ---------------------------
    def build_llr_float(self, qber, bob_bits, known_bits=None, out=None, stream=None):
        torch = _torch()
        F = bob_bits.shape[0]
        _need(bob_bits, torch.uint8, (F, self.nb8), "bob_bits")
        if known_bits is not None:
            _need(known_bits, torch.uint8, (F, self.nb8), "known_bits")
        out = out if out is not None else torch.empty((F, self.n), dtype=torch.float32, device=bob_bits.device)
        _check(lib().qkd_build_llr_float(self._h, float(qber), F, _ptr(bob_bits), _ptr(known_bits), _ptr(out),
                                         _stream(stream)))
        return out

    def decode_float(self, llr, syn, max_iter: int, early_stop: bool = True, want_state: bool = False,
                     workspace=None, stream=None, flooding: bool = False):
        """qkd_decode_float_batch: dict(bits, iters, success[, L, E]) as cuda tensors (asynchronous)."""
        torch = _torch()
        F = llr.shape[0]
        _need(llr, torch.float32, (F, self.n), "llr")
        _need(syn, torch.uint8, (F, self.mb8), "syn")
        dev = llr.device
        bits = torch.empty((F, self.nb8), dtype=torch.uint8, device=dev)
        iters = torch.empty(F, dtype=torch.int32, device=dev)
        succ = torch.empty(F, dtype=torch.uint8, device=dev)
        Lo = torch.empty((F, self.n_edges), dtype=torch.float32, device=dev) if want_state else None
        Eo = torch.empty((F, self.n), dtype=torch.float32, device=dev) if want_state else None
        if workspace is None:
            nbytes = lib().qkd_float_workspace_bytes(self._h, F)
            if nbytes == 0:
                _check(-6)
            workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        _check(lib().qkd_decode_float_batch(self._h, F, _ptr(llr), _ptr(syn), int(max_iter), int(bool(early_stop)),
                                            int(bool(flooding)), _ptr(workspace), workspace.numel(), _ptr(bits), _ptr(iters), _ptr(succ),
                                            _ptr(Lo), _ptr(Eo), _stream(stream)))
        r = dict(bits=bits, iters=iters, success=succ)
        if want_state:
            r["L"], r["E"] = Lo, Eo
        return r

    # -- interactive rate adaptation (DESIGN R25) ------------------------
    def reconcile_adaptive(self, qber, order, s0: int, delta: int, max_rounds: int, bob_bits, alice_bits, syn,
                           max_iter: int, work=None, stream=None):
        """qkd_reconcile_adaptive: reveal rounds over the reserved positions `order` (int32 cuda).
        Returns dict(bits, iters, rounds, success) as cuda tensors (the call synchronises once per round)."""
        torch = _torch()
        F = bob_bits.shape[0]
        _need(bob_bits, torch.uint8, (F, self.nb8), "bob_bits")
        _need(alice_bits, torch.uint8, (F, self.nb8), "alice_bits")
        _need(syn, torch.uint8, (F, self.mb8), "syn")
        d = order.numel()
        _need(order, torch.int32, (d,), "order")
        dev = bob_bits.device
        if work is None:
            nbytes = lib().qkd_adaptive_work_bytes(self._h, F)
            if nbytes == 0:
                _check(-4)
            work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        bits = torch.empty((F, self.nb8), dtype=torch.uint8, device=dev)
        iters = torch.empty(F, dtype=torch.int32, device=dev)
        rounds = torch.empty(F, dtype=torch.int32, device=dev)
        succ = torch.empty(F, dtype=torch.uint8, device=dev)
        _check(lib().qkd_reconcile_adaptive(self._h, float(qber), F, _ptr(order), d, int(s0), int(delta),
                                            int(max_rounds), _ptr(bob_bits), _ptr(alice_bits), _ptr(syn),
                                            int(max_iter), _ptr(work), work.numel(), _ptr(bits), _ptr(iters),
                                            _ptr(rounds), _ptr(succ), _stream(stream)))
        return dict(bits=bits, iters=iters, rounds=rounds, success=succ)

    # -- harness -----------------------------------------------------------------------
    def score(self, bits, alice_bits, success, counters=None, want_errors=False, stream=None):
        torch = _torch()
        F = bits.shape[0]
        errs = torch.empty(F, dtype=torch.int32, device=bits.device) if want_errors else None
        _check(lib().qkd_score_batch(self._h, F, _ptr(bits), _ptr(alice_bits), _ptr(success), _ptr(errs),
                                     _ptr(counters), _stream(stream)))
        return errs

    def reconcile_device_bytes(self, n_frames: int) -> int:
        return lib().qkd_reconcile_device_bytes(self._h, int(n_frames))

    def reconcile_host(self, qber, bob_bits, syndrome, max_iter, early_stop=True, known_bits=None,
                       device_buffer=None, out=None, stream=None):
        """End-to-end call on HOST buffers (numpy or pinned CPU tensors): H2D, LLR, decode, D2H.
        Returns (bits, iters, success) host arrays."""
        torch = _torch()

        def hp(a, dtype, shape, name):
            """Host pointer of a C-contiguous CPU array/tensor of exactly dtype and shape (the library
            copies F rows of fixed size from/to it, so anything else would be read/written out of bounds)."""
            if a is None:
                return None
            if isinstance(a, np.ndarray):
                ok = a.dtype == dtype and a.shape == tuple(shape) and a.flags["C_CONTIGUOUS"]
                got = f"numpy {a.dtype} {a.shape}"
                ptr = a.ctypes.data
            else:
                tdt = {np.uint8: torch.uint8, np.int32: torch.int32}[dtype]
                ok = (a.device.type == "cpu" and a.dtype == tdt and tuple(a.shape) == tuple(shape)
                      and a.is_contiguous())
                got = f"{a.device} {a.dtype} {tuple(a.shape)}"
                ptr = a.data_ptr()
            if not ok:
                raise QkdError(f"{name}: expected a C-contiguous host {np.dtype(dtype).name} array of shape "
                               f"{tuple(shape)}, got {got}")
            return ctypes.c_void_p(ptr)

        F = int(bob_bits.shape[0])
        if out is None:
            out = (np.empty((F, self.nb8), np.uint8), np.empty(F, np.int32), np.empty(F, np.uint8))
        if device_buffer is None:
            device_buffer = torch.empty(self.reconcile_device_bytes(F), dtype=torch.uint8, device="cuda")
        _need(device_buffer, torch.uint8, (device_buffer.numel(),), "device_buffer")
        args = (hp(bob_bits, np.uint8, (F, self.nb8), "bob_bits"), hp(known_bits, np.uint8, (F, self.nb8), "known_bits"),
                hp(syndrome, np.uint8, (F, self.mb8), "syndrome"), hp(out[0], np.uint8, (F, self.nb8), "out bits"),
                hp(out[1], np.int32, (F,), "out iters"), hp(out[2], np.uint8, (F,), "out success"))
        _check(lib().qkd_reconcile_host(self._h, float(qber), F, args[0], args[1], args[2],
                                        int(max_iter), int(bool(early_stop)), _ptr(device_buffer),
                                        device_buffer.numel(), args[3], args[4], args[5], _stream(stream)))
        return out
