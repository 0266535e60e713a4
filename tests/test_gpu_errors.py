"""Error behaviour of the C ABI as include/qkd_ldpc.h states it (GPU needed: creating a code uploads
its tables to the current device)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _err(gpu, fn, code_substr):
    with pytest.raises(gpu.QkdError) as ei:
        fn()
    assert code_substr in str(ei.value), str(ei.value)


def test_code_create_errors(gpu):
    _err(gpu, lambda: gpu.QCCode(np.array([[0, 5, 1]]), 4), "-3")                      # shift >= Z: QKD_ESHIFT
    with pytest.raises(gpu.QkdError) as ei:
        gpu.QCCode(np.array([[0, 1, 2], [3, 9, 1]]), 4)
    assert "(1,1)" in str(ei.value)                                                     # names the block
    _err(gpu, lambda: gpu.QCCode(np.array([[0, 1], [1, 0]]), 4), "-1")                 # Nb <= Mb: QKD_EINVAL
    _err(gpu, lambda: gpu.QCCode(np.zeros((1, 70), dtype=np.int32), 2), "-6")          # degree > 64: QKD_EUNSUP
    with pytest.raises(gpu.QkdError):
        gpu.QCCode(np.array([[0, 1, 2]]), 4, pos_kind=np.zeros(5, dtype=np.uint8))      # wrong pos_kind length


def test_call_errors(gpu):
    import torch

    code = gpu.QCCode(np.array([[0, 1, 2, 3], [2, -1, 1, 0]]), 8)
    F = 5
    y = torch.zeros((F, code.nb8), dtype=torch.uint8, device="cuda")
    _err(gpu, lambda: code.build_llr(0.0, y), "-1")                                    # qber outside (0, 0.5)
    _err(gpu, lambda: code.build_llr(0.5, y), "-1")
    llr = code.build_llr(0.05, y)
    syn = torch.zeros((F, code.mb8), dtype=torch.uint8, device="cuda")
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    _err(gpu, lambda: code.decode(llr, syn, 10, True, workspace=small), "-2")          # QKD_EDIM
    r = code.decode(llr[:0], syn[:0], 10, True)                                          # F = 0: no-op
    assert r["bits"].shape == (0, code.nb8)
    order = torch.arange(4, dtype=torch.int32, device="cuda")
    _err(gpu, lambda: code.reconcile_adaptive(0.05, order, 1, 0, 3, y, y, syn, 10), "-1")   # delta < 1
    _err(gpu, lambda: code.reconcile_adaptive(0.05, order, 9, 1, 3, y, y, syn, 10), "-1")   # s0 > d


def test_float_decoder_degree_limit(gpu):
    import torch

    code = gpu.QCCode(np.zeros((1, 34), dtype=np.int32), 3)                              # check degree 34 > 32
    F = 2
    y = torch.zeros((F, code.nb8), dtype=torch.uint8, device="cuda")
    llr = code.build_llr_float(0.05, y)
    syn = torch.zeros((F, code.mb8), dtype=torch.uint8, device="cuda")
    _err(gpu, lambda: code.decode_float(llr, syn, 5, True), "-6")
    assert code.decode(code.build_llr(0.05, y), syn, 5, True)["success"].all()          # int path: generic


def test_reconcile_host_validates_host_arrays(gpu):
    """qkd_reconcile_host copies F rows of fixed size from/to the host pointers: the binding refuses
    arrays of the wrong dtype, shape or layout instead of letting the library read/write past them."""
    code = gpu.QCCode(np.array([[0, 1, 2, 3], [2, -1, 1, 0]]), 8)
    F = 4
    y = np.zeros((F, code.nb8), np.uint8)
    syn = np.zeros((F, code.mb8), np.uint8)
    bits, iters, succ = code.reconcile_host(0.05, y, syn, 10)                          # well-formed: runs
    assert succ.all() and (iters == 0).all()
    with pytest.raises(gpu.QkdError):
        code.reconcile_host(0.05, y, syn[:, :1], 10)                                    # short syndrome rows
    with pytest.raises(gpu.QkdError):
        code.reconcile_host(0.05, y.astype(np.int32), syn, 10)                         # wrong dtype
    with pytest.raises(gpu.QkdError):
        code.reconcile_host(0.05, np.zeros((2 * F, code.nb8), np.uint8)[::2], syn, 10)   # not contiguous
    with pytest.raises(gpu.QkdError):
        code.reconcile_host(0.05, y, syn, 10, out=(np.empty((F, 1), np.uint8), iters, succ))


def test_decode_host_overhead(gpu):
    """Per-call host cost of qkd_decode_batch once a batch size has been seen (plans cached in the
    handle: no attribute calls or occupancy queries per call): the C call, timed from Python around
    the ctypes call with everything pre-marshalled, stays in the tens of microseconds (one kernel
    launch plus a memset)."""
    import ctypes
    import time

    import torch

    code = gpu.QCCode(np.array([[0, 1, 2, 3], [2, -1, 1, 0]]), 8)
    F = 64
    y = torch.zeros((F, code.nb8), dtype=torch.uint8, device="cuda")
    llr = code.build_llr(0.05, y)
    syn = torch.zeros((F, code.mb8), dtype=torch.uint8, device="cuda")
    ws = torch.empty(code.workspace_bytes(F), dtype=torch.uint8, device="cuda")
    out = code.decode(llr, syn, 5, True, workspace=ws)
    L = gpu.lib()
    p = ctypes.c_void_p
    args = (code._h, F, p(llr.data_ptr()), p(syn.data_ptr()), 5, 1, p(ws.data_ptr()), ws.numel(),
            p(out["bits"].data_ptr()), p(out["iters"].data_ptr()), p(out["success"].data_ptr()), None, None, None,
            p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        assert L.qkd_decode_batch(*args) == 0
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    med = float(np.median(ts)) * 1e6
    print(f"qkd_decode_batch host time: median {med:.1f} us")
    assert med < 50.0, med
