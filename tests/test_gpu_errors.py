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
