"""CPU-side checks of the C ABI: the library builds for sm_100a, loads without a GPU and
exports every function include/qkd_ldpc.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qkd_ldpc.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(qkd_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("qkd_code_create", "qkd_code_destroy", "qkd_decode_batch", "qkd_build_llr", "qkd_syndrome",
                 "qkd_workspace_bytes", "qkd_last_error", "qkd_reconcile_host", "qkd_score_batch"):
        assert must in names
    assert len(names) >= 14


def test_library_exports_every_declared_symbol(cuda_lib):
    L = ctypes.CDLL(cuda_lib.LIB_PATH)
    for name in declared_functions():
        assert hasattr(L, name), name


def test_library_is_sm100a_only(cuda_lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", cuda_lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for bad in ("sm_90", "sm_80", "sm_103"):
        assert bad not in out


def test_oracle_and_product_share_nothing():
    """The oracle (test infrastructure) and the CUDA product never import/include each other."""
    imp = re.compile(r"^\s*(import|from)\s+(\S+)|^\s*#\s*include\s*[<\"]([^>\"]+)", re.M)

    def deps(path):
        return [m.group(2) or m.group(3) for m in imp.finditer(open(path).read())]

    prod = os.path.join(ROOT, "paper_1903_10107_b200")
    for dirpath, _, files in os.walk(prod):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                for d in deps(os.path.join(dirpath, f)):
                    assert "oracle" not in d and "synth" not in d, (f, d)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            for d in deps(os.path.join(ROOT, "oracle", f)):
                assert "paper_1903_10107_b200" not in d and "qkd" not in d and "synth" not in d, (f, d)


def test_binding_fails_loudly_without_gpu(cuda_lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(cuda_lib.QkdError):
        cuda_lib.tau_table()
