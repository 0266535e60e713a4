"""Seeded random codes against the oracle (GPU): random base sizes, lifting sizes (powers of two and
not, below and above a warp), column/row degrees spanning every decode variant's range (1..40), random
full-range LLRs and syndromes, early stop on and off.  Complements the hand-picked edge cases of
test_gpu_parity.py; every output is compared byte for byte (bits, iters, success, final L and E)."""
import zlib

import numpy as np
import pytest

from _common import assert_same, gpu_decode, oracle_decode

pytestmark = pytest.mark.gpu


def _random_code(seed: int):
    rng = np.random.default_rng(seed)
    Mb = int(rng.integers(1, 7))
    Nb = int(rng.integers(Mb + 1, Mb + 40))
    Z = int(rng.choice([3, 8, 17, 32, 48, 64, 100, 128]))
    density = float(rng.choice([0.15, 0.4, 0.8, 1.0]))
    sh = np.where(rng.random((Mb, Nb)) < density, rng.integers(0, Z, (Mb, Nb)), -1)
    for J in range(Nb):                       # every column in at least one check
        if (sh[:, J] < 0).all():
            sh[int(rng.integers(0, Mb)), J] = int(rng.integers(0, Z))
    return sh.astype(np.int32), Z


@pytest.mark.parametrize("seed", range(24))
def test_random_codes(gpu, seed):
    shifts, Z = _random_code(1000 + seed)
    Mb, Nb = shifts.shape
    n, m = Nb * Z, Mb * Z
    rng = np.random.default_rng(zlib.crc32(f"fuzz/{seed}".encode()))
    F = int(rng.integers(1, 11))
    q = float(rng.choice([0.0, 0.02, 0.1]))
    base = np.where(rng.random((F, n)) < q, -1, 1) * int(rng.choice([4, 12, 18]))
    wild = rng.integers(-127, 128, size=(F, n))
    llr = np.where(rng.random((F, n)) < 0.3, wild, base).astype(np.int8)
    syn = rng.integers(0, 256, size=(F, (m + 7) // 8), dtype=np.uint8)
    if seed % 3 == 0:
        syn[:] = 0                              # all-zero target: the all-zero word is a codeword
    early = int(seed % 2 == 0)
    T = int(rng.integers(0, 12))
    g, code = gpu_decode(gpu, shifts, Z, None, llr, syn, T, early)
    o = oracle_decode(shifts, Z, llr, syn, T, early)
    assert_same(g, o)
