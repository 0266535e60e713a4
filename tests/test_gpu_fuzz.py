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


def _frames(shifts, Z, seed, F=None):
    Mb, Nb = shifts.shape
    n, m = Nb * Z, Mb * Z
    rng = np.random.default_rng(zlib.crc32(f"fuzz-frames/{seed}".encode()))
    F = F or int(rng.integers(1, 11))
    base = np.where(rng.random((F, n)) < 0.03, -1, 1) * int(rng.choice([10, 16]))
    wild = rng.integers(-127, 128, size=(F, n))
    llr = np.where(rng.random((F, n)) < 0.2, wild, base).astype(np.int8)
    syn = rng.integers(0, 256, size=(F, (m + 7) // 8), dtype=np.uint8)
    return llr, syn


@pytest.mark.parametrize("seed", range(6))
def test_random_long_codes(gpu, seed):
    """Frames too long for shared memory (n >= 60000): the global-E variants 7 / 8 / 4."""
    rng = np.random.default_rng(5000 + seed)
    Mb = int(rng.integers(1, 4))
    Z = int(rng.choice([1536, 2048, 3001]))
    Nb = int(max(Mb + 1, -(-60000 // Z) + int(rng.integers(0, 6))))
    density = float(rng.choice([0.3, 0.7, 1.0]))
    sh = np.where(rng.random((Mb, Nb)) < density, rng.integers(0, Z, (Mb, Nb)), -1)
    for J in range(Nb):
        if (sh[:, J] < 0).all():
            sh[int(rng.integers(0, Mb)), J] = int(rng.integers(0, Z))
    sh = sh.astype(np.int32)
    llr, syn = _frames(sh, Z, 5000 + seed, F=3)
    g, code = gpu_decode(gpu, sh, Z, None, llr, syn, 6, seed % 2)
    assert code.launch_info(3)["variant"] % 10 in (4, 7, 8)
    o = oracle_decode(sh, Z, llr, syn, 6, seed % 2)
    assert_same(g, o)


@pytest.mark.parametrize("mode", ["split", "refill"])
@pytest.mark.parametrize("seed", [2, 6, 12, 14, 15, 18, 20])
def test_random_codes_opt_in_variants(gpu, monkeypatch, mode, seed):
    """The opt-in scheduling variants on the random codes: lane-pair rows (QKD_SPLIT=1, degrees
    9..20) and per-frame lane refill forced on every variant (QKD_REFILL=1)."""
    monkeypatch.setenv("QKD_SPLIT" if mode == "split" else "QKD_REFILL", "1")
    shifts, Z = _random_code(1000 + seed)
    llr, syn = _frames(shifts, Z, seed, F=7)
    g, _ = gpu_decode(gpu, shifts, Z, None, llr, syn, 9, 1)
    o = oracle_decode(shifts, Z, llr, syn, 9, 1)
    assert_same(g, o)


@pytest.mark.parametrize("seed", range(24))
def test_random_syndrome_llr_score(gpu, seed):
    """Alice's syndrome (QC funnel-shift kernel when Z % 32 == 0, per-bit kernel otherwise), Bob's LLRs
    with random punctured/shortened patterns and known bits, and the error score, on the random codes."""
    import torch

    import oracle

    shifts, Z = _random_code(1000 + seed)
    Mb, Nb = shifts.shape
    n = Nb * Z
    rng = np.random.default_rng(zlib.crc32(f"fuzz-io/{seed}".encode()))
    F = int(rng.integers(1, 40))
    nb8 = (n + 7) // 8
    x = rng.integers(0, 256, size=(F, nb8), dtype=np.uint8)
    y = rng.integers(0, 256, size=(F, nb8), dtype=np.uint8)
    if n % 8:                                    # bits past n are zero in the packed inputs
        x[:, -1] &= (1 << (n % 8)) - 1
        y[:, -1] &= (1 << (n % 8)) - 1
    kind = rng.choice(np.array([0, 0, 0, 1, 2], dtype=np.uint8), size=n) if seed % 2 else None
    q = float(rng.choice([0.01, 0.03, 0.08, 0.2]))
    oc = oracle.Code(shifts, Z)
    code = gpu.QCCode(shifts, Z, kind)
    xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    assert np.array_equal(code.syndrome(xs).cpu().numpy(), oc.syndrome(x))
    llr = code.build_llr(q, ys, xs if kind is not None else None).cpu().numpy()
    assert np.array_equal(llr, oc.build_llr(q, y, kind, x if kind is not None else None))
    succ = torch.from_numpy(rng.integers(0, 2, F).astype(np.uint8)).cuda()
    errs = code.score(ys, xs, succ, want_errors=True).cpu().numpy()
    diff = np.unpackbits(x ^ y, axis=1, bitorder="little")[:, :n]
    if kind is not None:
        diff = diff[:, kind == 0]
    assert np.array_equal(errs, diff.sum(axis=1))


@pytest.mark.parametrize("flooding", [False, True])
@pytest.mark.parametrize("seed", [0, 2, 5, 8, 9, 12, 13, 16, 21])
def test_random_codes_float(gpu, seed, flooding):
    """Exact float BP (degrees <= 32) on the random codes: two sweeps of state against the fp64 oracle
    within the tolerance of tests/test_float_gpu.py."""
    import torch

    import oracle

    shifts, Z = _random_code(1000 + seed)
    if (shifts >= 0).sum(axis=1).max() > 32:
        pytest.skip("float decoder: check degree > 32")
    oc = oracle.Code(shifts, Z)
    rng = np.random.default_rng(zlib.crc32(f"fuzz-float/{seed}".encode()))
    F = 3
    y = rng.integers(0, 256, size=(F, (oc.n + 7) // 8), dtype=np.uint8)
    syn = rng.integers(0, 256, size=(F, (oc.m + 7) // 8), dtype=np.uint8)
    llr_o = oracle.build_llr_float(oc.n, 0.05, y)
    code = gpu.QCCode(shifts, Z)
    llr_g = code.build_llr_float(0.05, torch.from_numpy(y).cuda())
    for T in (1, 2):
        o = oracle.decode_float(oc, llr_o, syn, T, 0, flooding=flooding)
        g = code.decode_float(llr_g, torch.from_numpy(syn).cuda(), T, False, want_state=True, flooding=flooding)
        for k in ("E", "L"):
            gv = g[k].cpu().numpy()
            assert np.allclose(gv, o[k], rtol=1e-5, atol=2e-3 * T), (k, T, np.abs(gv - o[k]).max())
