"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit for bit, on
the same seeded inputs.  The decoder is integer-only, so every output --
hard decisions, iteration counts, success flags and the final int8 message state L and E --
must be identical."""
import zlib

import numpy as np
import pytest

import oracle
import synth
from _common import assert_same, gpu_decode, oracle_decode, to_np, workload_inputs

pytestmark = pytest.mark.gpu


def test_tau_table_exhaustive(gpu):
    t = gpu.tau_table().cpu().numpy()
    ref = np.array([[oracle.tau(p, q) for q in range(64)] for p in range(64)], dtype=np.uint8)
    assert np.array_equal(t, ref)


@pytest.mark.parametrize("name,F", [("C1", 64), ("C2", 64), ("C3", 8), ("C4@0.02", 4)])
def test_syndrome_and_llr_parity(gpu, name, F):
    import torch

    w, shifts, kind, x, y, llr, syn = workload_inputs(name, F)
    code = gpu.QCCode(shifts, w.Z, kind)
    xs = torch.from_numpy(x).cuda()
    ys = torch.from_numpy(y).cuda()
    s_gpu = code.syndrome(xs).cpu().numpy()
    assert np.array_equal(s_gpu, syn)
    l_gpu = code.build_llr(w.qber, ys, xs if kind is not None else None).cpu().numpy()
    assert np.array_equal(l_gpu, llr)


@pytest.mark.parametrize("name,F", [("C1", 64), ("C2", 192), ("C3", 12), ("C4@0.01", 4), ("C4@0.02", 4),
                                    ("C4@0.04", 4), ("C4@0.06", 4), ("C4@0.08", 4)])
def test_decode_parity_workloads(gpu, name, F):
    w, shifts, kind, x, y, llr, syn = workload_inputs(name, F)
    g, code = gpu_decode(gpu, shifts, w.Z, kind, llr, syn, w.max_iter, w.early_stop)
    o = oracle_decode(shifts, w.Z, llr, syn, w.max_iter, w.early_stop)
    assert_same(g, o)


def _tiny_cases():
    rng = np.random.default_rng(11)
    cases = {}
    cases["2x4_Z5"] = (np.array([[0, 1, 3, -1], [2, -1, 4, 0]]), 5)                # Z not pow2, Z < 32
    cases["2x3_Z7_n21"] = (np.array([[0, 3, 5], [6, -1, 1]]), 7)                   # n % 4 != 0
    cases["deg1_deg2"] = (np.array([[0, -1, -1, -1], [3, 1, -1, -1], [2, 0, 4, 1]]), 6)
    sh = rng.integers(0, 40, (3, 30))
    sh[1, rng.random(30) < 0.5] = -1
    sh[2, rng.random(30) < 0.8] = -1
    cases["deg30_Z40"] = (sh, 40)                                                  # degree 21..32, Z not pow2
    sh = rng.integers(0, 64, (4, 24))
    sh[rng.random((4, 24)) < 0.4] = -1
    cases["deg9to20"] = (sh, 64)
    sh = rng.integers(0, 96, (3, 9))
    cases["Z96_multiwarp"] = (sh, 96)                                              # Z%32==0, not pow2
    sh = np.full((4, 36), -1)
    for I in range(4):                                                             # degrees 21..32 (variant 6)
        cols = rng.permutation(36)[: int(rng.integers(21, 33))]
        sh[I, cols] = rng.integers(0, 64, len(cols))
    sh[0, (sh >= 0).sum(axis=0) == 0] = 5
    cases["deg21to32_pow2"] = (sh, 64)
    sh = rng.integers(0, 8, (2, 44))
    sh[1, rng.random(44) < 0.7] = -1
    sh[0, :4] = -1
    sh[1, :4] = rng.integers(0, 8, 4)
    cases["deg40_generic"] = (sh, 8)                                               # degree > 32
    cases["empty_row"] = (np.array([[0, 2, -1, 1], [-1, -1, -1, -1], [3, -1, 0, 2]]), 32)   # a degree-0 block row
    return cases


TINY = _tiny_cases()


@pytest.mark.parametrize("case", sorted(TINY))
@pytest.mark.parametrize("F", [1, 3, 7, 13])
@pytest.mark.parametrize("early_stop", [1, 0])
def test_decode_parity_edge_cases(gpu, case, F, early_stop):
    """Random full-range LLRs (saturated +-127, zeros, everything in between) and random
    target syndromes exercise the saturation guard, the 6-bit clamp, x = 0 ties and
    non-convergence; ragged batches exercise the padded frame lanes."""
    shifts, Z = TINY[case]
    shifts = np.asarray(shifts, dtype=np.int32)
    Mb, Nb = shifts.shape
    n, m = Nb * Z, Mb * Z
    rng = np.random.default_rng(zlib.crc32(f"{case}/{F}/{early_stop}".encode()))
    special = rng.choice(np.array([-127, -126, -64, -63, -20, -5, -1, 0, 1, 4, 17, 63, 64, 100, 126, 127]),
                         size=(F, n))
    uniform = rng.integers(-127, 128, size=(F, n))
    llr = np.where(rng.random((F, n)) < 0.5, special, uniform).astype(np.int8)
    syn = rng.integers(0, 256, size=(F, (m + 7) // 8), dtype=np.uint8)
    for T in (0, 1, 9):
        g, _ = gpu_decode(gpu, shifts, Z, None, llr, syn, T, early_stop)
        o = oracle_decode(shifts, Z, llr, syn, T, early_stop)
        assert_same(g, o)


def test_decode_parity_channel_frames_tiny(gpu):
    """Many channel-like frames on a tiny code (mix of convergence iterations)."""
    shifts, Z = TINY["2x4_Z5"]
    code = oracle.Code(shifts, Z)
    x, y, _ = synth.frames(code.n, 0.07, 99, 0, 997)
    syn = code.syndrome(x)
    llr = code.build_llr(0.07, y)
    g, _ = gpu_decode(gpu, shifts, Z, None, llr, syn, 25, 1)
    o = oracle_decode(shifts, Z, llr, syn, 25, 1)
    assert_same(g, o)
    assert len(np.unique(o["iters"])) > 3


def test_zero_error_frames_iteration_zero(gpu):
    w, shifts, kind, x, y, llr, syn = workload_inputs("C2", 9)
    oc = oracle.Code(shifts, w.Z)
    llr0 = oc.build_llr(w.qber, x)
    g, _ = gpu_decode(gpu, shifts, w.Z, None, llr0, syn, w.max_iter, 1)
    assert (g["iters"] == 0).all() and (g["success"] == 1).all()
    assert np.array_equal(g["bits"], x)
    assert not g["L"].any()


def test_batch_composition_invariance(gpu):
    """a frame's result does not depend on the batch around it."""
    w, shifts, kind, x, y, llr, syn = workload_inputs("C2", 40)
    full, _ = gpu_decode(gpu, shifts, w.Z, None, llr, syn, w.max_iter, 1)
    for a, b in ((0, 1), (3, 11), (17, 40), (5, 6)):
        part, _ = gpu_decode(gpu, shifts, w.Z, None, llr[a:b], syn[a:b], w.max_iter, 1)
        for k in full:
            assert np.array_equal(full[k][a:b], part[k]), (k, a, b)


def test_counters_and_score(gpu):
    import torch

    w, shifts, kind, x, y, llr, syn = workload_inputs("C2", 128)
    counters = torch.zeros(5, dtype=torch.int64, device="cuda")
    code = gpu.QCCode(shifts, w.Z, kind)
    r = code.decode(torch.from_numpy(llr).cuda(), torch.from_numpy(syn).cuda(), w.max_iter, True,
                    counters=counters)
    errs = code.score(r["bits"], torch.from_numpy(x).cuda(), r["success"], counters=counters, want_errors=True)
    c = counters.cpu().numpy()
    o = oracle_decode(shifts, w.Z, llr, syn, w.max_iter, 1, want_state=False)
    ob = np.unpackbits(o["bits"] ^ x, axis=1, bitorder="little")[:, : w.n].sum(1)
    assert np.array_equal(errs.cpu().numpy(), ob)
    assert c[0] == 128 and c[1] == o["success"].sum() and c[4] == o["iters"].sum()
    assert c[2] == (ob > 0).sum() and c[3] == ((ob > 0) & (o["success"] == 1)).sum()


def test_reconcile_host_matches_device_path(gpu):
    import torch

    w, shifts, kind, x, y, llr, syn = workload_inputs("C4@0.04", 4)
    code = gpu.QCCode(shifts, w.Z, kind)
    bits, iters, succ = code.reconcile_host(w.qber, y, syn, w.max_iter, True, known_bits=x)
    o = oracle_decode(shifts, w.Z, llr, syn, w.max_iter, 1, want_state=False)
    assert np.array_equal(bits, o["bits"]) and np.array_equal(iters, o["iters"])
    assert np.array_equal(succ, o["success"])


def test_reconcile_host_pipelined_chunks(gpu):
    """qkd_reconcile_host on enough frames to run in several pipelined chunks (two internal copy
    streams chained by events): identical to the device-resident path (syndrome + LLR + decode), which
    the tests above pin to the oracle; unpinned host memory on purpose (numpy arrays)."""
    import torch

    w = synth.workload("C5b")
    F = 90001                                           # > 2 chunks of >= 16 waves; ragged last chunk
    x, y, _ = w.gen(0, F)
    code = gpu.QCCode(w.shifts(), w.Z)
    xs, ys = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    syn = code.syndrome(xs)
    r = code.decode(code.build_llr(w.qber, ys), syn, w.max_iter, True)
    bits, iters, succ = code.reconcile_host(w.qber, y, syn.cpu().numpy(), w.max_iter, True)
    assert np.array_equal(bits, r["bits"].cpu().numpy())
    assert np.array_equal(iters, r["iters"].cpu().numpy())
    assert np.array_equal(succ, r["success"].cpu().numpy())


@pytest.mark.parametrize("name", ["C5b", "C5a"])
def test_full_size_sampled(gpu, name):
    """BASELINE configs[4] at full size (65536 frames) in the bench's launch configuration;
    sampled frames against the oracle one by one, plus success => syndrome match on a
    4096-frame slice checked by the oracle's own syndrome."""
    import torch

    w = synth.workload(name)
    F = w.frames
    shifts = w.shifts()
    x, y, _ = w.gen(0, F)
    code = gpu.QCCode(shifts, w.Z)
    xs = torch.from_numpy(x).cuda()
    syn = code.syndrome(xs)
    llr = code.build_llr(w.qber, torch.from_numpy(y).cuda())
    r = to_np(code.decode(llr, syn, w.max_iter, True))
    oc = oracle.Code(shifts, w.Z)
    rng = np.random.default_rng(5)
    sample = np.unique(np.concatenate([[0, 1, 2, 3, F - 1], rng.integers(0, F, 11)]))
    xo, yo = x[sample], y[sample]
    so = oc.syndrome(xo)
    assert np.array_equal(so, syn.cpu().numpy()[sample])
    o = oc.decode(oc.build_llr(w.qber, yo), so, w.max_iter, 1, want_state=False)
    for k in ("bits", "iters", "success"):
        assert np.array_equal(r[k][sample], o[k]), k
    sl = slice(F - 4096, F)
    s_bits = oc.syndrome(r["bits"][sl])
    ok = r["success"][sl] == 1
    assert np.array_equal(s_bits[ok], syn.cpu().numpy()[sl][ok])


@pytest.mark.parametrize("name,per_shard", [("C5b", 512), ("C5a", 512)])
def test_full_size_every_shard_full_state(gpu, name, per_shard):
    """SURVEY §8(c) parity contract for C5: frames covering every rank's shard (8 ranks x 8192 frames;
    4096 frames of each workload), from the full 65536-frame
    launch in the bench's configuration, bit-exact in bits, iters, success and the final L and E."""
    import torch

    w = synth.workload(name)
    F = w.frames
    shifts = w.shifts()
    x, y, _ = w.gen(0, F)
    code = gpu.QCCode(shifts, w.Z)
    syn = code.syndrome(torch.from_numpy(x).cuda())
    llr = code.build_llr(w.qber, torch.from_numpy(y).cuda())
    r = code.decode(llr, syn, w.max_iter, True, want_state=True)
    shard = F // 8
    sample = np.concatenate([np.arange(k * shard, k * shard + per_shard) for k in range(8)])
    idx = torch.from_numpy(sample).cuda()
    g = {k: v.index_select(0, idx).cpu().numpy() for k, v in r.items()}
    del r
    oc = oracle.Code(shifts, w.Z)
    o = oc.decode(oc.build_llr(w.qber, y[sample]), oc.syndrome(x[sample]), w.max_iter, 1)
    assert_same(g, o)


@pytest.mark.parametrize("case", ["deg9to20", "Z96_multiwarp"])
@pytest.mark.parametrize("F", [1, 7])
def test_split_variant_parity_edge_cases(gpu, monkeypatch, case, F):
    """The lane-pair kernel (variant 5, QKD_SPLIT=1 at code creation): same bits, iterations and
    final L/E as the oracle, including odd degrees (side A's empty slot) and Z % 16 != 0."""
    monkeypatch.setenv("QKD_SPLIT", "1")
    shifts, Z = TINY[case]
    shifts = np.asarray(shifts, dtype=np.int32)
    Mb, Nb = shifts.shape
    n, m = Nb * Z, Mb * Z
    rng = np.random.default_rng(zlib.crc32(f"split/{case}/{F}".encode()))
    llr = rng.integers(-127, 128, size=(F, n)).astype(np.int8)
    syn = rng.integers(0, 256, size=(F, (m + 7) // 8), dtype=np.uint8)
    for T, es in ((0, 1), (1, 0), (9, 1)):
        g, code = gpu_decode(gpu, shifts, Z, None, llr, syn, T, es)
        assert code.launch_info(F)["variant"] % 10 == 5
        assert_same(g, oracle_decode(shifts, Z, llr, syn, T, es))


@pytest.mark.parametrize("name,F", [("C3", 12), ("C5a", 9)])
def test_split_variant_parity_workloads(gpu, monkeypatch, name, F):
    monkeypatch.setenv("QKD_SPLIT", "1")
    w, shifts, kind, x, y, llr, syn = workload_inputs(name, F)
    g, code = gpu_decode(gpu, shifts, w.Z, kind, llr, syn, w.max_iter, w.early_stop)
    assert code.launch_info(F)["variant"] == 15
    assert_same(g, oracle_decode(shifts, w.Z, llr, syn, w.max_iter, w.early_stop))


@pytest.mark.parametrize("case", ["deg30_Z40", "deg21to32_pow2"])
def test_degree32_variant_against_generic(gpu, monkeypatch, case):
    """Degrees 21..32 run on the register kernel (variant 6); QKD_NO_D32=1 forces the generic one:
    both must equal the oracle."""
    shifts, Z = TINY[case]
    shifts = np.asarray(shifts, dtype=np.int32)
    code = gpu.QCCode(shifts, Z)
    assert code.launch_info(8)["variant"] % 10 == 6
    n, m = shifts.shape[1] * Z, shifts.shape[0] * Z
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    llr = rng.integers(-127, 128, size=(8, n)).astype(np.int8)
    syn = rng.integers(0, 256, size=(8, (m + 7) // 8), dtype=np.uint8)
    o = oracle_decode(shifts, Z, llr, syn, 7, 1)
    g, _ = gpu_decode(gpu, shifts, Z, None, llr, syn, 7, 1)
    assert_same(g, o)
    monkeypatch.setenv("QKD_NO_D32", "1")
    assert gpu.QCCode(shifts, Z).launch_info(8)["variant"] % 10 == 3
    g, _ = gpu_decode(gpu, shifts, Z, None, llr, syn, 7, 1)
    assert_same(g, o)


@pytest.mark.parametrize("greg", ["1", "0"])
def test_global_e_variants(gpu, monkeypatch, greg):
    """C4 (E does not fit in shared memory, check degree <= 8): the register-row kernel with E in
    global memory (variant 7) and, with QKD_NO_GREG=1, the generic one (variant 4)."""
    if greg == "0":
        monkeypatch.setenv("QKD_NO_GREG", "1")
    w, shifts, kind, x, y, llr, syn = workload_inputs("C4@0.04", 5)
    g, code = gpu_decode(gpu, shifts, w.Z, kind, llr, syn, 9, 0)
    assert code.launch_info(5)["variant"] % 10 == (7 if greg == "1" else 4)
    o = oracle_decode(shifts, w.Z, llr, syn, 9, 0)
    assert_same(g, o)


@pytest.mark.parametrize("greg", ["1", "0"])
def test_global_e_high_degree_variant(gpu, monkeypatch, greg):
    """The N3 stable profile lifted to the paper's ~100 kb frames (n = 102400, check degree 27-28: E does
    not fit in shared memory): register rows with E in global memory (variant 8) and, with
    QKD_NO_GREG=1, the generic kernel (variant 4), on channel frames at 1.75 %."""
    if greg == "0":
        monkeypatch.setenv("QKD_NO_GREG", "1")
    cols = [8] * 16 + [3] * 21 + [2] * 13
    shifts = synth.girth6_shifts(synth.peg_mask(8, cols, 7), 2048, 8)
    oc = oracle.Code(shifts, 2048)
    x, y, _ = synth.frames(oc.n, 0.0175, 203, 0, 5)
    syn = oc.syndrome(x)
    llr = oc.build_llr(0.0175, y)
    g, code = gpu_decode(gpu, shifts, 2048, None, llr, syn, 50, 1)
    assert code.launch_info(5)["variant"] == (8 if greg == "1" else 4)
    o = oracle_decode(shifts, 2048, llr, syn, 50, 1)
    assert_same(g, o)


def test_stable_profile_code_parity(gpu):
    """The best stable degree profile of profiles/r1_degree_profiles.md (check degree 27-28, variant 6)
    on channel frames at QBER 1.75 %, bit-exact against the oracle."""
    import torch

    cols = [8] * 16 + [3] * 21 + [2] * 13
    shifts = synth.girth6_shifts(synth.peg_mask(8, cols, 7), 1024, 8)
    code = gpu.QCCode(shifts, 1024)
    assert code.launch_info(8)["variant"] == 16
    x, y, _ = synth.frames(50 * 1024, 0.0175, 203, 0, 6)
    oc = oracle.Code(shifts, 1024)
    syn = oc.syndrome(x)
    llr = oc.build_llr(0.0175, y)
    g, _ = gpu_decode(gpu, shifts, 1024, None, llr, syn, 50, 1)
    o = oracle_decode(shifts, 1024, llr, syn, 50, 1)
    assert_same(g, o)


@pytest.mark.parametrize("name,F", [("C1", 64), ("C2", 192), ("C3", 12), ("C4@0.08", 4)])
def test_refill_variant_parity(gpu, monkeypatch, name, F):
    """Per-frame lane refill (QKD_REFILL=1): every frame's bits, iterations, success and final L/E
    are the oracle's, whatever frames share its 4-lane group and whenever its lane was refilled."""
    monkeypatch.setenv("QKD_REFILL", "1")
    w, shifts, kind, x, y, llr, syn = workload_inputs(name, F)
    for T, es in ((w.max_iter, 1), (3, 0), (0, 1)):
        g, code = gpu_decode(gpu, shifts, w.Z, kind, llr, syn, T, es)
        assert_same(g, oracle_decode(shifts, w.Z, llr, syn, T, es))


@pytest.mark.parametrize("case", sorted(TINY))
def test_refill_variant_edge_cases(gpu, monkeypatch, case):
    monkeypatch.setenv("QKD_REFILL", "1")
    shifts, Z = TINY[case]
    shifts = np.asarray(shifts, dtype=np.int32)
    Mb, Nb = shifts.shape
    n, m = Nb * Z, Mb * Z
    rng = np.random.default_rng(zlib.crc32(f"refill/{case}".encode()))
    F = 23
    llr = rng.integers(-127, 128, size=(F, n)).astype(np.int8)
    llr[::3] = np.where(rng.random((len(llr[::3]), n)) < 0.9, 100, -100)   # some frames converge fast
    syn = rng.integers(0, 256, size=(F, (m + 7) // 8), dtype=np.uint8)
    syn[::3] = 0
    for T, es in ((9, 1), (1, 0)):
        g, _ = gpu_decode(gpu, shifts, Z, None, llr, syn, T, es)
        assert_same(g, oracle_decode(shifts, Z, llr, syn, T, es))


def test_de_profile_code_parity(gpu):
    """The density-evolution profile of profiles/r2_density_evolution.md (base 16 x 100, Z = 512,
    n = 51200, rate 0.84; column degrees 2:10, 3:66, 12:24; check degree 31-32, variant 6) built as
    tools/de_codes.py builds it, on channel frames at QBER 1.8 %, bit-exact against the oracle."""
    cols = [12] * 24 + [3] * 66 + [2] * 10
    shifts = synth.girth6_shifts(synth.peg_mask(16, cols, 7), 512, 8)
    code = gpu.QCCode(shifts, 512)
    assert code.launch_info(8)["variant"] == 16
    x, y, _ = synth.frames(100 * 512, 0.018, 203, 0, 6)
    oc = oracle.Code(shifts, 512)
    syn = oc.syndrome(x)
    llr = oc.build_llr(0.018, y)
    g, _ = gpu_decode(gpu, shifts, 512, None, llr, syn, 50, 1)
    o = oracle_decode(shifts, 512, llr, syn, 50, 1)
    assert_same(g, o)
