"""Pins of tools/de_search.py, the density evolution behind SURVEY §8(f) N3 (profiles/r2_density_evolution.md).
CPU only, a few seconds."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import de_search as de  # noqa: E402


def test_tau_is_algorithm_1():
    """The tool's tau is Algorithm 1: spot values worked by hand from the pseudo-code."""
    assert de.tau(10, 10) == 8            # l = 10 > 2, d = 0: 10 - 1 - 1
    assert de.tau(10, 13) == 9            # d = 3: 10 - 0 - 1
    assert de.tau(10, 17) == 10           # d = 7: no correction
    assert de.tau(2, 2) == 1 and de.tau(2, 7) == 2 and de.tau(1, 1) == 0 and de.tau(0, 40) == 0
    assert de.tau(100, 200) == de.tau(63, 63) == 61   # inputs clamp to MSG_max = 63


def test_pairwise_check_combination_is_exact():
    """cnode() is the exact distribution of sign(a) sign(b) tau(|a|, |b|): compare with enumeration."""
    rng = np.random.default_rng(5)
    Pa = rng.random(de.NV); Pa /= Pa.sum()
    Pb = rng.random(de.NV); Pb /= Pb.sum()
    ref = np.zeros(de.NV)
    for i, a in enumerate(range(-63, 64)):
        for j, b in enumerate(range(-63, 64)):
            s = (1 if a > 0 else -1) * (1 if b > 0 else -1)
            ref[s * de.tau(abs(a), abs(b)) + 63] += Pa[i] * Pb[j]
    assert np.allclose(de.cnode(Pa, Pb), ref, atol=1e-15)


def test_variable_node_of_a_degree_1_column_is_the_clamped_channel():
    Q = np.zeros(de.NV); Q[63] = 1.0      # no check information
    out = de.var_out(Q, 1, 16, 0.02)
    assert math.isclose(out[63 + 16], 0.98) and math.isclose(out[63 - 16], 0.02)
    out = de.var_out(Q, 2, 100, 0.02)     # |LLR| > 63 clamps to the message range
    assert math.isclose(out[126], 0.98) and math.isclose(out[0], 0.02)


def test_thresholds_order_the_measured_profiles():
    """DE reproduces what the GPU measured (profiles/r1_degree_profiles.md, r2_density_evolution.md):
    C3's profile fails at 1 % while the round-1 Monte-Carlo best converges at 1.5 % and fails at 2 %."""
    assert not de.run_de({2: 25, 3: 20, 6: 5}, 8, 0.01, 100)[0]
    assert de.run_de({2: 13, 3: 21, 8: 16}, 8, 0.015, 100)[0]
    assert not de.run_de({2: 13, 3: 21, 8: 16}, 8, 0.02, 100)[0]


def test_profile_edge_perspective():
    lam, rho, E = de.profile({2: 13, 3: 21, 8: 16}, 8)
    assert E == 217 and math.isclose(sum(lam.values()), 1.0) and math.isclose(sum(rho.values()), 1.0)
    assert set(rho) == {27, 28} and math.isclose(rho[28], 28 * 1 / 217)   # 217 = 7 x 27 + 1 x 28
