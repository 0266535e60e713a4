"""Code construction ("girth ... at least 6", "standard PEG algorithm"; SPEC
code-model S:60-78): PEG base masks and girth >= 6 circulant shifts, checked by an exact
breadth-first girth computation on the expanded Tanner graph (independent of the construction)."""
from collections import deque

import numpy as np
import pytest

import oracle
import synth


def girth_of(H: np.ndarray) -> float:
    """Exact girth of the Tanner graph of H (inf for a forest): BFS from every node; a non-tree edge
    between u and v closes a cycle of length d(u) + d(v) + 1 through the root's BFS tree."""
    m, n = H.shape
    adj = [[] for _ in range(n + m)]
    for i, j in zip(*np.nonzero(H)):
        adj[j].append(n + i)
        adj[n + i].append(j)
    best = np.inf
    for root in range(n + m):
        dist = {root: 0}
        parent = {root: -1}
        q = deque([root])
        while q:
            u = q.popleft()
            for v in adj[u]:
                if v not in dist:
                    dist[v] = dist[u] + 1
                    parent[v] = u
                    q.append(v)
                elif parent[u] != v:
                    best = min(best, dist[u] + dist[v] + 1)
    return best


def expand(shifts, Z):
    oc = oracle.Code(np.asarray(shifts, dtype=np.int32), Z)
    rows, cols = oc.expand()
    H = np.zeros((oc.m, oc.n), dtype=np.uint8)
    H[rows, cols] = 1
    return H


def test_girth_of_spec_examples():
    assert girth_of(np.ones((2, 2), dtype=np.uint8)) == 4                 # smallest Tanner cycle
    assert girth_of(np.hstack([np.eye(3), np.eye(3)]).astype(np.uint8)) == np.inf   # [I | I]: forest
    H = np.array([[1, 1, 0], [0, 1, 1], [1, 0, 1]], dtype=np.uint8)      # one 6-cycle
    assert girth_of(H) == 6


@pytest.mark.parametrize("Mb,Nb,Z,fracs,seed", [
    (4, 8, 16, {2: 0.5, 3: 0.5}, 1),
    (6, 12, 24, {3: 1.0}, 2),
    (8, 16, 32, {2: 0.45, 3: 0.35, 6: 0.2}, 3),
])
def test_peg_girth6_codes(Mb, Nb, Z, fracs, seed):
    sh = synth.peg_qc_code(Mb, Nb, Z, fracs, seed)
    cnt = synth.degree_counts(Nb, fracs)
    col = (sh >= 0).sum(axis=0)
    assert sorted(col.tolist()) == sorted(d for d, c in cnt.items() for _ in range(c))
    rows = (sh >= 0).sum(axis=1)
    assert rows.max() - rows.min() <= 2                                   # PEG balances check degrees
    assert girth_of(expand(sh, Z)) >= 6


def test_q17_rule_codes_do_have_4_cycles():
    """Contrast: the BASELINE config rule (uniform shifts, no filter, Q17) leaves 4-cycles at small Z."""
    sh = synth.qc_code(6, 12, 8, {3: 1.0}, 5)
    assert girth_of(expand(sh, 8)) == 4
