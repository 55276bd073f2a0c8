"""Pins for oracle/graver.py and oracle/postprocess.py: SPEC examples, closed-form Graver
bases (all-ones rows, semi-assignment, 3x3 assignment circuits, primitive partition identities),
Prop. 2 Graver expression, and the filter's edge cases."""
import itertools
import math

import numpy as np
import pytest

from oracle import graver as Gv
from oracle import postprocess as PP


def _pm(S):
    return S | {tuple(-v for v in g) for g in S}


def test_conforms_examples():
    assert Gv.conforms((1, -1), (2, -2))
    assert not Gv.conforms((1, 1), (2, -2))
    assert Gv.conforms((0, 0), (5, -7))
    with pytest.raises(ValueError):
        Gv.conforms((1,), (1, 2))


def test_enumerate_examples():
    assert Gv.enumerate_kernel_in_box([[1, 1]], [-2, -2], [2, 2]) == {(1, -1), (-1, 1), (2, -2), (-2, 2)}
    assert Gv.enumerate_kernel_in_box([[1, 1]], [0, 0], [2, 2]) == set()
    assert Gv.enumerate_kernel_in_box([[1, 2]], [-2, -2], [2, 2]) == {(2, -1), (-2, 1)}


def test_graver_examples():
    assert Gv.graver_in_box([[1, 1]], [-3] * 2, [3] * 2) == {(1, -1), (-1, 1)}
    assert Gv.graver_in_box([[1, 1, 1]], [-2] * 3, [2] * 3) == _pm({(1, -1, 0), (1, 0, -1), (0, 1, -1)})
    assert Gv.graver_in_box([[1, 2]], [-4] * 2, [4] * 2) == {(2, -1), (-2, 1)}


def _ei_ej(n, groups):
    S = set()
    for g in groups:
        for i, j in itertools.combinations(g, 2):
            v = [0] * n
            v[i], v[j] = 1, -1
            S.add(tuple(v))
    return S


def test_all_ones_closed_form():
    """Graver basis of the 1 x 4 all-ones row = {e_i - e_j}: 12 elements (BASELINE configs[0])."""
    G = Gv.graver_in_box([[1, 1, 1, 1]], [-3] * 4, [3] * 4)
    assert G == _pm(_ei_ej(4, [range(4)]))
    assert len(G) == 12


def test_semi_assignment_closed_form():
    A = [[1, 1, 1, 0, 0, 0], [0, 0, 0, 1, 1, 1]]
    G = Gv.graver_in_box(A, [-1] * 6, [1] * 6)
    assert G == _pm(_ei_ej(6, [range(3), range(3, 6)]))
    assert len(G) == 12


def test_assignment_3x3_circuits():
    """3x3 assignment (totally unimodular): Graver = circuits = alternating cycles of K_{3,3}:
    2 * sum_j C(3,j)^2 (j!)^2 / (2j) = 30 elements."""
    from synth import assignment
    inst = assignment(3)
    G = Gv.graver_in_box(inst.A, [-1] * 9, [1] * 9)
    k = 3
    assert len(G) == 2 * sum(math.comb(k, j) ** 2 * math.factorial(j) ** 2 // (2 * j) for j in range(2, k + 1))


@pytest.mark.parametrize("k,expected", [
    (2, {(2, -1)}),
    (3, {(2, -1, 0), (3, 0, -1), (1, 1, -1), (1, -2, 1), (0, 3, -2)}),
])
def test_primitive_partition_identities(k, expected):
    A = [list(range(1, k + 1))]
    G = Gv.graver_in_box(A, [-4] * k, [4] * k)
    assert {Gv.canonical(g) for g in G} == expected


def test_primitive_partition_identities_1234_stable():
    A = [[1, 2, 3, 4]]
    G4 = {Gv.canonical(g) for g in Gv.graver_in_box(A, [-4] * 4, [4] * 4)}
    G5 = {Gv.canonical(g) for g in Gv.graver_in_box(A, [-5] * 4, [5] * 4)}
    assert G4 == G5 and len(G4) == 15


@pytest.mark.parametrize("seed", range(12))
def test_oracle_suite_minimal_negation_closed_complete(seed):
    """SPEC acceptance #4: minimal, negation-closed and complete on random small A."""
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 3))
    n = int(rng.integers(m + 1, 5))
    A = rng.integers(-3, 4, size=(m, n))
    K = Gv.enumerate_kernel_in_box(A, [-3] * n, [3] * n)
    G = Gv.minimal_elements(K)
    assert G == {tuple(-v for v in g) for g in G}
    for g in G:
        assert not any(h != g and Gv.conforms(h, g) for h in G)
    for y in K:
        assert any(Gv.conforms(g, y) for g in G)


@pytest.mark.parametrize("seed", range(8))
def test_prop2_graver_expression(seed):
    """Prop. 2(i): x - xbar is a sign-compatible sum of Graver elements ⊑ it (greedy peel)."""
    from synth import random_small
    inst = random_small(1, 4, seed, lo=-2, hi=3, ubox=2)
    M = (inst.u - inst.l).tolist()
    G = Gv.graver_in_box(inst.A, [-v for v in M], M)
    pts = [np.array(p) for p in itertools.product(*[range(int(a), int(b) + 1) for a, b in zip(inst.l, inst.u)])
           if np.all(inst.A @ np.array(p) == inst.b)]
    rng = np.random.default_rng(seed)
    for _ in range(10):
        x, xb = pts[rng.integers(len(pts))], pts[rng.integers(len(pts))]
        dvec = tuple(int(v) for v in x - xb)
        steps = 0
        while any(dvec):
            g = next(g for g in G if Gv.conforms(g, dvec))
            dvec = tuple(a - b for a, b in zip(dvec, g))
            steps += 1
        assert steps <= 2 * 4 * 4


# ---- postprocess: filter by definition, pinned against the closed forms above ----

def test_filter_reproduces_closed_form_from_kernel_box():
    K = Gv.enumerate_kernel_in_box([[1, 1, 1, 1]], [-3] * 4, [3] * 4)
    S = PP.dedupe(list(K))
    assert PP.minimal_filter(S) == _ei_ej(4, [range(4)])


def test_filter_edge_cases():
    assert PP.minimal_filter(set()) == set()
    assert PP.minimal_filter({(1, -1)}) == {(1, -1)}
    # sign-twin domination: (1,0,-1) dominates (2,0,-2) and, through -g, nothing else
    S = {(1, 0, -1), (2, 0, -2), (1, -1, 0)}
    keep, wit = PP.minimal_filter(S, return_witness=True)
    assert keep == {(1, 0, -1), (1, -1, 0)}
    assert wit == {(2, 0, -2): (1, 0, -1)}
    # -h ⊑ g: canonical (1,-1) dominates (−1,1)'s canonical twin; (0,1,1,-2) is dominated by (0,-0,...)?
    S = {(0, 1, -1, 0), (1, -1, 0, 1)}
    assert PP.minimal_filter(S) == S
    S = {(0, 1, -1), (1, -2, 2)}      # -(0,1,-1) = (0,-1,1) ⊑ (1,-2,2)
    assert PP.minimal_filter(S) == {(0, 1, -1)}
    assert PP.is_antichain({(0, 1, -1), (1, 0, 0)})
    assert not PP.is_antichain({(0, 1, -1), (1, -2, 2)})


def test_check_rows_and_dedupe():
    A = np.array([[1, 1, 1]])
    rows = np.array([[1, -1, 0], [-1, 1, 0], [1, 1, 0], [0, 0, 0], [3, -3, 0], [2, -1, -1]])
    ok = PP.check_rows(A, np.zeros(3), np.full(3, 2), rows)
    assert ok.tolist() == [True, True, False, False, False, True]
    assert PP.dedupe(rows[ok]) == {(1, -1, 0), (2, -1, -1)}
    assert Gv.canonical((0, -2, 1)) == (0, 2, -1)
