"""Pins for oracle/lattice.py: SPEC worked examples, Prop. 1 invariants, Def. 'reduced basis'
(P:136-144), Theorem 1. Independent checkers (exact rational solves, Bareiss det) written here."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import lattice as L


def _matmul(A, B):
    return [[sum(A[i][k] * B[k][j] for k in range(len(B))) for j in range(len(B[0]))] for i in range(len(A))]


def _exact_solve(B1, B2):
    """X with B1 X = B2 over the rationals (B1 full column rank), via normal equations."""
    n, d = len(B1), len(B1[0])
    G = [[Fraction(sum(B1[r][i] * B1[r][j] for r in range(n))) for j in range(d)] for i in range(d)]
    R = [[Fraction(sum(B1[r][i] * B2[r][j] for r in range(n))) for j in range(len(B2[0]))] for i in range(d)]
    M = [G[i] + R[i] for i in range(d)]
    for c in range(d):
        p = next(r for r in range(c, d) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        M[c] = [x / M[c][c] for x in M[c]]
        for r in range(d):
            if r != c and M[r][c] != 0:
                M[r] = [a - M[r][c] * b for a, b in zip(M[r], M[c])]
    return [row[d:] for row in M]


def same_lattice(B1, B2) -> bool:
    X = _exact_solve(B1, B2)
    if any(x.denominator != 1 for row in X for x in row):
        return False
    Xi = [[int(x) for x in row] for row in X]
    if _matmul(B1, Xi) != [list(map(int, r)) for r in B2]:
        return False
    return abs(L.bareiss_det(Xi)) == 1


def test_hnf_spec_examples():
    H, C = L.hnf([[1, 0], [0, 1]])
    assert H == [[1, 0], [0, 1]] and C == [[1, 0], [0, 1]]
    H, C = L.hnf([[2, 4, 4]])
    assert H == [[2]]                                                # S:51, gcd(2,4,4) = 2
    assert _matmul([[2, 4, 4]], C) == [[2, 0, 0]]
    H, C = L.hnf([[3, 1], [1, 2]])
    assert H == [[1, 0], [2, 5]]
    assert abs(L.bareiss_det(C)) == 1


def test_hnf_rank_deficient():
    with pytest.raises(L.RankDeficient):
        L.hnf([[1, 2, 3], [2, 4, 6]])


@pytest.mark.parametrize("seed", range(60))
def test_hnf_random_suite(seed):
    """SPEC acceptance #1: A C = (H|0) exactly, H normalised, |det C| = 1."""
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 6))
    n = int(rng.integers(m, 9))
    while True:
        A = rng.integers(-9, 10, size=(m, n))
        if np.linalg.matrix_rank(A.astype(float)) == m:
            break
    H, C = L.hnf(A)
    AC = _matmul(A.tolist(), C)
    for i in range(m):
        assert AC[i][m:] == [0] * (n - m)
        assert AC[i][:m] == H[i]
        assert H[i][i] > 0
        for j in range(m):
            if j > i:
                assert H[i][j] == 0
            elif j < i:
                assert 0 <= H[i][j] < H[i][i]
    assert abs(L.bareiss_det(C)) == 1


def test_kernel_basis_examples():
    B = L.kernel_basis([[1, 1]])
    assert [r[0] for r in B] in ([1, -1], [-1, 1])
    B = L.kernel_basis([[1, 2]])
    assert [r[0] for r in B] in ([2, -1], [-2, 1])
    with pytest.raises(L.FullRankKernel):
        L.kernel_basis([[1, 0], [0, 1]])


def test_gso_examples():
    bstar, mu = L.gram_schmidt([[1, 0], [0, 1]])
    assert bstar == [[1, 0], [0, 1]] and mu[1][0] == 0
    bstar, mu = L.gram_schmidt([[1, 1], [0, 1]])                     # columns (1,0), (1,1)
    assert bstar[1] == [0, 1] and mu[1][0] == 1


def test_lll_examples():
    assert L.lll_reduce([[1, 0], [0, 1]]) == [[1, 0], [0, 1]]
    assert L.lll_reduce([[1, 1], [0, 1]]) == [[1, 0], [0, 1]]        # (1,0),(1,1) -> (1,0),(0,1)
    assert L.lll_reduce([[3], [4]]) == [[3], [4]]                    # S:79 single column
    assert L.is_lll_reduced([[1, 0], [0, 1]])
    assert not L.is_lll_reduced([[1, 1], [0, 1]])                    # S:87 (mu = 1 > 1/2)


@pytest.mark.parametrize("seed", range(40))
def test_lll_random_suite(seed):
    """SPEC acceptance #2: output reduced (exact rational recheck) and spans the same lattice."""
    rng = np.random.default_rng(100 + seed)
    d = int(rng.integers(1, 6))
    n = int(rng.integers(d, 9))
    while True:
        B = rng.integers(-9, 10, size=(n, d))
        if np.linalg.matrix_rank(B.astype(float)) == d:
            break
    R = L.lll_reduce(B)
    assert L.is_lll_reduced(R)
    assert same_lattice(B.tolist(), R) and same_lattice(R, B.tolist())


def test_siegel_condition_is_the_papers():
    """Def. (ii) is Siegel's factor 2, not Lovasz delta=3/4: a basis with ||B1*||^2 = 2 ||B2*||^2 and
    |mu| <= 1/2 is reduced."""
    B = [[2, 0], [0, 1], [0, 1]]     # columns (2,0,0), (0,1,1): ||B1*||^2 = 4, ||B2*||^2 = 2
    assert L.is_lll_reduced(B)
    assert L.lll_reduce(B) == B


@pytest.mark.parametrize("seed", range(40))
def test_theorem1_isomorphism(seed):
    """SPEC acceptance #3 + Thm. 1: A(Bz) = 0, B is a basis of Ker_Z(A), and B^+(Bz) = z."""
    rng = np.random.default_rng(500 + seed)
    m = int(rng.integers(1, 4))
    n = int(rng.integers(m + 1, 8))
    while True:
        A = rng.integers(-4, 5, size=(m, n))
        if np.linalg.matrix_rank(A.astype(float)) == m:
            break
    B = L.lll_reduce(L.kernel_basis(A))
    assert L.is_kernel_basis(A, B)
    Bn = np.array(B, dtype=np.int64)
    z = rng.integers(-3, 4, size=Bn.shape[1])
    g = Bn @ z
    assert np.all(A @ g == 0)
    np.testing.assert_allclose(L.pinv(B) @ g, z, atol=1e-9)


def test_kernel_basis_detects_non_saturated():
    A = [[1, 1, 1]]
    B = [[2, 0], [-2, 1], [0, -1]]     # columns 2(e1-e2) and e2-e3: index-2 sublattice
    assert not L.is_kernel_basis(A, B)
    assert L.is_kernel_basis(A, [[1, 0], [-1, 1], [0, -1]])


def test_bareiss_against_closed_forms():
    assert L.bareiss_det([[2, 0], [0, 3]]) == 6
    assert L.bareiss_det([[0, 1], [1, 0]]) == -1
    assert L.bareiss_det([[1, 2], [2, 4]]) == 0
    V = [[i ** j for j in range(4)] for i in range(1, 5)]   # Vandermonde: prod_{i<j}(x_j - x_i) = 12
    assert L.bareiss_det(V) == 12
