"""Exact integer lattice algorithms (oracle). Python ints / Fractions only — no floating point except pinv.

PAPER.md §2.2: lattice L(B), Hermite normal form (Def. P:124-126, Prop. 1),
Gram-Schmidt orthogonalisation, reduced basis (Def. P:136-144), LLL (Alg. 1).
§4.1: C = (D | B) from the HNF, Theorem 1 (Ker_Z(A) = L(B)), pseudoinverse remark.

Readings: HNF pivot rule = smallest nonzero |entry| in the pivot row, ties leftmost
(SPEC S:98); Alg. 1 control flow per SURVEY §8(c)-2 #5 (fully size-reduce b_k against j=k-1..1, then the
Siegel test ||B*_{k-1}||^2 > 2 ||B*_k||^2 -> swap and k <- max(k-1, 2), else k <- k+1).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


class RankDeficient(ValueError):
    pass


class FullRankKernel(ValueError):
    pass


def _mat(A):
    return [[int(v) for v in row] for row in np.asarray(A).tolist()]


def hnf(A):
    """Column-style HNF (Prop. 1): returns (H, C) with A C = (H | 0), C unimodular,
    H lower-triangular, h_ii > 0, 0 <= h_ij < h_ii for j < i (Def. P:124-126). Raises RankDeficient."""
    M = _mat(A)
    m, n = len(M), len(M[0])
    C = [[int(i == j) for j in range(n)] for i in range(n)]

    def col_axpy(j, p, q):  # col_j -= q * col_p, in M and C
        for r in range(m):
            M[r][j] -= q * M[r][p]
        for r in range(n):
            C[r][j] -= q * C[r][p]

    def col_swap(i, j):
        for r in range(m):
            M[r][i], M[r][j] = M[r][j], M[r][i]
        for r in range(n):
            C[r][i], C[r][j] = C[r][j], C[r][i]

    def col_neg(i):
        for r in range(m):
            M[r][i] = -M[r][i]
        for r in range(n):
            C[r][i] = -C[r][i]

    for i in range(m):
        while True:
            nz = [j for j in range(i, n) if M[i][j] != 0]
            if not nz:
                raise RankDeficient(f"row {i} has no pivot (rank(A) < m)")
            if len(nz) == 1:
                break
            p = min(nz, key=lambda j: (abs(M[i][j]), j))
            for j in nz:
                if j != p:
                    col_axpy(j, p, M[i][j] // M[i][p])
        col_swap(i, nz[0])
        if M[i][i] < 0:
            col_neg(i)
        for j in range(i):
            col_axpy(j, i, M[i][j] // M[i][i])
    H = [row[:m] for row in M]
    return H, C


def kernel_basis(A):
    """B = last d = n - m columns of C (Thm. 1 setup; Alg. 3 line 2-3). Returns n x d list."""
    A = np.asarray(A)
    m, n = A.shape
    if m >= n:
        raise FullRankKernel("d = n - m = 0: the kernel is {0}")
    _, C = hnf(A)
    return [row[m:] for row in C]


def _cols(B):
    B = _mat(B)
    n, d = len(B), len(B[0])
    return [[B[r][j] for r in range(n)] for j in range(d)]


def _uncols(cols):
    n, d = len(cols[0]), len(cols)
    return [[cols[j][r] for j in range(d)] for r in range(n)]


def _dot(x, y):
    return sum(a * b for a, b in zip(x, y))


def gram_schmidt(B):
    """Exact GSO (with the B_J^* typo read as B_j^*): returns (Bstar, mu) over Fractions,
    B_i^* = B_i - sum_{j<i} mu_ij B_j^*, mu_ij = <B_i, B_j^*> / <B_j^*, B_j^*>."""
    cols = _cols(B)
    d = len(cols)
    bstar, mu = [], [[Fraction(0)] * d for _ in range(d)]
    for i in range(d):
        v = [Fraction(x) for x in cols[i]]
        for j in range(i):
            nj = _dot(bstar[j], bstar[j])
            if nj == 0:
                raise RankDeficient("dependent columns")
            mu[i][j] = _dot(cols[i], bstar[j]) / nj
            v = [a - mu[i][j] * b for a, b in zip(v, bstar[j])]
        bstar.append(v)
    for v in bstar:
        if all(x == 0 for x in v):
            raise RankDeficient("dependent columns")
    return bstar, mu


def is_lll_reduced(B):
    """Def. 'reduced basis', exactly: (i) |mu_ij| <= 1/2 for j < i; (ii) ||B_j^*||^2 <=
    2 ||B_{j+1}^*||^2."""
    bstar, mu = gram_schmidt(B)
    d = len(bstar)
    for i in range(d):
        for j in range(i):
            if abs(mu[i][j]) > Fraction(1, 2):
                return False
    for j in range(d - 1):
        if _dot(bstar[j], bstar[j]) > 2 * _dot(bstar[j + 1], bstar[j + 1]):
            return False
    return True


def lll_reduce(B):
    """LLL (Alg. 1) with the Siegel swap test of the paper (factor 2), in exact integer
    arithmetic (integral-GSO bookkeeping: d_i = prod_{j<=i} ||B_j^*||^2, lam_ij = d_j mu_ij).
    Input / output: n x d integer matrix (columns = basis vectors)."""
    b = _cols(B)
    d = len(b)
    if d <= 1:
        return _uncols(b)
    # D[i+1] = d_i (D[0] = 1); lam[k][j] for j < k
    D = [1] + [0] * d
    lam = [[0] * d for _ in range(d)]
    kmax = -1

    def gso_row(k):
        for j in range(k + 1):
            u = _dot(b[k], b[j])
            for i in range(j):
                u = (D[i + 1] * u - lam[k][i] * lam[j][i]) // D[i]
            if j < k:
                lam[k][j] = u
            else:
                if u == 0:
                    raise RankDeficient("dependent columns")
                D[k + 1] = u

    def red(k, l):
        # size-reduce b_k against b_l: q = nearest integer to mu_kl = lam_kl / d_l (half up)
        dl = D[l + 1]
        if 2 * abs(lam[k][l]) > dl:
            q = (2 * lam[k][l] + dl) // (2 * dl)
            b[k] = [x - q * y for x, y in zip(b[k], b[l])]
            lam[k][l] -= q * dl
            for i in range(l):
                lam[k][i] -= q * lam[l][i]

    def swap(k):
        b[k], b[k - 1] = b[k - 1], b[k]
        for j in range(k - 1):
            lam[k][j], lam[k - 1][j] = lam[k - 1][j], lam[k][j]
        lk = lam[k][k - 1]
        Bn = (D[k - 1] * D[k + 1] + lk * lk) // D[k]
        for i in range(k + 1, kmax + 1):
            t = lam[i][k]
            lam[i][k] = (D[k + 1] * lam[i][k - 1] - lk * t) // D[k]
            lam[i][k - 1] = (Bn * t + lk * lam[i][k]) // D[k + 1]
        D[k] = Bn

    gso_row(0)
    kmax = 0
    k = 1
    while k < d:
        if k > kmax:
            kmax = k
            gso_row(k)
        for l in range(k - 1, -1, -1):
            red(k, l)
        # Siegel: ||B*_{k-1}||^2 = D[k]/D[k-1] > 2 ||B*_k||^2 = 2 D[k+1]/D[k]
        if D[k] * D[k] > 2 * D[k + 1] * D[k - 1]:
            swap(k)
            k = max(k - 1, 1)
        else:
            k += 1
    return _uncols(b)


def pinv(B):
    """B^{-1} := (B^T B)^{-1} B^T in fp64 (Remark P:321-324); a library solve is the step."""
    Bf = np.asarray(B, dtype=np.float64)
    return np.linalg.solve(Bf.T @ Bf, Bf.T)


def bareiss_det(M):
    """Exact determinant by fraction-free Gaussian elimination (used for saturation checks)."""
    M = _mat(M)
    n = len(M)
    sign, prev = 1, 1
    for k in range(n - 1):
        if M[k][k] == 0:
            sw = next((r for r in range(k + 1, n) if M[r][k] != 0), None)
            if sw is None:
                return 0
            M[k], M[sw] = M[sw], M[k]
            sign = -sign
        for i in range(k + 1, n):
            for j in range(k + 1, n):
                M[i][j] = (M[i][j] * M[k][k] - M[i][k] * M[k][j]) // prev
        prev = M[k][k]
    return sign * M[n - 1][n - 1]


def is_kernel_basis(A, B) -> bool:
    """Thm. 1 as a check: A B = 0 exactly, rank d = n - m, and L(B) = Ker_Z(A) (saturation:
    the HNF of B^T has unit diagonal, i.e. the gcd of the d x d minors of B is 1)."""
    A = np.asarray(A, dtype=object)
    Bm = np.asarray(_mat(B), dtype=object)
    m, n = A.shape
    if Bm.shape != (n, n - m):
        return False
    if np.any(A.dot(Bm) != 0):
        return False
    try:
        H, _ = hnf(Bm.T)
    except RankDeficient:
        return False
    return all(H[i][i] == 1 for i in range(len(H)))
