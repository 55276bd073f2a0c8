"""Conformal order and brute-force Graver bases (oracle).

Def. 1: x ⊑ y iff x_i y_i >= 0 and |x_i| <= |y_i| for all i.
Def. 2: G(A) = the ⊑-minimal elements of Ker_Z(A) \\ {0}.
§3.1: the finite test set Ker_Z(A) ∩ M with M = [l - u, u - l].

enumerate_kernel_in_box is a plain product-space scan (tiny n only); graver_in_box keeps the ⊑-minimal
elements of it by the definition (pairwise test). When the box contains M, graver_in_box(A, M) is
G(A) ∩ M, the part of the Graver basis usable under bounds l, u.
"""
from __future__ import annotations

import itertools

import numpy as np


def conforms(x, y) -> bool:
    """x ⊑ y (Def. 1)."""
    x = np.asarray(x)
    y = np.asarray(y)
    if x.shape != y.shape:
        raise ValueError("LengthMismatch")
    return bool(np.all(x * y >= 0) and np.all(np.abs(x) <= np.abs(y)))


def enumerate_kernel_in_box(A, lo, hi, budget: int = 5_000_000):
    """{g in Z^n : A g = 0, lo <= g <= hi, g != 0} by scanning the box (product enumeration)."""
    A = np.asarray(A, dtype=np.int64)
    lo = np.asarray(lo, dtype=np.int64)
    hi = np.asarray(hi, dtype=np.int64)
    size = int(np.prod(hi - lo + 1))
    if size > budget:
        raise ValueError("TooLarge")
    axes = [range(int(a), int(b) + 1) for a, b in zip(lo, hi)]
    out = []
    # vectorised over the last coordinate block to keep the scan fast yet plain
    G = np.array(list(itertools.product(*axes)), dtype=np.int64)
    mask = np.all(G @ A.T == 0, axis=1) & np.any(G != 0, axis=1)
    for g in G[mask]:
        out.append(tuple(int(v) for v in g))
    return set(out)


def minimal_elements(S):
    """The ⊑-minimal elements of a finite set S of integer tuples (Def. 2 applied to S)."""
    S = list(S)
    if not S:
        return set()
    M = np.array(S, dtype=np.int64)
    keep = set()
    for i, g in enumerate(M):
        dom = np.all(M * g >= 0, axis=1) & np.all(np.abs(M) <= np.abs(g), axis=1)
        dom[i] = False
        if not dom.any():
            keep.add(S[i])
    return keep


def graver_in_box(A, lo, hi, budget: int = 5_000_000):
    """G(A) ∩ [lo, hi] by Def. 2 over the enumerated box (SPEC graver_oracle)."""
    return minimal_elements(enumerate_kernel_in_box(A, lo, hi, budget))


def canonical(g):
    """Sign-twin representative: the one of {g, -g} whose first nonzero entry is positive."""
    g = tuple(int(v) for v in g)
    for v in g:
        if v != 0:
            return g if v > 0 else tuple(-x for x in g)
    return g
