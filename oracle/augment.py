"""Graver-best augmentation (Alg. 2) and MAPLE's multi-start best (§4.3) — oracle.

Objective convention f(x) = 1/2 x^T Q x + c^T x + c0 (reading #20), or a separable
f(x) = c0 + sum_j f_j(x_j) given by value tables over the box (Prop. 3; reading #27). When Q, c and c0 are
integer-valued the comparison uses 2 f(x) in exact Python integers (no rounding at all); otherwise fp64.

Readings: #17 steps (g, lambda) with g in D = S ∪ -S (both signs), lambda in Z_+ = {1, 2, ...},
x + lambda g in S (bounds; A g = 0 keeps Ax = b), strict improvement f(x + lambda g) < f(x); the argmin
over f(x + lambda g) breaks ties by lexicographically smallest g (in D's sorted order), then smaller lambda.
#18 every lambda in [1, lambda_max(x, g)] is evaluated (lambda_max <= max(u - l) in the configs; a step cap
guards wide boxes). #19 the multi-start best breaks ties by lexicographically smallest x.
"""
from __future__ import annotations

import math

import numpy as np


class InfeasibleStart(ValueError):
    pass


def _integral(a) -> bool:
    a = np.asarray(a, dtype=np.float64)
    return bool(np.all(np.isfinite(a)) and np.all(a == np.round(a)) and np.all(np.abs(a) < 2 ** 40))


class Objective:
    """f(x) = 1/2 x^T Q x + c^T x + c0, evaluated by its definition."""

    def __init__(self, Q, c, c0=0.0):
        self.Q = np.asarray(Q, dtype=np.float64)
        self.c = np.asarray(c, dtype=np.float64)
        self.c0 = float(c0)
        self.exact = _integral(self.Q) and _integral(self.c) and _integral([self.c0])
        if self.exact:
            self.Qi = np.asarray(np.round(self.Q), dtype=object)
            self.ci = np.asarray(np.round(self.c), dtype=object)
            self.c0i = int(round(self.c0))

    def key(self, x):
        """A value ordered like f(x): 2 f(x) as an exact int when the data are integral, else f(x)."""
        x = np.asarray(x)
        if self.exact:
            xa = np.abs(x).astype(np.float64).sum()
            if (np.abs(self.Q).max(initial=0) * xa * xa + 2 * np.abs(self.c).sum() * xa
                    + 2 * abs(self.c0) < 2.0 ** 62):
                xi = x.astype(np.int64)   # exact: every partial sum is bounded by 2^62
                Qi = self.Qi.astype(np.int64)
                return int(xi @ Qi @ xi + 2 * (xi @ self.ci.astype(np.int64)) + 2 * self.c0i)
            xi = np.asarray([int(v) for v in x], dtype=object)
            return int(xi.dot(self.Qi.dot(xi)) + 2 * xi.dot(self.ci) + 2 * self.c0i)
        xf = x.astype(np.float64)
        return float(0.5 * xf @ self.Q @ xf + self.c @ xf + self.c0)

    def value(self, x) -> float:
        k = self.key(x)
        return k / 2.0 if self.exact else k


class SeparableTable:
    """f(x) = c0 + sum_j f_j(x_j) (the separable form of Prop. 3), each f_j given by its values on the
    integer box: tables[j][k] = f_j(l_j + k). Evaluated by its definition: an exact integer sum when every
    value is integral, else the correctly rounded fp64 sum (math.fsum)."""

    def __init__(self, tables, l, c0=0.0):
        self.tables = [np.asarray(t, dtype=np.float64) for t in tables]
        self.l = [int(v) for v in l]
        self.c0 = float(c0)
        self.exact = all(_integral(t) for t in self.tables) and _integral([self.c0])
        if self.exact:
            self.ti = [[int(round(v)) for v in t] for t in self.tables]
            self.c0i = int(round(self.c0))

    def key(self, x):
        idx = [int(v) - lj for v, lj in zip(x, self.l)]
        if self.exact:
            return self.c0i + sum(t[k] for t, k in zip(self.ti, idx))
        return math.fsum([self.c0] + [float(t[k]) for t, k in zip(self.tables, idx)])

    def value(self, x) -> float:
        return float(self.key(x))


def max_step_length(x, g, l, u) -> int:
    """Largest lambda >= 0 with l <= x + lambda g <= u."""
    lam = None
    for xi, gi, li, ui in zip(x, g, l, u):
        if gi > 0:
            s = (int(ui) - int(xi)) // int(gi)
        elif gi < 0:
            s = (int(xi) - int(li)) // (-int(gi))
        else:
            continue
        lam = s if lam is None else min(lam, s)
    if lam is None:
        raise ValueError("ZeroDirection")
    return max(lam, 0)


def feasible(A, b, l, u, x) -> bool:
    x = np.asarray(x, dtype=np.int64)
    return bool(np.all(np.asarray(A, np.int64) @ x == np.asarray(b, np.int64))
                and np.all(x >= l) and np.all(x <= u))


def best_step(f: Objective, x, g, l, u, step_cap: int = 1_000_000):
    """argmin over lambda in [1, lambda_max] of f(x + lambda g) among strict improvements; ties -> smaller
    lambda. Returns (lambda, key) or None."""
    fx = f.key(x)
    lmax = min(max_step_length(x, g, l, u), step_cap)
    best = None
    for lam in range(1, lmax + 1):
        k = f.key(np.asarray(x) + lam * np.asarray(g))
        if k < fx and (best is None or k < best[1]):
            best = (lam, k)
    return best


def direction_list(S):
    """D = S ∪ -S sorted lexicographically (the tie-break order)."""
    D = set(tuple(int(v) for v in g) for g in S)
    D |= {tuple(-v for v in g) for g in D}
    return sorted(D)


def graver_best_augment(f: Objective, A, b, l, u, x0, S, step_cap: int = 1_000_000, max_iter: int = 100_000):
    """Alg. 2 from one feasible x0 with test set S (canonical rows; both signs are used).
    Returns (x, iterations)."""
    if not feasible(A, b, l, u, x0):
        raise InfeasibleStart("x0 violates Ax = b or l <= x <= u")
    D = direction_list(S)
    x = np.asarray(x0, dtype=np.int64).copy()
    it = 0
    while it < max_iter:
        best = None  # (key, g index, lambda)
        for gi, g in enumerate(D):
            r = best_step(f, x, g, l, u, step_cap)
            if r is None:
                continue
            lam, k = r
            if best is None or (k, gi, lam) < best:
                best = (k, gi, lam)
        if best is None:
            break
        x = x + best[2] * np.asarray(D[best[1]], dtype=np.int64)
        it += 1
    return x, it


def multi_start(f: Objective, A, b, l, u, X0, S, step_cap: int = 1_000_000):
    """MAPLE's |S0| parallel augmentations; best by f, ties lexicographically smallest x.
    Returns (x_best, f_best, per-start finals)."""
    finals = [graver_best_augment(f, A, b, l, u, x0, S, step_cap)[0] for x0 in np.asarray(X0)]
    if not finals:
        return None, None, []
    best = min(finals, key=lambda x: (f.key(x), tuple(int(v) for v in x)))
    return best, f.value(best), finals
