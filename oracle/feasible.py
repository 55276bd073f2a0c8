"""Initial feasible solutions, Eq. 4 (§4.3) — oracle.

    min_{x in [l,u]^n}  ||A x - b||_2^2 + lambda3 * sum_i (x_i - floor x_i)(ceil x_i - x_i),   lambda3 = 0.1

"can be efficiently optimized from diversified initial points using Adam"; every optimal solution
is a feasible point of model (1). Readings:
  F1 starts: x0 ~ U(l, u) continuous per coordinate from the splitmix64 counter of extraction.py keyed by
     (seed ^ FEAS_SALT, start i, coordinate j): x0_j = l_j + U (u_j - l_j).
  F2 gradient: 2 A^T (A x - b) + lambda3 (ceil x + floor x - 2x) (0 at integers).
  F3 Adam (torch.optim.Adam formula, scalars in double) followed by the projection x <- clip(x, l, u)
     after every step (the box of Eq. 4).
  F4 after T steps: x_int = round half away from zero; kept iff A x_int = b exactly and l <= x_int <= u;
     duplicates collapse; the result is sorted lexicographically.
"""
from __future__ import annotations

import numpy as np

from .extraction import round_half_away, splitmix64

FEAS_SALT = 0x5EED_F00D_CAFE_0001


def starts(l, u, seed: int, idx) -> np.ndarray:
    """x0 ~ U(l, u) (reading F1), fp64, shape (len(idx), n)."""
    l = np.asarray(l, dtype=np.int64)
    u = np.asarray(u, dtype=np.int64)
    n = l.shape[0]
    idx = np.asarray(idx, dtype=np.uint64)
    key = idx[:, None] * np.uint64(n) + np.arange(n, dtype=np.uint64)[None, :] + np.uint64(1)
    x = splitmix64(np.uint64((seed ^ FEAS_SALT) & 0xFFFFFFFFFFFFFFFF) ^ splitmix64(key))
    U = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return l.astype(np.float64)[None, :] + U * (u - l).astype(np.float64)[None, :]


def loss(x, A, b, lam3: float = 0.1) -> float:
    """Eq. 4 objective at x."""
    x = np.asarray(x, dtype=np.float64)
    r = np.asarray(A, np.float64) @ x - np.asarray(b, np.float64)
    return float(r @ r + lam3 * np.sum((x - np.floor(x)) * (np.ceil(x) - x)))


def grad(X, A, b, lam3: float = 0.1):
    """Row-wise gradient (reading F2) for a batch X (N, n), in X's dtype."""
    dt = X.dtype
    A = np.asarray(A, np.float64).astype(dt)
    R = X @ A.T - np.asarray(b, np.float64).astype(dt)[None, :]
    return dt.type(2.0) * (R @ A) + dt.type(lam3) * (np.ceil(X) + np.floor(X) - dt.type(2.0) * X)


def descend(X0, A, b, l, u, steps, lr, lam3=0.1, beta1=0.9, beta2=0.999, eps=1e-8, dtype=np.float64):
    """Projected Adam on Eq. 4 (readings F2, F3). Scalars as in extraction.descend (reading #9: computed in
    Python double, used in `dtype`), so dtype=float32 is PyTorch's fp32 Adam followed by the projection."""
    dt = np.dtype(dtype)
    X = np.asarray(X0, dtype=np.float64).astype(dt)
    lo = np.asarray(l, np.float64).astype(dt)[None, :]
    hi = np.asarray(u, np.float64).astype(dt)[None, :]
    m = np.zeros_like(X)
    v = np.zeros_like(X)
    b1, b2 = dt.type(beta1), dt.type(beta2)
    omb1, omb2 = dt.type(1.0 - beta1), dt.type(1.0 - beta2)
    for t in range(1, steps + 1):
        G = grad(X, A, b, lam3)
        m = b1 * m + omb1 * G
        v = b2 * v + omb2 * G * G
        step = dt.type(lr / (1.0 - beta1 ** t))
        denom = np.sqrt(v) / dt.type(np.sqrt(1.0 - beta2 ** t)) + dt.type(eps)
        X = np.minimum(np.maximum(X - step * m / denom, lo), hi)
    return X


def feasible_set(A, b, l, u, k: int, steps: int, lr: float, seed: int, lam3: float = 0.1, dtype=np.float64):
    """Eq. 4 from k diversified starts (reading F4): sorted unique feasible integer points, and the final
    continuous iterates."""
    A = np.asarray(A, np.int64)
    X = descend(starts(l, u, seed, np.arange(k)), A, b, l, u, steps, lr, lam3, dtype=dtype)
    R = round_half_away(X.astype(np.float64))
    ok = np.all(R @ A.T == np.asarray(b, np.int64)[None, :], axis=1)
    ok &= np.all(R >= np.asarray(l)[None, :], axis=1) & np.all(R <= np.asarray(u)[None, :], axis=1)
    pts = sorted({tuple(int(v) for v in r) for r in R[ok]})
    return pts, X
