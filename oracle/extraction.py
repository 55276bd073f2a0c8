"""Parallel extraction, Algorithm 3, step by step in the paper's order (oracle).

For t in [T]: one Adam step on Eq. 3; then if B⌈z⌋ ∈ [l-u, u-l]: 𝒢 ← 𝒢 ∪ {B⌈z⌋}.
Every start is independent ("performs in parallel"); numpy arrays carry all starts side by side,
but each row's arithmetic is the per-start algorithm (no cross-start coupling).

Readings:
  #1/#2 starts: g ~ U(l-u, u-l) continuous per coordinate, drawn from a splitmix64 counter keyed by
        (seed, global start i, coordinate j): x = mix(seed ^ mix(i*n + j + 1)), U = (x >> 11) * 2^-53,
        g = (l_j - u_j) + U * (2 (u_j - l_j)); z0 = B^+ g in fp64.
  #7/#8 subgradient of Eq. 3: B^T sign(Bz) (sign(0) = 0) + lam1 (ceil z + floor z - 2 z) (0 at integers)
        + e_k * (-lam2 sign(z_k) / max(z_k^2, 1e-8)) when ||z||_inf < 1, k = lowest-index argmax |z_i|.
  #9    Adam with the torch.optim.Adam formula (PyTorch 2.1.0): beta = (0.9, 0.999), eps = 1e-8,
        m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2; z <- z - (lr / (1 - b1^t)) m / (sqrt(v)/sqrt(1-b2^t) + eps).
  #10   loss summed per start (no 1/N), so each start is independent of N.
  #6    ⌈·⌋ rounds half away from zero.
  #11/#12 harvest after each update t = 1..T; g = 0 is excluded.
  #13   set semantics with one canonical representative per ± pair (first nonzero > 0).
  #24   optimizer variants ("first-order methods such as Adam"): plain GD
        z <- z - lr g and sign-GD z <- z - lr sign(g) (sign(0) = 0), lr rounded once to the working dtype.
  #25   harvest-final-only variant: Alg. 3 line 9 applied to the final iterate z_T only.
"""
from __future__ import annotations

import numpy as np

from .graver import canonical  # noqa: F401  (re-exported for tests)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniforms(seed: int, starts: np.ndarray, n: int) -> np.ndarray:
    """U[i, j] in [0, 1) for the given global start indices (reading #2)."""
    starts = np.asarray(starts, dtype=np.uint64)
    key = starts[:, None] * np.uint64(n) + np.arange(n, dtype=np.uint64)[None, :] + np.uint64(1)
    x = splitmix64(np.uint64(seed) ^ splitmix64(key))
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def sample_starts(l, u, Bplus, seed: int, starts) -> tuple[np.ndarray, np.ndarray]:
    """Alg. 3 lines 4-5: g0 ~ Uniform(l-u, u-l), z0 = B^{-1} g0. Returns (g0, z0) in fp64."""
    l = np.asarray(l, dtype=np.int64)
    u = np.asarray(u, dtype=np.int64)
    U = uniforms(seed, np.asarray(starts), l.shape[0])
    a = (l - u).astype(np.float64)
    w = (2 * (u - l)).astype(np.float64)
    g0 = a[None, :] + U * w[None, :]
    z0 = g0 @ np.asarray(Bplus, dtype=np.float64).T
    return g0, z0


def loss(z, B, lam1: float = 0.85, lam2: float = 1.0, eps_div: float = 1e-8) -> float:
    """Eq. 3: ||Bz||_1 + lam1 sum (z - floor z)(ceil z - z) + lam2 max{1/||z||_inf - 1, 0},
    with 1/max(||z||_inf, eps_div) at z = 0 (reading #7)."""
    z = np.asarray(z, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    t1 = np.abs(B @ z).sum()
    t2 = np.sum((z - np.floor(z)) * (np.ceil(z) - z))
    zinf = np.abs(z).max() if z.size else 0.0
    t3 = max(1.0 / max(zinf, eps_div) - 1.0, 0.0)
    return float(t1 + lam1 * t2 + lam2 * t3)


def subgrad(Z, B, lam1, lam2, eps_div=1e-8):
    """Row-wise subgradient of Eq. 3 (readings #7, #8). Z: (N, d) in its working dtype."""
    dt = Z.dtype
    Bt = B.astype(dt)
    Y = Z @ Bt.T                                  # (N, n): B z per start
    S = np.sign(Y)                                # sign(0) = 0
    G = S @ Bt                                    # (N, d): B^T sign(B z)
    G = G + dt.type(lam1) * (np.ceil(Z) + np.floor(Z) - dt.type(2) * Z)
    if Z.shape[1] > 0:
        A = np.abs(Z)
        k = np.argmax(A, axis=1)                  # first index of the maximum = lowest-index tie-break
        rows = np.arange(Z.shape[0])
        zk = Z[rows, k]
        act = A[rows, k] < dt.type(1)
        extra = -dt.type(lam2) * np.sign(zk) / np.maximum(zk * zk, dt.type(eps_div))
        G[rows[act], k[act]] += extra[act]
    return G


def round_half_away(Z) -> np.ndarray:
    """⌈z⌋ = nearest integer, halves away from zero (reading #6); exact: z - trunc(z) is exact."""
    t = np.trunc(Z)
    f = Z - t
    return (t + np.where(np.abs(f) >= 0.5, np.sign(Z), 0)).astype(np.int64)


def canonicalize_rows(G: np.ndarray) -> np.ndarray:
    """Multiply each row by the sign of its first nonzero entry (rows of zeros stay zero)."""
    nz = G != 0
    first = np.argmax(nz, axis=1)
    s = np.sign(G[np.arange(G.shape[0]), first])
    s[s == 0] = 1
    return G * s[:, None]


def harvest(Z, B, l, u):
    """Alg. 3 lines 9-10 for every row: g = B ⌈z⌋, kept iff g in [l-u, u-l] and g != 0; canonical rows."""
    R = round_half_away(Z)
    Bi = np.asarray(B, dtype=np.int64)
    # B r exactly: a float64 product of integers is exact while every partial sum stays below 2^53
    if R.size and np.abs(R).max() * np.abs(Bi).sum(axis=1).max() < 2.0 ** 53:
        G = (R.astype(np.float64) @ Bi.T.astype(np.float64)).astype(np.int64)
    else:
        G = R @ Bi.T
    box = (u - l).astype(np.int64)
    keep = np.all(np.abs(G) <= box[None, :], axis=1) & np.any(G != 0, axis=1)
    return canonicalize_rows(G[keep])


OPTIMIZERS = ("adam", "gd", "signgd")


def descend(z0, B, steps, lr, lam1=0.85, lam2=1.0, beta1=0.9, beta2=0.999, eps=1e-8, dtype=np.float64,
            l=None, u=None, pool=None, trace=None, optimizer="adam", harvest_final=False):
    """Alg. 3 lines 6-11 for a batch of starts. Returns the final iterates Z (dtype). If l, u and `pool`
    (a set) are given, every step's harvest (only the last one with harvest_final, reading #25) is added to
    the pool as canonical int tuples. `optimizer` selects line 8's update (reading #24): "adam" (default),
    "gd" (z - lr g) or "signgd" (z - lr sign(g)).

    Scalars follow torch.optim.Adam (reading #9; PyTorch 2.1.0): beta, 1 - beta, the step size
    lr / (1 - beta1^t) and sqrt(1 - beta2^t) are computed in Python double and then used in `dtype`
    arithmetic (so the fp32 mode is PyTorch's fp32 Adam; in fp64 mode this is exact)."""
    dt = np.dtype(dtype)
    Z = np.asarray(z0).astype(dt)
    Bd = np.asarray(B, dtype=np.float64)
    m = np.zeros_like(Z)
    v = np.zeros_like(Z)
    b1, b2 = dt.type(beta1), dt.type(beta2)
    omb1, omb2 = dt.type(1.0 - beta1), dt.type(1.0 - beta2)
    if optimizer not in OPTIMIZERS:
        raise ValueError(f"optimizer must be one of {OPTIMIZERS}")
    lr_d = dt.type(lr)
    for t in range(1, steps + 1):
        G = subgrad(Z, Bd, lam1, lam2)
        if optimizer == "adam":
            m = b1 * m + omb1 * G
            v = b2 * v + omb2 * G * G
            step = dt.type(lr / (1.0 - beta1 ** t))
            bc2s = dt.type(np.sqrt(1.0 - beta2 ** t))
            denom = np.sqrt(v) / bc2s + dt.type(eps)
            Z = Z - step * m / denom
        elif optimizer == "gd":
            Z = Z - lr_d * G
        else:
            Z = Z - lr_d * np.sign(G).astype(dt)
        if trace is not None:
            trace.append(Z.copy())
        if pool is not None and (not harvest_final or t == steps):
            H = harvest(Z, B, np.asarray(l, np.int64), np.asarray(u, np.int64))
            if H.shape[0]:
                for row in np.unique(H, axis=0):
                    pool.add(tuple(int(x) for x in row))
    return Z


def extract_pool(B, Bplus, l, u, n_starts, steps, lr, seed, starts=None, dtype=np.float64,
                 lam1=0.85, lam2=1.0, chunk=8192, optimizer="adam", harvest_final=False):
    """Alg. 3 over global start indices `starts` (default range(n_starts)): the harvested direction
    set 𝒢 (canonical tuples, before the exact check / ⊑ filter) and the final iterates."""
    if starts is None:
        starts = np.arange(n_starts)
    starts = np.asarray(starts)
    pool: set = set()
    finals = []
    for s0 in range(0, len(starts), chunk):
        idx = starts[s0:s0 + chunk]
        _, z0 = sample_starts(l, u, Bplus, seed, idx)
        if np.dtype(dtype) == np.float32:
            z0 = z0.astype(np.float32)
        finals.append(descend(z0, B, steps, lr, lam1=lam1, lam2=lam2, dtype=dtype, l=l, u=u, pool=pool,
                              optimizer=optimizer, harvest_final=harvest_final))
    Z = np.concatenate(finals) if finals else np.zeros((0, np.asarray(B).shape[1]))
    return pool, Z
