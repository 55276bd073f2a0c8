"""Synthetic INLP instances of model (1) (Eq. 1): min f(x) s.t. Ax=b, l<=x<=u, x in Z^n.

Recipes follow SURVEY.md §8(d)-1 (configs C1-C5 of BASELINE.json). Everything is integer and seeded:
b is always A @ x_plant for a planted feasible x_plant, so every instance is feasible by construction;
f(x) = 1/2 x^T Q x + c^T x + c0 with integer Q, c (SPEC S:401 objective convention).

Feasible incumbents are drawn by random walks from x_plant along moves that are kernel elements *by
construction of the instance* (e.g. e_i - e_j inside an all-ones group); no lattice arithmetic is done here.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Instance:
    name: str
    A: np.ndarray          # int64 (m, n)
    b: np.ndarray          # int64 (m,)
    l: np.ndarray          # int64 (n,)
    u: np.ndarray          # int64 (n,)
    Q: np.ndarray          # float64 (n, n), symmetric, integer-valued
    c: np.ndarray          # float64 (n,), integer-valued
    c0: float
    x_plant: np.ndarray    # int64 (n,), feasible
    moves: list = field(default_factory=list)   # construction-known kernel moves for incumbent sampling
    n_starts: int = 1024
    steps: int = 200
    lr: float = 0.01
    seed: int = 1

    @property
    def m(self) -> int:
        return int(self.A.shape[0])

    @property
    def n(self) -> int:
        return int(self.A.shape[1])

    @property
    def d(self) -> int:
        return self.n - self.m


def _sym_int(rng: np.random.Generator, n: int, lo: int, hi: int) -> np.ndarray:
    U = rng.integers(lo, hi + 1, size=(n, n))
    Q = np.triu(U) + np.triu(U, 1).T
    return Q.astype(np.float64)


def _finish(name, A, l, u, x, Q, c, moves, **kw) -> Instance:
    A = np.asarray(A, dtype=np.int64)
    x = np.asarray(x, dtype=np.int64)
    return Instance(name=name, A=A, b=A @ x, l=np.asarray(l, np.int64), u=np.asarray(u, np.int64),
                    Q=np.asarray(Q, np.float64), c=np.asarray(c, np.float64), c0=0.0, x_plant=x,
                    moves=moves, **kw)


def _group_moves(groups):
    mv = []
    for g in groups:
        for i in g:
            for j in g:
                if i < j:
                    mv.append((i, j))
    return mv


def all_ones(n: int, lo: int = 0, hi: int = 3) -> Instance:
    """1 x n all-ones row; its Graver basis is {e_i - e_j} (closed form)."""
    A = np.ones((1, n), np.int64)
    x = np.zeros(n, np.int64)
    x[0] = hi
    return _finish(f"all_ones{n}", A, np.full(n, lo), np.full(n, hi), x, np.eye(n) * 2, np.zeros(n),
                   _group_moves([list(range(n))]))


def c1() -> Instance:
    """BASELINE.json configs[0]: A = all-ones row, n=4, l=0, u=3, separable quadratic f (seed 101)."""
    rng = np.random.default_rng(101)
    n = 4
    q = rng.integers(1, 5, size=n)
    c = rng.integers(-8, 9, size=n)
    return _finish("C1", np.ones((1, n)), np.zeros(n), np.full(n, 3), [3, 0, 2, 1], np.diag(q), c,
                   _group_moves([list(range(n))]), n_starts=1024, steps=200, lr=0.01, seed=1)


def semi_assignment(k: int, s: int, gen_seed: int = 202, b_r=None, name=None, **kw) -> Instance:
    """k disjoint all-ones rows of width s over a binary box (Graver = e_i - e_j within groups)."""
    rng = np.random.default_rng(gen_seed)
    n = k * s
    A = np.zeros((k, n), np.int64)
    groups = [list(range(r * s, (r + 1) * s)) for r in range(k)]
    x = np.zeros(n, np.int64)
    for r, g in enumerate(groups):
        A[r, g] = 1
        ones = 1 if b_r is None else int(b_r[r])
        x[rng.choice(g, size=ones, replace=False)] = 1
    Q = _sym_int(rng, n, -10, 10)
    c = rng.integers(-10, 11, size=n)
    return _finish(name or f"semi{k}x{s}", A, np.zeros(n), np.ones(n), x, Q, c, _group_moves(groups), **kw)


def c2a() -> Instance:
    """configs[1] (pinned variant): 5 all-ones rows over 5 disjoint groups of 10, binary, b_r = 1.
    Graver basis = 5 * C(10,2) = 225 canonical elements (closed form)."""
    return semi_assignment(5, 10, gen_seed=202, name="C2a", n_starts=65536, steps=200, lr=0.01, seed=2)


def c2b() -> Instance:
    """configs[1] knapsack/assignment variant: 4 group rows over x_0..x_39 + 1 knapsack row over all 50
    (w in U{1..5}), u_j in U{1,2,3}, l = 0, b = A x_plant. Unpinned."""
    rng = np.random.default_rng(203)
    n, k, s = 50, 4, 10
    A = np.zeros((k + 1, n), np.int64)
    for r in range(k):
        A[r, r * s:(r + 1) * s] = 1
    w = rng.integers(1, 6, size=n)
    A[k] = w
    u = rng.integers(1, 4, size=n)
    x = np.array([rng.integers(0, ui + 1) for ui in u], np.int64)
    Q = _sym_int(rng, n, -10, 10)
    c = rng.integers(-10, 11, size=n)
    # construction-known moves: e_i - e_j with equal group membership and equal knapsack weight
    grp = [i // s if i < k * s else -1 for i in range(n)]
    mv = [(i, j) for i in range(n) for j in range(i + 1, n) if grp[i] == grp[j] and w[i] == w[j]]
    return _finish("C2b", A, np.zeros(n), u, x, Q, c, mv, n_starts=65536, steps=200, lr=0.01, seed=2)


def _identity_block(name, m, n, vals, p, gen_seed, **kw) -> Instance:
    """A = [I_m | W] Pi (columns permuted), W_ij in vals with probability p, binary box, b = A x_plant."""
    rng = np.random.default_rng(gen_seed)
    d = n - m
    mask = rng.random((m, d)) < p
    W = np.where(mask, rng.choice(np.asarray(vals), size=(m, d)), 0)
    A0 = np.concatenate([np.eye(m, dtype=np.int64), W.astype(np.int64)], axis=1)
    perm = rng.permutation(n)
    A = A0[:, perm]
    # planted x: free part random binary, identity part chosen so that A x = b with b = A x (any x works)
    x0 = np.concatenate([rng.integers(0, 2, size=m), rng.integers(0, 2, size=d)])
    x = x0[perm]
    Q = _sym_int(rng, n, -10, 10)
    c = rng.integers(-10, 11, size=n)
    # kernel moves by construction: column j of [-W; I] in the unpermuted order, mapped through Pi
    inv = np.argsort(perm)
    moves = []
    for j in range(d):
        v = np.zeros(n, np.int64)
        v[:m] = -W[:, j]
        v[m + j] = 1
        moves.append(v[perm])
    del inv
    return _finish(name, A, np.zeros(n), np.ones(n), x, Q, c, moves, **kw)


def c3() -> Instance:
    """configs[2]: n=300, m=20, [I_20 | W] Pi with W in {+-1} at p=0.1 (about two constraints per free
    variable), binary box, dense Q. (SURVEY §8(d)-1 proposed W in {+-1,+-2} at p=0.3; with that recipe no
    binary-box kernel element is ever reached — 0 harvested by both the oracle and the GPU at T=200 — so the
    config would measure nothing.)"""
    return _identity_block("C3", 20, 300, [-1, 1], 0.1, 3, n_starts=1 << 20, steps=200, lr=0.01, seed=3)


def c5() -> Instance:
    """configs[4]: n=1000, m=100, sparse [I_100 | W] Pi with W in {+-1} at p=0.02, binary."""
    return _identity_block("C5", 100, 1000, [-1, 1], 0.02, 5, n_starts=1 << 22, steps=200, lr=0.01, seed=5)


def c4_batch(n_inst: int = 1000, incumbents: int = 256):
    """configs[3]: the C2a matrix A shared by n_inst (f, b) instances (seed 1000+k); group sums b_r in
    U{1..9}; `incumbents` uniform feasible points each (seed 5000+k). Returns (base, [(Q, c, b, x0)])."""
    base = c2a()
    out = []
    for k in range(n_inst):
        rng = np.random.default_rng(1000 + k)
        b_r = rng.integers(1, 10, size=5)
        inst = semi_assignment(5, 10, gen_seed=1000 + k, b_r=b_r, name=f"C4_{k}")
        x0 = feasible_points(inst, incumbents, seed=5000 + k)
        out.append((inst.Q, inst.c, inst.b, x0))
    return base, out


def assignment(k: int) -> Instance:
    """k x k assignment (row sums and column sums = 1) with one redundant row dropped (m = 2k-1)."""
    n = k * k
    rows = []
    for i in range(k):
        r = np.zeros(n, np.int64)
        r[i * k:(i + 1) * k] = 1
        rows.append(r)
    for j in range(k):
        r = np.zeros(n, np.int64)
        r[j::k] = 1
        rows.append(r)
    A = np.array(rows[:-1])
    x = np.eye(k, dtype=np.int64).reshape(-1)
    return _finish(f"assign{k}", A, np.zeros(n), np.ones(n), x, np.eye(n), np.zeros(n), [])


def partition_row(k: int, box: int) -> Instance:
    """A = [[1, 2, ..., k]] on [-box, box]^k style bounds (l = 0, u = box): primitive partition identities."""
    A = np.arange(1, k + 1, dtype=np.int64)[None, :]
    return _finish(f"partition{k}", A, np.zeros(k), np.full(k, box), np.zeros(k), np.eye(k), np.zeros(k), [])


def random_small(m: int, n: int, seed: int, lo: int = -3, hi: int = 3, ubox: int = 2) -> Instance:
    """Random full-row-rank integer A (entries in [lo, hi]) for property tests; box [0, ubox]^n."""
    rng = np.random.default_rng(seed)
    while True:
        A = rng.integers(lo, hi + 1, size=(m, n))
        if np.linalg.matrix_rank(A.astype(np.float64)) == m:
            break
    x = rng.integers(0, ubox + 1, size=n)
    Q = np.diag(rng.integers(1, 5, size=n)).astype(np.float64)
    c = rng.integers(-6, 7, size=n)
    return _finish(f"rand{m}x{n}s{seed}", A, np.zeros(n), np.full(n, ubox), x, Q, c, [])


def feasible_points(inst: Instance, k: int, seed: int, walk: int = 64) -> np.ndarray:
    """k feasible incumbents (int64 (k, n)) by random walks of `walk` accepted-or-rejected moves from
    x_plant. Moves are construction-known kernel elements, so A x = b is preserved exactly."""
    rng = np.random.default_rng(seed)
    n = inst.n
    vecs = []
    for mv in inst.moves:
        if isinstance(mv, tuple):
            v = np.zeros(n, np.int64)
            v[mv[0]] = 1
            v[mv[1]] = -1
            vecs.append(v)
        else:
            vecs.append(np.asarray(mv, np.int64))
    X = np.empty((k, n), np.int64)
    for t in range(k):
        x = inst.x_plant.copy()
        if vecs:
            for _ in range(walk):
                v = vecs[rng.integers(len(vecs))] * (1 if rng.random() < 0.5 else -1)
                y = x + v
                if np.all(y >= inst.l) and np.all(y <= inst.u):
                    x = y
        X[t] = x
    return X


_CONFIGS = {"C1": c1, "C2a": c2a, "C2b": c2b, "C3": c3, "C5": c5}


def config(name: str) -> Instance:
    return _CONFIGS[name]()
