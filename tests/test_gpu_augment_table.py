"""GPU parity of the augmentation with separable value tables (MAPLE_OBJ_TABLE, reading #27): f(x) = c0 +
sum_j f_j(x_j) (the separable form of Prop. 3), f_j given by its values on the box. Gate G4: same best
x as the oracle (lexicographic tie-break), objective within 1e-9 relative, per-start iteration counts equal;
Prop. 3 with convex non-quadratic f_j and the true Graver basis reaches the brute-force optimum."""
import itertools

import numpy as np
import pytest

from oracle import augment as OA
from oracle import graver as OG

pytestmark = pytest.mark.gpu


def _rows_set(ds):
    return {tuple(int(v) for v in r) for r in ds.rows().tolist()}


def _flat(tables):
    return np.concatenate([np.asarray(t, np.float64) for t in tables])


def _random_tables(rng, l, u, integer):
    """Seeded synthetic tables: non-convex in general (any real f_j is allowed)."""
    out = []
    for a, b in zip(l, u):
        w = int(b) - int(a) + 1
        out.append(rng.integers(-20, 21, size=w).astype(np.float64) if integer else rng.uniform(-10, 10, size=w))
    return out


@pytest.mark.parametrize("seed", range(8))
def test_prop3_table_convex_nonquadratic(gpu_lib, seed):
    rng = np.random.default_rng(300 + seed)
    n, m = 5, 2
    A = rng.integers(-2, 3, size=(m, n))
    while np.linalg.matrix_rank(A.astype(float)) < m:
        A = rng.integers(-2, 3, size=(m, n))
    l, u = np.zeros(n, np.int64), np.full(n, 3)
    b = A @ rng.integers(0, 4, size=n)
    a = rng.integers(0, 4, size=n) + 0.5 * rng.integers(0, 2, size=n)
    fns = [(lambda t, a=a[j]: abs(t - a) ** 3) if j % 2 else (lambda t, a=a[j]: 2.0 ** abs(t - a)) for j in range(n)]
    tables = [[fj(t) for t in range(0, 4)] for fj in fns]
    f = OA.SeparableTable(tables, l, 0.5)
    G = {OG.canonical(g) for g in OG.graver_in_box(A, -(u - l), u - l)}
    feas = [np.array(p) for p in itertools.product(range(4), repeat=n) if np.all(A @ np.array(p) == b)]
    opt = min(f.key(p) for p in feas)
    ctx = gpu_lib.Context(A, l, u)
    ds = ctx.dirset_from_host(np.array(sorted(G)), filter_minimal=False)
    X0 = np.array(feas[:: max(1, len(feas) // 8)])
    xb, fb, st, _ = ctx.augment(ds, _flat(tables), None, 0.5, b, X0, kind=gpu_lib.OBJ_TABLE)
    assert st == 0 and np.all(A @ xb == b)
    assert abs(fb - opt) <= 1e-12 * max(1.0, abs(opt)) and f.key(xb) == opt


@pytest.mark.parametrize("name,k0,integer", [("C1", 64, True), ("C2a", 24, True), ("C2b", 16, True),
                                             ("C2a", 24, False), ("C2b", 16, False)])
def test_table_multistart_matches_oracle(gpu_lib, name, k0, integer):
    from synth import config, feasible_points
    inst = config(name)
    ctx = gpu_lib.Context(inst.A, inst.l, inst.u)
    ds = ctx.extract(2048 if name != "C1" else 1024, inst.steps, inst.lr, inst.seed)
    S = _rows_set(ds)
    X0 = feasible_points(inst, k0, seed=78)
    rng = np.random.default_rng(17)
    tables = _random_tables(rng, inst.l, inst.u, integer)
    xb, fb, st, it = ctx.augment(ds, _flat(tables), None, 2.0, inst.b, X0, kind=gpu_lib.OBJ_TABLE)
    f = OA.SeparableTable(tables, inst.l, 2.0)
    xo, fo, _ = OA.multi_start(f, inst.A, inst.b, inst.l, inst.u, X0, S)
    assert xb.tolist() == xo.tolist()
    assert abs(fb - fo) <= 1e-9 * max(1.0, abs(fo))
    if integer:
        assert fb == fo
    its = [OA.graver_best_augment(f, inst.A, inst.b, inst.l, inst.u, x0, S)[1] for x0 in X0[:6]]
    assert it[:6].tolist() == its


def test_table_equals_separable_quadratic(gpu_lib):
    """The table of 1/2 q_j t^2 + c_j t is the SEPARABLE quadratic: identical x, f and iteration counts."""
    from synth import config, feasible_points
    inst = config("C2b")
    ctx = gpu_lib.Context(inst.A, inst.l, inst.u)
    ds = ctx.extract(2048, inst.steps, inst.lr, inst.seed)
    rng = np.random.default_rng(5)
    q = rng.integers(-4, 5, size=inst.A.shape[1]).astype(float)
    c = rng.integers(-9, 10, size=inst.A.shape[1]).astype(float)
    tables = [[0.5 * q[j] * t * t + c[j] * t for t in range(int(inst.l[j]), int(inst.u[j]) + 1)] for j in range(inst.A.shape[1])]
    X0 = feasible_points(inst, 32, seed=3)
    x1, f1, _, it1 = ctx.augment(ds, q, c, 1.0, inst.b, X0, kind=gpu_lib.OBJ_SEPARABLE)
    x2, f2, _, it2 = ctx.augment(ds, _flat(tables), None, 1.0, inst.b, X0, kind=gpu_lib.OBJ_TABLE)
    assert x1.tolist() == x2.tolist() and f1 == f2 and it1.tolist() == it2.tolist()


def test_table_many_matches_single_and_rejects_mixed(gpu_lib):
    from synth import c4_batch
    base, insts = c4_batch(n_inst=5, incumbents=8)
    ctx = gpu_lib.Context(base.A, base.l, base.u)
    ds = ctx.extract(2048, 200, 0.01, 2)
    rng = np.random.default_rng(9)
    tabs = [_flat(_random_tables(rng, base.l, base.u, integer=True)) for _ in insts]
    bs = [b for _, _, b, _ in insts]
    X0s = np.stack([x0 for _, _, _, x0 in insts])
    xb, fb = ctx.augment_many(ds, tabs, None, [0.0] * 5, bs, X0s, kind=gpu_lib.OBJ_TABLE)
    for t in range(5):
        x1, f1, _, _ = ctx.augment(ds, tabs[t], None, 0.0, bs[t], X0s[t], kind=gpu_lib.OBJ_TABLE)
        assert xb[t].tolist() == x1.tolist() and fb[t] == f1
    # mixed kinds in one batch are rejected (include/maple.h, MAPLE_OBJ_TABLE)
    with pytest.raises(gpu_lib.MapleError) as e:
        ctx.augment_many(ds, [tabs[0], insts[1][0]], [None, insts[1][1]], [0.0, 0.0], bs[:2], X0s[:2],
                         kind=[gpu_lib.OBJ_TABLE, gpu_lib.OBJ_QUADRATIC])
    assert e.value.name == "BAD_ARG"


def test_table_large_set_local_optimality(gpu_lib):
    """C3 (n = 300) with |D| > 16,384 (the 1,024-thread, unstaged path): every result is feasible, f_best is
    the table sum at x_best, and x_best is a local optimum of Alg. 2 over D (no feasible improving step)."""
    from synth import c3, feasible_points
    inst = c3()
    ctx = gpu_lib.Context(inst.A, inst.l, inst.u)
    ds = ctx.extract(16384, inst.steps, inst.lr, inst.seed)
    S = ds.rows().astype(np.int64)
    assert 2 * len(S) > 16384
    D = np.concatenate([S, -S])
    rng = np.random.default_rng(11)
    tables = _random_tables(rng, inst.l, inst.u, integer=True)
    X0 = feasible_points(inst, 4, seed=21)
    xb, fb, _, _ = ctx.augment(ds, _flat(tables), None, 0.0, inst.b, X0, kind=gpu_lib.OBJ_TABLE)
    f = OA.SeparableTable(tables, inst.l, 0.0)
    x = xb.astype(np.int64)
    assert np.all(inst.A @ x == inst.b) and np.all(x >= inst.l) and np.all(x <= inst.u)
    assert fb == f.key(x)
    assert fb <= min(f.key(x0) for x0 in X0)
    T = np.full((inst.A.shape[1], int(np.max(inst.u - inst.l)) + 1), np.nan)
    for j, t in enumerate(tables):
        T[j, :len(t)] = t
    base = T[np.arange(inst.A.shape[1]), x - inst.l].sum()
    for lam in (1, 2):
        y = x[None, :] + lam * D
        ok = np.all((y >= inst.l) & (y <= inst.u), axis=1)
        vals = T[np.arange(inst.A.shape[1])[None, :], np.clip(y[ok] - inst.l, 0, T.shape[1] - 1)].sum(axis=1)
        assert np.all(vals >= base)
