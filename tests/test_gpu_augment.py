"""GPU parity of the multi-start augmentation (Alg. 2; §4.3) — gate G4: same best x
(lexicographic tie-break) and objective within 1e-9 relative of the oracle, given the same set and x0."""
import numpy as np
import pytest

from oracle import augment as OA
from oracle import graver as OG

pytestmark = pytest.mark.gpu


def _rows_set(ds):
    return {tuple(int(v) for v in r) for r in ds.rows().tolist()}


def test_spec_worked_instance(gpu_lib):
    A = np.array([[1, 1]])
    ctx = gpu_lib.Context(A, [0, 0], [3, 3])
    ds = ctx.dirset_from_host([[1, -1]])
    xb, fb, st, it = ctx.augment(ds, 2 * np.eye(2), [-4.0, -4.0], 8.0, [4], [[3, 1]])
    assert xb.tolist() == [2, 2] and fb == 0.0 and st == 0 and it.tolist() == [1]
    xb, fb, st, it = ctx.augment(ds, 2 * np.eye(2), [-4.0, -4.0], 8.0, [4], [[2, 2]])
    assert xb.tolist() == [2, 2] and it.tolist() == [0]
    empty = ctx.dirset_from_host(np.zeros((0, 2), np.int32))
    xb, fb, st, it = ctx.augment(empty, 2 * np.eye(2), [-4.0, -4.0], 8.0, [4], [[3, 1]])
    assert xb.tolist() == [3, 1] and it.tolist() == [0]
    with pytest.raises(gpu_lib.MapleError) as e:
        ctx.augment(ds, 2 * np.eye(2), [-4.0, -4.0], 8.0, [4], [[3, 3]])
    assert e.value.name == "INFEASIBLE"
    xb, fb, st, it = ctx.augment(ds, 2 * np.eye(2), [-4.0, -4.0], 8.0, [4], np.zeros((0, 2)))
    assert st == gpu_lib.STATUS_NO_FEASIBLE


@pytest.mark.parametrize("seed", range(10))
def test_prop3_with_true_graver_basis(gpu_lib, seed):
    """Prop. 3: with G(A) and separable convex f the GPU augmentation reaches the brute-force optimum."""
    rng = np.random.default_rng(seed)
    n, m = 5, 2
    A = rng.integers(-2, 3, size=(m, n))
    while np.linalg.matrix_rank(A.astype(float)) < m:
        A = rng.integers(-2, 3, size=(m, n))
    l, u = np.zeros(n, np.int64), np.full(n, 3)
    xp = rng.integers(0, 4, size=n)
    b = A @ xp
    q = rng.integers(1, 4, size=n).astype(float)
    c = rng.integers(-8, 9, size=n).astype(float)
    G = {OG.canonical(g) for g in OG.graver_in_box(A, -(u - l), u - l)}
    import itertools
    feas = [np.array(p) for p in itertools.product(range(4), repeat=n) if np.all(A @ np.array(p) == b)]
    f = OA.Objective(np.diag(q), c)
    opt = min(f.key(p) for p in feas)
    ctx = gpu_lib.Context(A, l, u)
    ds = ctx.dirset_from_host(np.array(sorted(G)), filter_minimal=False)
    X0 = np.array(feas[:: max(1, len(feas) // 8)])
    for kind, Q in ((gpu_lib.OBJ_QUADRATIC, np.diag(q)), (gpu_lib.OBJ_SEPARABLE, q)):
        xb, fb, st, _ = ctx.augment(ds, Q, c, 0.0, b, X0, kind=kind)
        assert 2 * fb == opt


@pytest.mark.parametrize("name,k0", [("C1", 64), ("C2a", 24), ("C2b", 16)])
def test_multistart_matches_oracle(gpu_lib, name, k0):
    from synth import config, feasible_points
    inst = config(name)
    ctx = gpu_lib.Context(inst.A, inst.l, inst.u)
    ds = ctx.extract(2048 if name != "C1" else 1024, inst.steps, inst.lr, inst.seed)
    S = _rows_set(ds)
    X0 = feasible_points(inst, k0, seed=77)
    xb, fb, st, it = ctx.augment(ds, inst.Q, inst.c, inst.c0, inst.b, X0)
    f = OA.Objective(inst.Q, inst.c, inst.c0)
    xo, fo, finals = OA.multi_start(f, inst.A, inst.b, inst.l, inst.u, X0, S)
    assert xb.tolist() == xo.tolist()
    assert abs(fb - fo) <= 1e-9 * max(1.0, abs(fo))
    its = [OA.graver_best_augment(f, inst.A, inst.b, inst.l, inst.u, x0, S)[1] for x0 in X0[:6]]
    assert it[:6].tolist() == its
    assert np.all(inst.A @ xb == inst.b)


def test_augment_many_matches_single(gpu_lib):
    from synth import c4_batch
    base, insts = c4_batch(n_inst=6, incumbents=8)
    ctx = gpu_lib.Context(base.A, base.l, base.u)
    ds = ctx.extract(2048, 200, 0.01, 2)
    Qs, cs, bs, X0s = zip(*[(Q, c, b, x0) for Q, c, b, x0 in insts])
    xb, fb = ctx.augment_many(ds, Qs, cs, [0.0] * 6, bs, np.stack(X0s))
    S = _rows_set(ds)
    for t in range(6):
        x1, f1, _, _ = ctx.augment(ds, Qs[t], cs[t], 0.0, bs[t], X0s[t])
        assert xb[t].tolist() == x1.tolist() and fb[t] == f1
        f = OA.Objective(Qs[t], cs[t])
        xo, fo, _ = OA.multi_start(f, base.A, bs[t], base.l, base.u, X0s[t], S)
        assert xb[t].tolist() == xo.tolist() and abs(fb[t] - fo) <= 1e-9 * max(1, abs(fo))


def test_c4_full_batch_properties(gpu_lib):
    """configs[3] at full size: 1,000 (f, b) instances x 256 incumbents against one C2a extraction (65,536
    starts). Properties that hold at any size, checked exactly on the host for every instance: x_best is
    feasible, f_best = f(x_best), no incumbent is better, and x_best is a local optimum of Alg. 2 (no g in
    S ∪ -S with a feasible step λ >= 1 improves f). Sampled instances equal the single-instance call."""
    from synth import c4_batch
    base, insts = c4_batch()
    ctx = gpu_lib.Context(base.A, base.l, base.u)
    ds = ctx.extract(base.n_starts, base.steps, base.lr, base.seed)
    S = ds.rows().astype(np.int64)
    D = np.concatenate([S, -S])
    Qs, cs, bs, X0s = zip(*insts)
    xb, fb = ctx.augment_many(ds, Qs, cs, [0.0] * len(insts), bs, np.stack(X0s))
    l, u = base.l.astype(np.int64), base.u.astype(np.int64)
    for t, (Q, c, b, X0) in enumerate(insts):
        Qi, ci = np.asarray(Q, np.int64), np.asarray(c, np.int64)
        x = xb[t].astype(np.int64)
        assert np.all(base.A @ x == b) and np.all(x >= l) and np.all(x <= u)
        two_f = int(x @ Qi @ x + 2 * ci @ x)
        assert fb[t] == two_f / 2
        X = np.asarray(X0, np.int64)
        assert two_f <= int(np.min(np.einsum("ki,ij,kj->k", X, Qi, X) + 2 * X @ ci))
        # local optimality: 2Δ(λ) = 2λ gᵀ(Qx + c) + λ² gᵀQg >= 0 for every g in D and feasible λ >= 1
        with np.errstate(divide="ignore"):
            up = np.where(D > 0, (u - x)[None, :] // np.where(D > 0, D, 1), np.iinfo(np.int64).max)
            dn = np.where(D < 0, (x - l)[None, :] // np.where(D < 0, -D, 1), np.iinfo(np.int64).max)
        lam_max = np.minimum(up.min(axis=1), dn.min(axis=1))
        lin, quad = D @ (Qi @ x + ci), np.einsum("ki,ij,kj->k", D, Qi, D)
        for lam in range(1, int(lam_max.max(initial=0)) + 1):
            ok = lam <= lam_max
            assert np.all(2 * lam * lin[ok] + lam * lam * quad[ok] >= 0), (t, lam)
    for t in (0, 499, 999):
        x1, f1, _, _ = ctx.augment(ds, Qs[t], cs[t], 0.0, bs[t], X0s[t])
        assert xb[t].tolist() == x1.tolist() and fb[t] == f1


def test_c3_large_set_properties(gpu_lib):
    """C3 (n = 300) with a direction set large enough for the 1,024-thread, unstaged augmentation path
    (|D| > 16,384, slot-major ELL read from global memory with the early exit at the first blocked coordinate):
    every incumbent's result is exact and locally optimal over D (Alg. 2's stopping rule), checked on the host
    in exact integers, and the best is the lexicographic argmin over the incumbents (reading #19)."""
    from synth import c3, feasible_points
    inst = c3()
    ctx = gpu_lib.Context(inst.A, inst.l, inst.u)
    ds = ctx.extract(16384, inst.steps, inst.lr, inst.seed)
    S = ds.rows().astype(np.int64)
    assert 2 * len(S) > 16384
    D = np.concatenate([S, -S])
    X0 = feasible_points(inst, 6, seed=5)
    Qi, ci = np.asarray(inst.Q, np.int64), np.asarray(inst.c, np.int64)
    l, u = inst.l.astype(np.int64), inst.u.astype(np.int64)
    finals = []
    for x0 in X0:
        xb, fb, st, it = ctx.augment(ds, inst.Q, inst.c, inst.c0, inst.b, x0[None, :])
        x = xb.astype(np.int64)
        assert np.all(inst.A @ x == inst.b) and np.all(x >= l) and np.all(x <= u)
        two_f = int(x @ Qi @ x + 2 * ci @ x + 2 * inst.c0)
        assert 2 * fb == two_f
        assert two_f <= int(x0 @ Qi @ x0 + 2 * ci @ x0 + 2 * inst.c0)
        with np.errstate(divide="ignore"):
            up = np.where(D > 0, (u - x)[None, :] // np.where(D > 0, D, 1), np.iinfo(np.int64).max)
            dn = np.where(D < 0, (x - l)[None, :] // np.where(D < 0, -D, 1), np.iinfo(np.int64).max)
        lam_max = np.minimum(up.min(axis=1), dn.min(axis=1))
        lin, quad = D @ (Qi @ x + ci), np.einsum("ki,ij,kj->k", D, Qi, D)
        for lam in range(1, int(lam_max.max(initial=0)) + 1):
            ok = lam <= lam_max
            assert np.all(2 * lam * lin[ok] + lam * lam * quad[ok] >= 0), lam
        finals.append((two_f, x.tolist()))
    xb, fb, _, _ = ctx.augment(ds, inst.Q, inst.c, inst.c0, inst.b, X0)
    assert (2 * fb, xb.tolist()) == min(finals)
