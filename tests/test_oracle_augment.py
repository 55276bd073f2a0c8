"""Pins for oracle/augment.py: SPEC worked examples, Prop. 3 — with the true
Graver basis, augmentation on separable convex f reaches the brute-force optimum from every feasible
start — and the monotonicity / feasibility invariants of Alg. 2."""
import itertools

import numpy as np
import pytest

from oracle import augment as AU
from oracle import graver as Gv


def test_max_step_length_examples():
    assert AU.max_step_length((3, 1), (-1, 1), (0, 0), (3, 3)) == 2
    assert AU.max_step_length((1,), (1,), (0,), (5,)) == 4
    assert AU.max_step_length((3,), (1,), (0,), (3,)) == 0
    with pytest.raises(ValueError):
        AU.max_step_length((1, 1), (0, 0), (0, 0), (3, 3))


def test_best_step_example():
    f = AU.Objective(2 * np.eye(2), np.zeros(2))                          # f = x1^2 + x2^2
    lam, key = AU.best_step(f, (3, 1), (-1, 1), (0, 0), (3, 3))
    assert lam == 1 and key / 2 == 8
    assert AU.best_step(f, (0, 0), (1, -1), (0, 0), (3, 3)) is None       # lambda_max = 0
    assert AU.best_step(f, (1, 1), (1, -1), (0, 0), (3, 3)) is None       # no improvement


def test_augment_worked_instance():
    """A=[[1,1]], b=4, bounds [0,3]^2, f=(x1-2)^2+(x2-2)^2, pool {±(1,-1)}, start (3,1) -> (2,2)."""
    f = AU.Objective(2 * np.eye(2), [-4.0, -4.0], 8.0)
    x, it = AU.graver_best_augment(f, [[1, 1]], [4], [0, 0], [3, 3], [3, 1], [(1, -1)])
    assert x.tolist() == [2, 2] and it == 1 and f.value(x) == 0.0
    x, it = AU.graver_best_augment(f, [[1, 1]], [4], [0, 0], [3, 3], [2, 2], [(1, -1)])
    assert x.tolist() == [2, 2] and it == 0
    x, it = AU.graver_best_augment(f, [[1, 1]], [4], [0, 0], [3, 3], [3, 1], [])
    assert x.tolist() == [3, 1] and it == 0
    with pytest.raises(AU.InfeasibleStart):
        AU.graver_best_augment(f, [[1, 1]], [4], [0, 0], [3, 3], [3, 3], [(1, -1)])


def test_tie_break_lexicographic_g_then_lambda():
    # f = 0 everywhere except it rewards moving off x0 equally in two directions: ties broken by lex g
    f = AU.Objective(np.zeros((3, 3)), [1.0, 0.0, 0.0])
    S = [(1, -1, 0), (1, 0, -1)]
    x, it = AU.graver_best_augment(f, [[1, 1, 1]], [2], [0, 0, 0], [2, 2, 2], [2, 0, 0], S)
    # D sorted: (-1,0,1) < (-1,1,0) < (1,-1,0) < (1,0,-1); both -g decrease f by 1 per unit; lambda=2
    assert x.tolist() == [0, 0, 2] and it == 1


def _brute_optimum(f, A, b, l, u):
    pts = [np.array(p) for p in itertools.product(*[range(int(a), int(c) + 1) for a, c in zip(l, u)])]
    feas = [p for p in pts if np.all(np.asarray(A) @ p == b)]
    return feas, min(f.key(p) for p in feas)


@pytest.mark.parametrize("seed", range(20))
def test_prop3_separable_convex_reaches_optimum(seed):
    """SPEC acceptance #5: G(A) is a test set for separable convex f (Prop. 3)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 6))
    m = int(rng.integers(1, 3))
    A = rng.integers(-2, 3, size=(m, n))
    if np.linalg.matrix_rank(A.astype(float)) < m:
        A[0, 0] = 7
    u = np.full(n, 3)
    l = np.zeros(n, np.int64)
    xp = rng.integers(0, 4, size=n)
    b = A @ xp
    q = rng.integers(1, 4, size=n)                      # separable convex quadratic
    c = rng.integers(-8, 9, size=n)
    f = AU.Objective(np.diag(q).astype(float), c.astype(float))
    G = Gv.graver_in_box(A, -(u - l), u - l)
    S = {Gv.canonical(g) for g in G}
    feas, opt = _brute_optimum(f, A, b, l, u)
    for x0 in feas[:: max(1, len(feas) // 6)]:
        x, _ = AU.graver_best_augment(f, A, b, l, u, x0, S)
        assert AU.feasible(A, b, l, u, x)
        assert f.key(x) == opt


def test_monotone_and_feasible_trajectory():
    from synth import semi_assignment, feasible_points
    inst = semi_assignment(2, 4, gen_seed=5)
    f = AU.Objective(inst.Q, inst.c)
    S = {Gv.canonical(g) for g in Gv.graver_in_box(inst.A, [-1] * 8, [1] * 8)}
    D = AU.direction_list(S)
    for x0 in feasible_points(inst, 5, seed=9):
        x = x0.copy()
        prev = f.key(x)
        while True:
            best = None
            for gi, g in enumerate(D):
                r = AU.best_step(f, x, g, inst.l, inst.u)
                if r and (best is None or (r[1], gi, r[0]) < best):
                    best = (r[1], gi, r[0])
            if best is None:
                break
            x = x + best[2] * np.array(D[best[1]])
            assert AU.feasible(inst.A, inst.b, inst.l, inst.u, x)
            assert f.key(x) < prev
            prev = f.key(x)
        xa, _ = AU.graver_best_augment(f, inst.A, inst.b, inst.l, inst.u, x0, S)
        assert xa.tolist() == x.tolist()


def test_multi_start_best_tie_break():
    f = AU.Objective(np.zeros((2, 2)), np.zeros(2))
    xb, fb, finals = AU.multi_start(f, [[1, 1]], [2], [0, 0], [2, 2], [[2, 0], [1, 1], [0, 2]], [])
    assert xb.tolist() == [0, 2] and fb == 0.0 and len(finals) == 3


def test_exact_integer_objective():
    f = AU.Objective([[2, 1], [1, 2]], [3, -1], 5)
    assert f.exact
    x = np.array([4, -7])
    assert f.key(x) == int(x @ np.array([[2, 1], [1, 2]]) @ x + 2 * (3 * 4 + 7) + 10)
    g = AU.Objective(np.eye(2) * 0.5, [0.1, 0.2])
    assert not g.exact and g.value([1, 1]) == pytest.approx(0.5 + 0.3)


# ---- separable value tables (reading #27; Prop. 3: f(x) = sum_j f_j(x^j)) ----

def _tables(fns, l, u):
    return [[fj(t) for t in range(int(a), int(c) + 1)] for fj, a, c in zip(fns, l, u)]


def test_table_worked_value():
    """SeparableConvex f_j(t) = (t - 2)^2, x = (3, 1) -> 1 + 1 = 2."""
    f = AU.SeparableTable(_tables([lambda t: (t - 2) ** 2] * 2, [0, 0], [3, 3]), [0, 0])
    assert f.exact and f.value((3, 1)) == 2.0
    assert AU.SeparableTable(_tables([lambda t: (t - 2) ** 2] * 2, [-1, 1], [3, 3]), [-1, 1]).value((3, 1)) == 2.0


def test_table_matches_diagonal_quadratic():
    """The table of 1/2 q_j t^2 + c_j t is the SEPARABLE quadratic (Objective with diag Q): same ordering on
    every point of a box with a nonzero lower bound (catches an offset / index slip in the table lookup)."""
    rng = np.random.default_rng(4)
    n = 4
    l, u = rng.integers(-3, 1, size=n), rng.integers(1, 4, size=n)
    q, c = rng.integers(1, 5, size=n), rng.integers(-6, 7, size=n)
    fq = AU.Objective(np.diag(q).astype(float), c.astype(float), 3.0)
    ft = AU.SeparableTable(_tables([lambda t, a=a, b=b: 0.5 * a * t * t + b * t for a, b in zip(q, c)], l, u), l, 3.0)
    for p in itertools.product(*[range(int(a), int(b) + 1) for a, b in zip(l, u)]):
        assert ft.value(p) == fq.value(p)


@pytest.mark.parametrize("seed", range(12))
def test_prop3_table_convex_nonquadratic_reaches_optimum(seed):
    """Prop. 3 beyond quadratics: with the true Graver basis, augmentation on separable convex
    non-quadratic f_j (|t - a|^3, piecewise-linear max(w1 (a - t), w2 (t - a)), and 2^|t - a|) reaches the
    brute-force optimum from every feasible start."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 6))
    m = int(rng.integers(1, 3))
    A = rng.integers(-2, 3, size=(m, n))
    if np.linalg.matrix_rank(A.astype(float)) < m:
        A[0, 0] = 7
    l, u = np.zeros(n, np.int64), np.full(n, 3)
    b = A @ rng.integers(0, 4, size=n)
    fns = []
    for j in range(n):
        a = float(rng.integers(0, 4)) + 0.5 * float(rng.integers(0, 2))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            fns.append(lambda t, a=a: abs(t - a) ** 3)
        elif kind == 1:
            w1, w2 = int(rng.integers(1, 6)), int(rng.integers(1, 6))
            fns.append(lambda t, a=a, w1=w1, w2=w2: max(w1 * (a - t), w2 * (t - a)))
        else:
            fns.append(lambda t, a=a: 2.0 ** abs(t - a))
    f = AU.SeparableTable(_tables(fns, l, u), l, c0=1.25)
    S = {Gv.canonical(g) for g in Gv.graver_in_box(A, -(u - l), u - l)}
    feas, opt = _brute_optimum(f, A, b, l, u)
    for x0 in feas[:: max(1, len(feas) // 6)]:
        x, _ = AU.graver_best_augment(f, A, b, l, u, x0, S)
        assert AU.feasible(A, b, l, u, x)
        assert f.key(x) == opt
