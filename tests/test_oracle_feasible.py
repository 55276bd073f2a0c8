"""Pins for oracle/feasible.py — Eq. 4: SPEC worked examples S:319-330, finite differences of
the gradient, projection invariant, and the claim of P:428 (an exact zero of Eq. 4 is a feasible point)."""
import itertools

import numpy as np
import pytest

from oracle import feasible as F


def test_loss_examples():
    assert F.loss([2, 2], [[1, 1]], [4]) == 0.0                       # S:319 feasible integer -> 0
    assert F.loss([0.5], [[1]], [1]) == pytest.approx(0.275)
    assert F.loss([1, 1], [[1, 1]], [4]) == pytest.approx(4.0)


def test_gradient_finite_differences():
    rng = np.random.default_rng(2)
    for _ in range(200):
        m, n = rng.integers(1, 4), rng.integers(2, 6)
        A = rng.integers(-3, 4, size=(m, n))
        b = rng.integers(-4, 5, size=m)
        x = rng.uniform(-2, 3, size=n)
        if np.min(np.abs(x - np.round(x))) < 1e-3:
            continue
        g = F.grad(x[None, :], A, b)[0]
        h = 1e-6
        fd = np.array([(F.loss(x + h * e, A, b) - F.loss(x - h * e, A, b)) / (2 * h) for e in np.eye(n)])
        np.testing.assert_allclose(g, fd, rtol=1e-4, atol=1e-4)


def test_feasible_set_examples():
    pts, X = F.feasible_set([[1, 1]], [4], [0, 0], [3, 3], 64, 300, 0.05, seed=1)
    assert set(pts) <= {(1, 3), (2, 2), (3, 1)} and len(pts) >= 1
    assert F.feasible_set([[2, 2]], [3], [0, 0], [3, 3], 64, 300, 0.05, seed=1)[0] == []   # S:329 parity
    pts, _ = F.feasible_set([[1, 2]], [5], [1, 2], [1, 2], 8, 50, 0.05, seed=1)           # S:330 l = u = x0
    assert pts == [(1, 2)]
    assert np.all(X >= 0) and np.all(X <= 3)                               # projection onto [l, u]


def test_results_are_exactly_the_feasible_points_found():
    from synth import semi_assignment
    inst = semi_assignment(3, 4, gen_seed=3)
    pts, _ = F.feasible_set(inst.A, inst.b, inst.l, inst.u, 128, 300, 0.05, seed=5)
    S = {p for p in itertools.product(*[range(int(a), int(c) + 1) for a, c in zip(inst.l, inst.u)])
         if np.all(inst.A @ np.array(p) == inst.b)}
    assert set(pts) <= S and len(pts) > 0
    assert pts == sorted(pts)


def test_projected_adam_matches_torch():
    """Readings F2-F3 pinned to library routines: the Eq. 4 loss differentiated by torch autograd (not F.grad),
    stepped by torch.optim.Adam (the paper's optimizer, PyTorch 2.1.0 P:452) and projected with clamp_
    onto [l, u] after every step, equals feasible.descend in fp64 (a bias-correction, projection-order or
    gradient slip fails this)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(12)
    for trial in range(6):
        m, n = int(rng.integers(1, 4)), int(rng.integers(3, 7))
        A = rng.integers(-3, 4, size=(m, n))
        b = rng.integers(-4, 5, size=m)
        l = rng.integers(-2, 1, size=n)
        u = l + rng.integers(1, 4, size=n)
        X0 = F.starts(l, u, 7 + trial, np.arange(5))
        steps, lr, lam3 = 40, 0.05, 0.1
        ref = F.descend(X0, A, b, l, u, steps, lr, lam3=lam3)
        x = torch.tensor(X0, dtype=torch.float64, requires_grad=True)
        At = torch.tensor(A, dtype=torch.float64)
        bt = torch.tensor(b, dtype=torch.float64)
        lo = torch.tensor(l, dtype=torch.float64)
        hi = torch.tensor(u, dtype=torch.float64)
        opt = torch.optim.Adam([x], lr=lr, betas=(0.9, 0.999), eps=1e-8)
        for _ in range(steps):
            opt.zero_grad()
            r = x @ At.T - bt
            f = (r * r).sum() + lam3 * ((x - torch.floor(x)) * (torch.ceil(x) - x)).sum()
            f.backward()
            opt.step()
            with torch.no_grad():
                x.clamp_(min=lo, max=hi)
        np.testing.assert_allclose(x.detach().numpy(), ref, rtol=1e-10, atol=1e-10)
