"""Pins for oracle/extraction.py: Eq. 3 worked values, finite differences,
the Adam formula against torch.optim.Adam (the library routine the paper ran), start sampling
(P:386), and end-to-end Alg. 3 against closed-form Graver bases (BASELINE configs[0])."""
import numpy as np
import pytest

from oracle import extraction as X
from oracle import graver as Gv
from oracle import lattice as L
from oracle import postprocess as PP


def test_loss_worked_examples():
    B = np.array([[1.0], [-1.0]])
    assert X.loss([2.0], B) == pytest.approx(4.0)
    assert X.loss([0.5], B) == pytest.approx(2.2125, abs=1e-12)
    assert X.loss([0.0], B) == pytest.approx(1.0 * (1e8 - 1.0))         # S:229 (clamped)
    # lam1 term by hand at z = 1.25: (0.25)(0.75) = 0.1875
    assert X.loss([1.25], B) == pytest.approx(2.5 + 0.85 * 0.1875)


def test_subgradient_worked_examples():
    B = np.array([[1.0], [-1.0]])
    # z = 0.5: B^T sign(Bz) = 2, lam1-term derivative 0 at the midpoint, lam2 term -1/0.25 = -4
    assert X.subgrad(np.array([[0.5]]), B, 0.85, 1.0)[0, 0] == pytest.approx(-2.0)
    # integer z, ||z||_inf >= 1, Bz without zeros: exactly B^T sign(Bz)
    B2 = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, -1.0]])
    g = X.subgrad(np.array([[2.0, -1.0]]), B2, 0.85, 1.0)[0]
    np.testing.assert_array_equal(g, B2.T @ np.sign(B2 @ np.array([2.0, -1.0])))
    # sign(0) = 0 and the lam2 term is 0 at z = 0
    assert np.all(X.subgrad(np.zeros((1, 2)), B2, 0.85, 1.0) == 0)


def test_subgradient_finite_differences():
    """central differences (h = 1e-6) match to 1e-4 relative at 300 random non-kink points."""
    rng = np.random.default_rng(7)
    checked = 0
    while checked < 300:
        n, d = rng.integers(2, 7), rng.integers(1, 5)
        B = rng.integers(-3, 4, size=(n, d)).astype(float)
        z = rng.uniform(-2.5, 2.5, size=d)
        Bz = B @ z
        frac = np.abs(z - np.round(z))
        zinf = np.abs(z).max()
        if (np.min(np.abs(Bz)) < 1e-3 or np.min(np.abs(frac - 0.0)) < 1e-3 or abs(zinf - 1) < 1e-3
                or (np.sort(np.abs(z))[-2:] if d > 1 else [0, 1])[0] > zinf - 1e-3 and d > 1):
            continue
        g = X.subgrad(z[None, :], B, 0.85, 1.0)[0]
        h = 1e-6
        fd = np.array([(X.loss(z + h * e, B) - X.loss(z - h * e, B)) / (2 * h) for e in np.eye(d)])
        np.testing.assert_allclose(g, fd, rtol=1e-4, atol=1e-4)
        checked += 1


def test_adam_matches_torch():
    """Reading #9: the update is torch.optim.Adam's (P:452 used PyTorch 2.1.0); fp64, 25 steps."""
    torch = pytest.importorskip("torch")
    B = np.array([[1, -1, 0], [0, 1, -1], [1, 0, 1], [2, -1, 1]], dtype=np.float64)
    rng = np.random.default_rng(3)
    z0 = rng.uniform(-2, 2, size=(5, 3))
    ours = X.descend(z0, B, steps=25, lr=0.05)
    p = torch.tensor(z0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([p], lr=0.05, betas=(0.9, 0.999), eps=1e-8)
    for _ in range(25):
        opt.zero_grad()
        p.grad = torch.from_numpy(X.subgrad(p.detach().numpy().copy(), B, 0.85, 1.0))
        opt.step()
    np.testing.assert_allclose(ours, p.detach().numpy(), rtol=1e-11, atol=1e-12)


def test_round_half_away():
    z = np.array([-2.5, -1.5, -0.5, -0.49999999999999994, 0.0, 0.4999999, 0.5, 1.5, 2.5, 2.4999999])
    assert X.round_half_away(z).tolist() == [-3, -2, -1, 0, 0, 0, 1, 2, 3, 2]
    assert X.round_half_away(np.float32([0.5, -0.5, 1.49999988])).tolist() == [1, -1, 1]


def test_rng_and_starts():
    U = X.uniforms(1, np.arange(4096), 8)
    assert U.min() >= 0 and U.max() < 1
    assert abs(U.mean() - 0.5) < 0.01
    # splitmix64 reference value: the published first output of splitmix64 seeded with 0 is
    # 0xE220A8397B1DCDAF, i.e. mix(0x9E3779B97F4A7C15 - 0x9E3779B97F4A7C15 + ...) = mix(0)
    assert int(X.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    inst_l, inst_u = np.zeros(3, np.int64), np.full(3, 2)
    B = np.array([[1, 0], [-1, 1], [0, -1]])
    Bp = L.pinv(B)
    g0, z0 = X.sample_starts(inst_l, inst_u, Bp, 5, np.arange(10))
    assert np.all(g0 >= -2) and np.all(g0 < 2)
    _, z0b = X.sample_starts(inst_l, inst_u, Bp, 5, np.arange(4, 10))       # range invariance
    np.testing.assert_array_equal(z0[4:], z0b)
    _, zd = X.sample_starts(inst_u, inst_u, Bp, 5, np.arange(10))           # l = u -> g = 0 -> z = 0
    assert np.all(zd == 0)


def _c1_problem():
    from synth import c1
    inst = c1()
    B = L.lll_reduce(L.kernel_basis(inst.A))
    return inst, np.array(B, dtype=np.int64)


def test_c1_extraction_recovers_graver_closed_form():
    """BASELINE configs[0]: N=1024, T=200, lr=0.01; ⊑-minimal set of the pool = {e_i - e_j} (6 canonical)."""
    inst, B = _c1_problem()
    pool, Z = X.extract_pool(B, L.pinv(B), inst.l, inst.u, 1024, 200, 0.01, seed=1)
    assert Z.shape == (1024, 3)
    rows = np.array(sorted(pool))
    assert np.all(PP.check_rows(inst.A, inst.l, inst.u, rows))                  # soundness (C1-C3)
    minimal = PP.minimal_filter(pool)
    expected = {Gv.canonical(g) for g in Gv.graver_in_box(inst.A, [-3] * 4, [3] * 4)}
    assert minimal == expected and len(minimal) == 6


def test_extraction_start_partition_invariance():
    """S:270 / SPEC acceptance #6: the pool is the same for any partition of the starts."""
    inst, B = _c1_problem()
    Bp = L.pinv(B)
    full, Zf = X.extract_pool(B, Bp, inst.l, inst.u, 256, 50, 0.01, seed=3)
    a, Za = X.extract_pool(B, Bp, inst.l, inst.u, 256, 50, 0.01, seed=3, starts=np.arange(0, 100))
    b, Zb = X.extract_pool(B, Bp, inst.l, inst.u, 256, 50, 0.01, seed=3, starts=np.arange(100, 256))
    assert full == a | b
    np.testing.assert_array_equal(Zf, np.concatenate([Za, Zb]))


def test_semi_assignment_extraction_sound_and_near_complete():
    """Semi-assignment 5 x 6 (closed form: 5 * C(6,2) = 75 canonical). Every minimal element found is a
    Graver element (soundness) and the recall is high."""
    from synth import semi_assignment
    inst = semi_assignment(5, 6, gen_seed=11)
    B = np.array(L.lll_reduce(L.kernel_basis(inst.A)), dtype=np.int64)
    pool, _ = X.extract_pool(B, L.pinv(B), inst.l, inst.u, 512, 200, 0.01, seed=4)
    minimal = PP.minimal_filter(pool)
    closed = set()
    for r in range(5):
        for i in range(6):
            for j in range(i + 1, 6):
                v = [0] * 30
                v[6 * r + i], v[6 * r + j] = 1, -1
                closed.add(tuple(v))
    assert minimal <= closed
    assert len(minimal) >= 0.95 * len(closed)


def test_fp32_mode_runs_same_algorithm():
    inst, B = _c1_problem()
    Bp = L.pinv(B)
    _, z0 = X.sample_starts(inst.l, inst.u, Bp, 1, np.arange(64))
    Z64 = X.descend(z0, B, 5, 0.01)
    Z32 = X.descend(z0.astype(np.float32), B, 5, 0.01, dtype=np.float32)
    assert Z32.dtype == np.float32
    np.testing.assert_allclose(Z32, Z64, rtol=1e-5, atol=1e-5)


def test_gd_matches_torch_sgd():
    """Reading #24, plain GD (a first-order method): z <- z - lr g is torch.optim.SGD without momentum."""
    torch = pytest.importorskip("torch")
    B = np.array([[1, -1, 0], [0, 1, -1], [1, 0, 1], [2, -1, 1]], dtype=np.float64)
    z0 = np.random.default_rng(4).uniform(-2, 2, size=(5, 3))
    ours = X.descend(z0, B, steps=25, lr=0.05, optimizer="gd")
    p = torch.tensor(z0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([p], lr=0.05)
    for _ in range(25):
        opt.zero_grad()
        p.grad = torch.from_numpy(X.subgrad(p.detach().numpy().copy(), B, 0.85, 1.0))
        opt.step()
    np.testing.assert_allclose(ours, p.detach().numpy(), rtol=1e-13, atol=1e-14)


def test_signgd_moves_each_coordinate_by_lr_against_the_subgradient():
    """Reading #24, sign-GD: every coordinate moves by exactly lr (or 0 where the subgradient is 0), opposite
    to the subgradient's sign; at the λ1 = λ2 = 0 limit on B = (1, -1)^T from z = 0.3 the ℓ1 term alone
    walks z down by lr per step until it crosses 0, then oscillates within lr of 0."""
    B = np.array([[1, -1, 0], [0, 1, -1], [1, 0, 1], [2, -1, 1]], dtype=np.float64)
    z0 = np.random.default_rng(5).uniform(-2, 2, size=(64, 3))
    g = X.subgrad(z0, B, 0.85, 1.0)
    z1 = X.descend(z0, B, steps=1, lr=0.0625, optimizer="signgd")   # lr = 2^-4: z0 - lr is exact here
    step = z0 - z1
    np.testing.assert_array_equal(np.abs(step)[g != 0], 0.0625)
    np.testing.assert_array_equal(np.sign(step), np.sign(g))
    traj = []
    X.descend(np.array([[0.3]]), np.array([[1.0], [-1.0]]), steps=8, lr=0.0625, lam1=0.0, lam2=0.0,
              optimizer="signgd", trace=traj)
    zs = [float(t[0, 0]) for t in traj]
    assert zs[:4] == [0.3 - 0.0625 * k for k in range(1, 5)]
    assert all(abs(z) <= 0.0625 for z in zs[4:])


def test_variant_extractions_on_c1_are_graver():
    """Readings #24/#25 at BASELINE configs[0]: every optimizer variant and the final-only harvest yield
    kernel elements in the box (soundness), a ⊑-minimal set inside the closed form {e_i - e_j}, and the
    final-only pool is exactly the harvest of the final iterates (a subset of the every-step pool)."""
    inst, B = _c1_problem()
    expected = {Gv.canonical(g) for g in Gv.graver_in_box(inst.A, [-3] * 4, [3] * 4)}
    for opt in ("gd", "signgd"):
        pool, _ = X.extract_pool(B, L.pinv(B), inst.l, inst.u, 512, 200, 0.01, seed=1, optimizer=opt)
        rows = np.array(sorted(pool))
        assert len(pool) > 0 and np.all(PP.check_rows(inst.A, inst.l, inst.u, rows))
        assert PP.minimal_filter(pool) <= expected
    every, _ = X.extract_pool(B, L.pinv(B), inst.l, inst.u, 256, 100, 0.01, seed=2)
    final, Z = X.extract_pool(B, L.pinv(B), inst.l, inst.u, 256, 100, 0.01, seed=2, harvest_final=True)
    assert final <= every
    assert final == {tuple(int(x) for x in r) for r in X.harvest(Z, B, inst.l, inst.u)}
