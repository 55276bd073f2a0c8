"""GPU parity of the extraction path (C ABI) against the oracle, gates G1-G3 of DESIGN.md §4:

  G1 integer post-processing bit-exact given the same candidate multiset (check, dedupe + sign twins,
     ⊑ filter, lex sort), including edge cases (empty, single, duplicates, twins, ragged sizes);
  G2 descent iterates: every start within 1e-4 per coordinate at small T; at the stated T the fraction of
     starts within 1e-4 of the fp64 oracle is no worse than IEEE fp32 arithmetic of the same algorithm;
  G3 ⊑-minimal sets (same B, seed, starts): Jaccard >= 0.99, every disagreement passes the invariants.
"""
import numpy as np
import pytest

from oracle import extraction as OX
from oracle import lattice as OL
from oracle import graver as OG
from oracle import postprocess as OP

pytestmark = pytest.mark.gpu


SIMT, TC = 1, 2


def _ctx(maple, inst, kernel=0):
    ctx = maple.Context(inst.A, inst.l, inst.u, device=0)
    ctx.set_descent_kernel(kernel)
    return ctx


def _set(rows):
    return {tuple(int(v) for v in r) for r in np.asarray(rows).tolist()}


def _jaccard(a, b):
    return 1.0 if not (a | b) else len(a & b) / len(a | b)


def _pass_frac(Z, Zref, tol=1e-4):
    rel = np.abs(Z.astype(np.float64) - Zref) / np.maximum(1.0, np.abs(Zref))
    return float(np.mean(np.all(rel <= tol, axis=1)))


@pytest.mark.parametrize("name", ["C1", "C2a", "C2b"])
def test_basis_and_starts_match_oracle(gpu_lib, name):
    """The context's exported B is a saturated, LLL-reduced kernel basis by the oracle's exact checkers (Thm. 1,
    Def. P:136-144), and the device starts z0 = B+ g0 equal the oracle's (its own pseudoinverse of that B)."""
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst)
    assert OL.is_kernel_basis(inst.A, ctx.B.tolist())
    assert OL.is_lll_reduced(ctx.B.tolist())
    Z, Z0 = ctx.debug_descent(4096, 100, 612, 1, 0.01, 7)
    _, z0 = OX.sample_starts(inst.l, inst.u, OL.pinv(ctx.B), 7, np.arange(100, 612))
    np.testing.assert_allclose(Z0, z0, rtol=1e-12, atol=1e-12)     # fp64 on both sides


@pytest.mark.parametrize("kernel", [SIMT, TC])
@pytest.mark.parametrize("name,T", [("C1", 1), ("C1", 5), ("C2a", 1), ("C2a", 5), ("C2b", 5)])
def test_descent_iterates_small_T_all_starts(gpu_lib, name, T, kernel):
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst, kernel)
    N = 1000 if name == "C1" else 1000
    Z, _ = ctx.debug_descent(N, 0, N, T, inst.lr, 11)
    _, z0 = OX.sample_starts(inst.l, inst.u, OL.pinv(ctx.B), 11, np.arange(N))
    Zo = OX.descend(z0, ctx.B, T, inst.lr)
    assert _pass_frac(Z, Zo) >= 0.999


@pytest.mark.parametrize("kernel", [SIMT, TC])
@pytest.mark.parametrize("name,T", [("C1", 50), ("C1", 200), ("C2a", 50), ("C2a", 200)])
def test_descent_iterates_gate_g2(gpu_lib, name, T, kernel):
    """pass_frac(GPU vs fp64) >= pass_frac(fp32 oracle vs fp64) - 0.005 (the method is chaotic: even exact
    fp32 arithmetic loses 1e-4 agreement on some starts)."""
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst, kernel)
    N = 1024
    Z, _ = ctx.debug_descent(N, 0, N, T, inst.lr, inst.seed)
    _, z0 = OX.sample_starts(inst.l, inst.u, OL.pinv(ctx.B), inst.seed, np.arange(N))
    Z64 = OX.descend(z0, ctx.B, T, inst.lr)
    Z32 = OX.descend(z0.astype(np.float32), ctx.B, T, inst.lr, dtype=np.float32)
    gpu, ref = _pass_frac(Z, Z64), _pass_frac(Z32, Z64)
    print(f"{name} T={T} kernel={kernel}: gpu pass {gpu:.4f}, fp32-oracle pass {ref:.4f}")
    assert gpu >= ref - 0.005


@pytest.mark.parametrize("kernel", [SIMT, TC])
@pytest.mark.parametrize("name,N,filt", [("C1", 1024, 1), ("C1", 1024, 0), ("C2a", 1024, 1), ("C2a", 1024, 0),
                                         ("C2b", 512, 1)])
def test_postprocess_bit_exact_on_gpu_candidates(gpu_lib, name, N, filt, kernel):
    """G1: the oracle's check -> dedupe -> ⊑ filter -> lex sort of the GPU's candidate multiset equals the
    GPU's output byte for byte."""
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst, kernel)
    ctx.set_params(filter_minimal=bool(filt))
    ctx.set_debug(True)
    ds = ctx.extract(N, inst.steps, inst.lr, inst.seed)
    cand = ctx.candidates()
    assert cand.shape[0] > 0
    assert np.all(OP.check_rows(inst.A, inst.l, inst.u, cand))        # harvest soundness (C1-C3)
    ref, nbad = OP.postprocess(inst.A, inst.l, inst.u, cand, filter_minimal=bool(filt))
    assert nbad == 0
    assert [tuple(r) for r in ds.rows().tolist()] == ref
    assert ds.pool_size == len(OP.dedupe(cand))


@pytest.mark.parametrize("kernel", [SIMT, TC])
@pytest.mark.parametrize("name,N", [("C1", 1024), ("C2a", 1024)])
def test_sets_match_oracle_g3(gpu_lib, name, N, kernel):
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst, kernel)
    ds = ctx.extract(N, inst.steps, inst.lr, inst.seed)
    gpu_min = _set(ds.rows())
    pool, _ = OX.extract_pool(ctx.B, OL.pinv(ctx.B), inst.l, inst.u, N, inst.steps, inst.lr, inst.seed)
    ora_min = OP.minimal_filter(pool)
    j = _jaccard(gpu_min, ora_min)
    print(f"{name} kernel={kernel}: |gpu|={len(gpu_min)} |oracle|={len(ora_min)} jaccard={j:.4f}")
    assert j >= 0.99
    diff = np.array(sorted(gpu_min ^ ora_min), dtype=np.int64).reshape(-1, inst.n)
    if diff.size:
        assert np.all(OP.check_rows(inst.A, inst.l, inst.u, diff))
    assert OP.is_antichain(gpu_min)


def test_c1_minimal_is_closed_form(gpu_lib):
    from synth import c1
    inst = c1()
    ctx = _ctx(gpu_lib, inst)
    ds = ctx.extract(inst.n_starts, inst.steps, inst.lr, inst.seed)
    expected = {OG.canonical(g) for g in OG.graver_in_box(inst.A, [-3] * 4, [3] * 4)}
    assert _set(ds.rows()) == expected


def _random_kernel_rows(B, box, k, seed):
    rng = np.random.default_rng(seed)
    rows = []
    while len(rows) < k:
        z = rng.integers(-2, 3, size=B.shape[1]) * (rng.random(B.shape[1]) < 0.15)
        g = B @ z
        if np.any(g) and np.all(np.abs(g) <= box):
            rows.append(g if rng.random() < 0.7 else -g)
    rows = np.array(rows)
    dup = rows[rng.integers(0, len(rows), size=k // 3)]
    out = np.concatenate([rows, dup, -dup])
    return out[rng.permutation(len(out))]


@pytest.mark.parametrize("k", [0, 1, 2, 255, 256, 257, 1000, 5000])
@pytest.mark.parametrize("filt", [1, 0])
def test_merge_edge_cases_bit_exact(gpu_lib, k, filt):
    from synth import c2b
    inst = c2b()
    ctx = _ctx(gpu_lib, inst)
    box = inst.u - inst.l
    rows = _random_kernel_rows(ctx.B, box, max(k, 1), seed=k)[:k] if k else np.zeros((0, inst.n), np.int64)
    if k >= 2:  # a few invalid rows: not in the kernel, out of the box, zero
        bad = np.repeat(rows[:1], 3, axis=0)
        bad[0, 0] += 1
        bad[1, :] = 0
        bad[2, 0] = box[0] + 1 if box[0] < 127 else bad[2, 0]
        rows = np.concatenate([rows, bad])
    ds = ctx.dirset_from_host(rows, filter_minimal=bool(filt))
    ref, _ = OP.postprocess(inst.A, inst.l, inst.u, rows, filter_minimal=bool(filt))
    assert [tuple(r) for r in ds.rows().tolist()] == ref


def test_range_partition_invariance(gpu_lib):
    """maple_extract over N starts == merge of maple_extract_range over a 3-way partition (W-invariance)."""
    from synth import c2a
    inst = c2a()
    ctx = _ctx(gpu_lib, inst)
    N = 3000
    full = ctx.extract(N, 100, inst.lr, 5).rows()
    parts = [ctx.extract_range(N, a, b, 100, inst.lr, 5).rows() for a, b in ((0, 1000), (1000, 1001), (1001, 3000))]
    merged = ctx.dirset_from_host(np.concatenate(parts), filter_minimal=True).rows()
    np.testing.assert_array_equal(full, merged)
    again = ctx.extract(N, 100, inst.lr, 5).rows()
    np.testing.assert_array_equal(full, again)                       # determinism across runs


def test_merge_device_rows(gpu_lib):
    import torch
    from synth import c2a
    inst = c2a()
    ctx = _ctx(gpu_lib, inst)
    a = ctx.extract_range(2000, 0, 1000, 100, inst.lr, 9)
    b = ctx.extract_range(2000, 1000, 2000, 100, inst.lr, 9)
    st = a.stride
    buf = torch.zeros((a.size + b.size, st), dtype=torch.int8, device="cuda")
    ra, rb = torch.from_numpy(a.rows().astype(np.int8)), torch.from_numpy(b.rows().astype(np.int8))
    buf[:a.size, :inst.n] = ra.cuda()
    buf[a.size:, :inst.n] = -rb.cuda()          # negated twins must collapse too
    torch.cuda.synchronize()
    m = ctx.merge_device(buf.data_ptr(), a.size + b.size, st).rows()
    full = ctx.extract(2000, 100, inst.lr, 9).rows()
    np.testing.assert_array_equal(m, full)


def test_extract_errors(gpu_lib):
    from synth import c1
    inst = c1()
    ctx = _ctx(gpu_lib, inst)
    for args in [(0, 10, 0.01, 1), (10, 0, 0.01, 1), (10, 10, 0.0, 1), (10, 10, -1.0, 1)]:
        with pytest.raises(gpu_lib.MapleError) as e:
            ctx.extract(*args)
        assert e.value.name == "BAD_ARG"
    with pytest.raises(gpu_lib.MapleError) as e:
        ctx.extract_range(10, 5, 11, 10, 0.01, 1)
    assert e.value.name == "BAD_ARG"
    with pytest.raises(gpu_lib.MapleError) as e:
        gpu_lib.Context(inst.A, inst.u, inst.l)
    assert e.value.name == "BAD_BOUNDS"
    with pytest.raises(gpu_lib.MapleError) as e:
        ctx.set_params(lambda1=-1.0)
    assert e.value.name == "BAD_ARG"


def test_umma_selftest_exact(gpu_lib):
    """tcgen05 descriptors and operand layout: single-tile products of small integers are exact."""
    rng = np.random.default_rng(0)
    A1 = rng.integers(-3, 4, size=(128, 48)).astype(np.float32)
    B1 = rng.integers(-3, 4, size=(64, 48)).astype(np.float32)
    A2 = rng.integers(-3, 4, size=(128, 64)).astype(np.float32)
    B2 = rng.integers(-3, 4, size=(48, 64)).astype(np.float32)
    D1, D2 = gpu_lib.maple_selftest_umma(A1, B1, A2, B2)
    np.testing.assert_array_equal(D1, A1 @ B1.T)
    np.testing.assert_array_equal(D2, A2 @ B2.T)


@pytest.mark.parametrize("name", ["C1", "C2a"])
def test_tc_and_simt_kernels_agree(gpu_lib, name):
    """Both descent kernels implement the same fp32 algorithm: iterates agree at small T for every start,
    and the extracted ⊑-minimal sets agree at the stated T."""
    from synth import config
    inst = config(name)
    a, b = _ctx(gpu_lib, inst, SIMT), _ctx(gpu_lib, inst, TC)
    Za, _ = a.debug_descent(777, 0, 777, 10, inst.lr, 3)
    Zb, _ = b.debug_descent(777, 0, 777, 10, inst.lr, 3)
    assert _pass_frac(Zb, Za.astype(np.float64)) >= 0.999
    sa, sb = _set(a.extract(2048, inst.steps, inst.lr, 3).rows()), _set(b.extract(2048, inst.steps, inst.lr, 3).rows())
    assert _jaccard(sa, sb) >= 0.99


@pytest.mark.parametrize("name,N", [("C1", 1024), ("C2a", 8192), ("C2b", 8192), ("C3", 4096)])
def test_filter_algorithms_identical(gpu_lib, name, N):
    """The tiled, the indexed and the level-synchronous ⊑ filter enumerate different pairs but decide the same
    pairwise property: identical kept sets (bit for bit), and G1 against the oracle on the GPU candidates."""
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst)
    out = []
    for algo in (1, 2, 3):
        ctx.set_filter_algorithm(algo)
        ctx.set_debug(True)
        out.append(ctx.extract(N, inst.steps, inst.lr, inst.seed).rows())
        if name == "C1":   # (the other shapes' G1 tests run through the auto filter)
            ref, nbad = OP.postprocess(inst.A, inst.l, inst.u, ctx.candidates())
            assert nbad == 0 and [tuple(r) for r in out[-1].tolist()] == ref
    np.testing.assert_array_equal(out[0], out[1])
    np.testing.assert_array_equal(out[0], out[2])


@pytest.mark.parametrize("name,kernel", [("C1", TC), ("C1", SIMT), ("C2a", TC), ("C2a", SIMT), ("C3", SIMT)])
@pytest.mark.parametrize("opt", ["gd", "signgd"])
def test_descent_variants_iterates(gpu_lib, name, kernel, opt):
    """Readings #24 (GD, sign-GD): per-start iterates vs the fp64 oracle — every start within 1e-4 at T = 5;
    at T = 50 no worse than IEEE fp32 arithmetic of the same algorithm (gate G2)."""
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst, kernel)
    ctx.set_descent_variant(opt)
    N = 1000 if name != "C3" else 128
    _, z0 = OX.sample_starts(inst.l, inst.u, OL.pinv(ctx.B), inst.seed, np.arange(N))
    Z, _ = ctx.debug_descent(N, 0, N, 5, inst.lr, inst.seed)
    assert _pass_frac(Z, OX.descend(z0, ctx.B, 5, inst.lr, optimizer=opt)) >= 0.999
    Z, _ = ctx.debug_descent(N, 0, N, 50, inst.lr, inst.seed)
    Z64 = OX.descend(z0, ctx.B, 50, inst.lr, optimizer=opt)
    Z32 = OX.descend(z0.astype(np.float32), ctx.B, 50, inst.lr, optimizer=opt, dtype=np.float32)
    assert _pass_frac(Z, Z64) >= _pass_frac(Z32, Z64) - 0.005


@pytest.mark.parametrize("name,kernel", [("C1", TC), ("C2a", TC), ("C2a", SIMT), ("C2b", TC), ("C3", SIMT)])
@pytest.mark.parametrize("opt", ["adam", "signgd"])
def test_final_only_harvest_bit_exact(gpu_lib, name, kernel, opt):
    """Reading #25: with the final-only harvest the candidate set is exactly the oracle's harvest (B⌈z⌋ in
    the box, g != 0, canonical) of the GPU's own final iterates, and the post-processing of those candidates
    is bit-exact (G1)."""
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst, kernel)
    ctx.set_descent_variant(opt, harvest_final=True)
    N = 777 if name != "C3" else 96
    Z, _ = ctx.debug_descent(N, 0, N, inst.steps, inst.lr, inst.seed)
    ctx.set_debug(True)
    ds = ctx.extract(N, inst.steps, inst.lr, inst.seed)
    cand = ctx.candidates()
    assert _set(cand) == _set(OX.harvest(Z.astype(np.float64), ctx.B, inst.l, inst.u))
    ref, nbad = OP.postprocess(inst.A, inst.l, inst.u, cand)
    assert nbad == 0 and [tuple(r) for r in ds.rows().tolist()] == ref


def test_variant_c1_sets_within_closed_form(gpu_lib):
    """Every variant on BASELINE configs[0]: exact rows, ⊑-minimal set inside {e_i - e_j}."""
    from synth import c1
    inst = c1()
    expected = {OG.canonical(g) for g in OG.graver_in_box(inst.A, [-3] * 4, [3] * 4)}
    for opt in ("gd", "signgd"):
        for fin in (False, True):
            ctx = _ctx(gpu_lib, inst)
            ctx.set_descent_variant(opt, harvest_final=fin)
            rows = ctx.extract(1024, inst.steps, inst.lr, inst.seed).rows()
            assert np.all(OP.check_rows(inst.A, inst.l, inst.u, rows))
            assert _set(rows) <= expected


@pytest.mark.parametrize("name,N", [("C2b", 8192), ("C3", 4096)])
def test_level_filter_fallback_identical(gpu_lib, name, N, monkeypatch):
    """The level-synchronous filter falls back to the indexed pass when its G lists exceed their capacity
    (MAPLE_GL_CAP, a test hook, forces it): the kept set stays bit-identical to the indexed algorithm."""
    from synth import config
    inst = config(name)
    ctx = _ctx(gpu_lib, inst)
    ctx.set_filter_algorithm(2)
    ref = ctx.extract(N, inst.steps, inst.lr, inst.seed).rows()
    ctx.set_filter_algorithm(3)
    monkeypatch.setenv("MAPLE_GL_CAP", "1")
    forced = ctx.extract(N, inst.steps, inst.lr, inst.seed).rows()
    monkeypatch.delenv("MAPLE_GL_CAP")
    normal = ctx.extract(N, inst.steps, inst.lr, inst.seed).rows()
    np.testing.assert_array_equal(forced, ref)
    np.testing.assert_array_equal(normal, ref)
