"""CTA-pair tcgen05 descent (k_descent_tcp.cu, descent kernel 4) against the oracle: the large-shape path
(configs[2] = C3: n = 300, m = 20, d = 280). Gates of DESIGN.md §4 with the oracle's own pseudoinverse
(OL.pinv of the library's exported B): starts bit-for-bit in fp64 (1e-12), iterates at small T for every start,
G2 (fp32-relative, paired-noise slack >= 0.005) at the stated T, G1 (bit-exact post-processing of the GPU candidates) and
G3 (fp32-relative Jaccard, paired-noise slack >= 0.005; every disagreement passes the invariants)."""
import numpy as np
import pytest

from oracle import extraction as OX
from oracle import lattice as OL
from oracle import postprocess as OP

pytestmark = pytest.mark.gpu

TCP, SIMT = 4, 1


def _ctx(maple, inst, kernel):
    ctx = maple.Context(inst.A, inst.l, inst.u, device=0)
    ctx.set_descent_kernel(kernel)
    return ctx


def _pass_frac(Z, Zref, tol=1e-4):
    rel = np.abs(Z.astype(np.float64) - Zref) / np.maximum(1.0, np.abs(Zref))
    return float(np.mean(np.all(rel <= tol, axis=1)))


def _set(rows):
    return {tuple(int(v) for v in r) for r in np.asarray(rows).tolist()}


def _jac(a, b):
    return 1.0 if not (a | b) else len(a & b) / len(a | b)


@pytest.fixture(scope="module")
def c3():
    from synth import c3 as mk
    return mk()


def test_tcp_is_auto_choice_for_c3(gpu_lib, c3):
    ctx = gpu_lib.Context(c3.A, c3.l, c3.u)
    assert ctx.descent_kernel == "tcp"


@pytest.mark.parametrize("T", [1, 5])
def test_tcp_starts_and_small_T_iterates(gpu_lib, c3, T):
    """Every start within 1e-4 of the fp64 oracle after T in {1, 5} (ragged tail: 300 starts = 2 pairs + 44);
    the starts themselves equal the oracle's fp64 z0 = B+ g0 at 1e-12."""
    ctx = _ctx(gpu_lib, c3, TCP)
    N = 300
    Z, Z0 = ctx.debug_descent(N, 0, N, T, c3.lr, 11)
    _, z0 = OX.sample_starts(c3.l, c3.u, OL.pinv(ctx.B), 11, np.arange(N))
    np.testing.assert_allclose(Z0, z0, rtol=1e-12, atol=1e-12)
    Zo = OX.descend(z0, ctx.B, T, c3.lr)
    assert _pass_frac(Z, Zo) >= 0.999


def test_tcp_matches_simt_short(gpu_lib, c3):
    """Two fp32 implementations of the same algorithm (different summation orders) agree on almost every start
    after 10 steps; a rare start may already have been separated by a sign decided at rounding level."""
    a, b = _ctx(gpu_lib, c3, SIMT), _ctx(gpu_lib, c3, TCP)
    Za, _ = a.debug_descent(512, 0, 512, 10, c3.lr, 3)
    Zb, _ = b.debug_descent(512, 0, 512, 10, c3.lr, 3)
    assert _pass_frac(Zb, Za.astype(np.float64)) >= 0.99


@pytest.mark.parametrize("T", [50, 200])
def test_tcp_iterates_gate_g2(gpu_lib, c3, T):
    """pass(GPU vs fp64) >= pass(fp32 oracle vs fp64) - slack on 1024 starts, slack = max(0.005, two standard errors
    of the paired difference) (tests/test_gpu_fullsize.py:_g2)."""
    ctx = _ctx(gpu_lib, c3, TCP)
    N = 1024
    Z, _ = ctx.debug_descent(N, 0, N, T, c3.lr, c3.seed)
    _, z0 = OX.sample_starts(c3.l, c3.u, OL.pinv(ctx.B), c3.seed, np.arange(N))
    Z64 = OX.descend(z0, ctx.B, T, c3.lr)
    Z32 = OX.descend(z0.astype(np.float32), ctx.B, T, c3.lr, dtype=np.float32)
    ok_g = np.all(np.abs(Z.astype(np.float64) - Z64) / np.maximum(1, np.abs(Z64)) <= 1e-4, axis=1)
    ok_f = np.all(np.abs(Z32.astype(np.float64) - Z64) / np.maximum(1, np.abs(Z64)) <= 1e-4, axis=1)
    slack = max(0.005, 2.0 * np.sqrt(np.sum(ok_g != ok_f)) / N)
    print(f"C3 T={T} tcp: gpu pass {ok_g.mean():.4f}, fp32-oracle pass {ok_f.mean():.4f}, slack {slack:.4f}")
    assert ok_g.mean() >= ok_f.mean() - slack


def test_tcp_postprocess_bit_exact_g1(gpu_lib, c3):
    """G1: the oracle's check -> dedupe -> ⊑ filter -> lex sort of the GPU candidate multiset equals the output."""
    ctx = _ctx(gpu_lib, c3, TCP)
    ctx.set_debug(True)
    ds = ctx.extract(300, c3.steps, c3.lr, c3.seed)
    cand = ctx.candidates()
    assert cand.shape[0] > 0
    assert np.all(OP.check_rows(c3.A, c3.l, c3.u, cand))
    ref, nbad = OP.postprocess(c3.A, c3.l, c3.u, cand)
    assert nbad == 0
    assert [tuple(r) for r in ds.rows().tolist()] == ref


def test_tcp_sets_gate_g3(gpu_lib, c3):
    """G3 fp32-relative: Jaccard(GPU, fp64 oracle) >= Jaccard(fp32 oracle, fp64 oracle) - slack on the same
    256 starts; every row in a symmetric difference is an exact in-box kernel element."""
    ctx = _ctx(gpu_lib, c3, TCP)
    N = 256
    Bp = OL.pinv(ctx.B)
    g = _set(ctx.extract(N, c3.steps, c3.lr, c3.seed).rows())
    p64, _ = OX.extract_pool(ctx.B, Bp, c3.l, c3.u, N, c3.steps, c3.lr, c3.seed)
    p32, _ = OX.extract_pool(ctx.B, Bp, c3.l, c3.u, N, c3.steps, c3.lr, c3.seed, dtype=np.float32)
    m64, m32 = OP.minimal_filter(p64), OP.minimal_filter(p32)
    jg, j32 = _jac(g, m64), _jac(m32, m64)
    # the paired-noise slack of tests/test_gpu_fullsize.py:_g3
    slack = max(0.005, 2.0 * np.sqrt(len(g ^ m32)) / max(1, len(g | m32 | m64)))
    print(f"C3 G3 tcp: |gpu|={len(g)} |fp64|={len(m64)} jaccard {jg:.4f}, fp32-oracle {j32:.4f}, slack {slack:.4f}")
    assert jg >= j32 - slack
    diff = np.array(sorted(g ^ m64), dtype=np.int64).reshape(-1, c3.n)
    if diff.size:
        assert np.all(OP.check_rows(c3.A, c3.l, c3.u, diff))


def test_tcp_range_overflow_falls_back_to_simt(gpu_lib, c3):
    """An iterate beyond the f16 operand range of the CTA-pair kernel (|z| > 1023, here from a huge step size) sets
    its device flag; the extraction is redone on the SIMT kernel, so the result equals a SIMT-only context's."""
    lr = 500.0
    a = _ctx(gpu_lib, c3, TCP)
    b = _ctx(gpu_lib, c3, SIMT)
    ra = a.extract(512, 20, lr, c3.seed).rows()
    rb = b.extract(512, 20, lr, c3.seed).rows()
    assert a.descent_kernel == "simt"        # the context remembers the overflow
    np.testing.assert_array_equal(ra, rb)
