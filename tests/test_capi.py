"""CPU tests of the boundary: libmaple.so loads, exports every symbol include/maple.h declares, and its
host-only lattice step (maple_kernel_basis = the host part of maple_create) is checked against the
oracle's independent exact checkers (Thm. 1 saturation, Def. 'reduced basis', pseudoinverse)."""
import re
import os

import numpy as np
import pytest

from oracle import lattice as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def maple():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2412_13576_b200 import maple as M
    M.load()
    return M


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "maple.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(maple_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_all_exported(maple):
    import ctypes
    lib = ctypes.CDLL(maple.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(maple.exported_symbols()) == syms


def test_header_constants_match_binding(maple):
    """The binding's objective kinds and statuses are the header's #defines (include/maple.h)."""
    src = open(os.path.join(ROOT, "include", "maple.h")).read()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+(MAPLE_[A-Z_]+)\s+(-?\d+)", src)}
    assert defs["MAPLE_OBJ_QUADRATIC"] == maple.OBJ_QUADRATIC
    assert defs["MAPLE_OBJ_SEPARABLE"] == maple.OBJ_SEPARABLE
    assert defs["MAPLE_OBJ_TABLE"] == maple.OBJ_TABLE
    assert defs["MAPLE_STATUS_NO_FEASIBLE"] == maple.STATUS_NO_FEASIBLE


def test_binding_fails_loudly_without_library(tmp_path):
    from paper_2412_13576_b200 import maple as M
    saved = M._lib
    M._lib = None
    try:
        with pytest.raises(ImportError):
            M.load(str(tmp_path / "missing.so"))
    finally:
        M._lib = saved


@pytest.mark.parametrize("name", ["C1", "C2a", "C2b"])
def test_library_basis_is_reduced_kernel_basis(maple, name):
    from synth import config
    inst = config(name)
    B, Bp = maple.maple_kernel_basis(inst.A)
    assert L.is_kernel_basis(inst.A, B.tolist())          # A B = 0 and L(B) = Ker_Z(A) (Thm. 1)
    assert L.is_lll_reduced(B.tolist())                   # Def. P:136-144, exact rationals
    np.testing.assert_allclose(Bp, L.pinv(B), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(25))
def test_library_basis_random(maple, seed):
    rng = np.random.default_rng(900 + seed)
    m = int(rng.integers(1, 5))
    n = int(rng.integers(m + 1, 10))
    while True:
        A = rng.integers(-6, 7, size=(m, n))
        if np.linalg.matrix_rank(A.astype(float)) == m:
            break
    try:
        B, Bp = maple.maple_kernel_basis(A)
    except maple.MapleError as e:      # entries beyond the device int8 range are reported, never wrapped
        assert e.name in ("RANGE", "OVERFLOW")
        return
    assert L.is_kernel_basis(A, B.tolist())
    assert L.is_lll_reduced(B.tolist())


def _free_columns(A):
    """A = [I_m | W] Pi (synth identity-block recipe): one unit column e_r per row r is an identity column; the
    other d columns F are the free coordinates, and x -> x_F maps Ker_Z(A) bijectively onto Z^d (x_I = -W x_F)."""
    m, n = A.shape
    ident = []
    for r in range(m):
        ident.append(next(k for k in range(n) if A[r, k] == 1 and np.count_nonzero(A[:, k]) == 1))
    return np.array([k for k in range(n) if k not in set(ident)])


def _unimodular(M):
    """|det M| = 1 for a square integer M, certified exactly: X = round(inv(M)) and M X = I in exact int64
    arithmetic (entries bounded first) give det(M) det(X) = 1 with both determinants integers."""
    X = np.rint(np.linalg.inv(M.astype(np.float64)))
    if not np.all(np.isfinite(X)) or np.abs(X).max() >= 2.0 ** 40 / M.shape[0] / max(1, np.abs(M).max()):
        return False
    P = M.astype(np.int64) @ X.astype(np.int64)
    return np.array_equal(P, np.eye(M.shape[0], dtype=np.int64))


def _reduced_fp64(B, tol=1e-9):
    """Def. 'reduced basis' in fp64 with SPEC S:83's tolerance: |mu_ij| <= 1/2 + tol and
    ||B*_j||^2 <= 2 ||B*_{j+1}||^2 (1 + tol), the GSO from a Householder QR (|R_jj| = ||B*_j||, mu = R / R_jj).
    For these integer bases (|B| <= 3, d <= 900) the QR's backward error is ~1e-13 relative, far inside tol."""
    R = np.linalg.qr(B.astype(np.float64), mode="r")
    diag = np.abs(np.diag(R))
    mu = R / np.where(diag == 0, 1, diag)[:, None]
    return bool(np.all(np.abs(np.triu(mu, 1)) <= 0.5 + tol) and np.all(diag[:-1] ** 2 <= 2 * diag[1:] ** 2 * (1 + tol)))


@pytest.mark.parametrize("name,shape", [("C3", (300, 280)), ("C5", (1000, 900))])
def test_library_basis_large_saturated_and_reduced(maple, name, shape):
    """configs[2] / configs[4] shapes: Thm. 1 exactly — A B = 0 and L(B) = Ker_Z(A), the latter as
    unimodularity of B restricted to the free coordinates (an exact integer certificate) — and LLL-reducedness
    (Def. P:136-144) in fp64 at SPEC S:83's tolerance."""
    from synth import config
    inst = config(name)
    B, Bp = maple.maple_kernel_basis(inst.A)
    assert B.shape == shape
    assert np.all(inst.A.astype(np.int64) @ B.astype(np.int64) == 0)
    F = _free_columns(inst.A)
    assert len(F) == shape[1]
    assert _unimodular(B[F, :])
    assert _reduced_fp64(B)
    np.testing.assert_allclose(Bp, L.pinv(B), rtol=1e-9, atol=1e-12)


def test_unimodular_certificate_rejects():
    """The saturation certificate is not vacuous: a basis of an index-2 sublattice fails it."""
    M = np.eye(5, dtype=np.int64)
    M[2, 2] = 2
    assert not _unimodular(M)
    assert _unimodular(np.array([[2, 1], [1, 1]]))


def test_create_errors(maple):
    with pytest.raises(maple.MapleError) as e:
        maple.maple_kernel_basis(np.eye(2, dtype=np.int32))
    assert e.value.name == "FULL_RANK"
    with pytest.raises(maple.MapleError) as e:
        maple.maple_kernel_basis(np.array([[1, 2, 3], [2, 4, 6]]))
    assert e.value.name == "RANK_DEFICIENT"
