"""The oracle (and, where the library exposes the operation without a GPU, the C ABI) against the golden
fixtures in tests/golden/: values printed in the paper or its derived spec, typed in by hand with their
citations (see tests/golden/README.md). None of these values comes from oracle/ or from the CUDA path."""
import json
import os
from fractions import Fraction
from math import comb

import numpy as np
import pytest

from oracle import augment as OA
from oracle import extraction as OX
from oracle import feasible as OF
from oracle import graver as OG
from oracle import lattice as OL

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _from_columns(cols):
    return np.array(cols, dtype=np.int64).T


def _cases(name, key):
    return [pytest.param(c, id=c["cite"].split(" ")[0]) for c in _load(name)[key]]


def test_paper_hyperparameters_are_the_oracle_defaults():
    hp = _load("paper_hyperparameters.json")
    import inspect
    ex = inspect.signature(OX.loss).parameters
    fe = inspect.signature(OF.loss).parameters
    assert ex["lam1"].default == hp["lambda1"] and ex["lam2"].default == hp["lambda2"]
    assert fe["lam3"].default == hp["lambda3"]
    d = inspect.signature(OX.descend).parameters
    assert d["lam1"].default == hp["lambda1"] and d["lam2"].default == hp["lambda2"]


@pytest.mark.parametrize("case", _cases("spec_lattice.json", "hnf"))
def test_hnf(case):
    H, C = OL.hnf(case["A"])
    assert H == case["H"]
    if "C" in case:
        assert C == case["C"]
    A = np.array(case["A"], dtype=object)
    AC = A.dot(np.array(C, dtype=object))
    m = A.shape[0]
    assert AC[:, :m].tolist() == case["H"] and all(v == 0 for v in AC[:, m:].ravel())
    assert abs(OL.bareiss_det(C)) == 1


@pytest.mark.parametrize("case", _cases("spec_lattice.json", "kernel_basis"))
def test_kernel_basis(case):
    if "error" in case:
        with pytest.raises(Exception):
            OL.kernel_basis(case["A"])
        return
    B = np.array(OL.kernel_basis(case["A"]), dtype=np.int64)
    col = B[:, 0].tolist()
    assert col in (case["column_up_to_sign"], [-v for v in case["column_up_to_sign"]])


@pytest.mark.parametrize("case", _cases("spec_lattice.json", "gram_schmidt"))
def test_gram_schmidt(case):
    bstar, mu = OL.gram_schmidt(_from_columns(case["B_columns"]).tolist())
    assert [[Fraction(v) for v in c] for c in case["bstar_columns"]] == [list(c) for c in bstar]
    assert mu[1][0] == case["mu21"]


@pytest.mark.parametrize("case", _cases("spec_lattice.json", "lll_reduce"))
def test_lll_reduce(case):
    out = np.array(OL.lll_reduce(_from_columns(case["B_columns"]).tolist()), dtype=np.int64)
    assert out.T.tolist() == case["out_columns"]


@pytest.mark.parametrize("case", _cases("spec_lattice.json", "is_lll_reduced"))
def test_is_lll_reduced(case):
    assert OL.is_lll_reduced(_from_columns(case["B_columns"]).tolist()) == case["reduced"]


@pytest.mark.parametrize("case", _cases("spec_lattice.json", "to_coords"))
def test_to_coords(case):
    B = _from_columns(case["B_columns"])
    z = np.asarray(OL.pinv(B.tolist()), dtype=np.float64) @ np.array(case["g"], dtype=np.float64)
    np.testing.assert_allclose(z, case["z"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("case", _cases("spec_graver.json", "conforms"))
def test_conforms(case):
    assert OG.conforms(case["x"], case["y"]) == case["result"]


@pytest.mark.parametrize("case", _cases("spec_graver.json", "enumerate_kernel_in_box"))
def test_enumerate_kernel(case):
    got = {tuple(int(v) for v in g) for g in OG.enumerate_kernel_in_box(case["A"], case["lo"], case["hi"])}
    assert got == {tuple(g) for g in case["set"]}


@pytest.mark.parametrize("case", _cases("spec_graver.json", "graver_in_box"))
def test_graver_in_box(case):
    got = {tuple(int(v) for v in g) for g in OG.graver_in_box(case["A"], case["lo"], case["hi"])}
    assert got == {tuple(g) for g in case["set"]}


@pytest.mark.parametrize("case", _cases("spec_losses.json", "eq3_loss"))
def test_eq3_loss(case):
    B = _from_columns(case["B_columns"])
    v = OX.loss(np.array(case["z"]), B, case["lambda1"], case["lambda2"])
    assert abs(v - case["value"]) <= 1e-12


@pytest.mark.parametrize("case", _cases("spec_losses.json", "eq4_loss"))
def test_eq4_loss(case):
    v = OF.loss(np.array(case["x"]), np.array(case["A"]), np.array(case["b"]), case["lambda3"])
    assert abs(v - case["value"]) <= 1e-12


@pytest.mark.parametrize("case", _cases("spec_augment.json", "max_step_length"))
def test_max_step_length(case):
    assert OA.max_step_length(case["x"], case["g"], case["l"], case["u"]) == case["lambda"]


@pytest.mark.parametrize("case", _cases("spec_augment.json", "best_step"))
def test_best_step(case):
    f = OA.Objective(case["Q"], case["c"])
    lam, key = OA.best_step(f, case["x"], case["g"], case["l"], case["u"])
    assert lam == case["lambda"]
    assert f.value(np.array(case["x"]) + lam * np.array(case["g"])) == case["value"]


@pytest.mark.parametrize("case", _cases("spec_augment.json", "graver_best_augment"))
def test_graver_best_augment(case):
    f = OA.Objective(case["Q"], case["c"], case["c0"])
    x, it = OA.graver_best_augment(f, case["A"], case["b"], case["l"], case["u"], case["x0"], case["S"])
    assert np.asarray(x).tolist() == case["x"] and it == case["iterations"]
    assert f.value(x) == case["f"]


@pytest.mark.parametrize("case", _cases("spec_augment.json", "feasible_set"))
def test_feasible_set(case):
    pts, _ = OF.feasible_set(case["A"], case["b"], case["l"], case["u"], 64, 300, 0.05, seed=1)
    assert {tuple(p) for p in pts} <= {tuple(p) for p in case["subset_of"]}
    if case["subset_of"]:
        assert len(pts) >= 1


def test_closed_form_all_ones_row():
    cf = _load("closed_forms.json")["cases"][0]
    lo = [li - ui for li, ui in zip(cf["l"], cf["u"])]
    hi = [ui - li for li, ui in zip(cf["l"], cf["u"])]
    got = {OG.canonical(g) for g in OG.graver_in_box(cf["A"], lo, hi)}
    assert len(got) == cf["count_canonical"]
    assert got == {tuple(g) for g in cf["set_canonical"]}


def test_closed_form_semi_assignment_count():
    cf = _load("closed_forms.json")["cases"][1]
    assert cf["groups"] * comb(cf["group_size"], 2) == cf["count_canonical"]


# ---- the C ABI's host-only lattice step against the same fixtures (no GPU needed) ----

@pytest.mark.parametrize("case", [c for c in _load("spec_lattice.json")["kernel_basis"] if "error" not in c],
                         ids=lambda c: c["cite"].split(" ")[0])
def test_library_kernel_basis_fixture(case):
    from paper_2412_13576_b200 import maple
    B, Bp = maple.maple_kernel_basis(np.array(case["A"], dtype=np.int32))
    col = B[:, 0].tolist()
    assert col in (case["column_up_to_sign"], [-v for v in case["column_up_to_sign"]])
    np.testing.assert_allclose(Bp @ B, np.eye(B.shape[1]), atol=1e-12)
