"""CTA-pair (cta_group::2) tcgen05 + TMA conventions the large-shape descent kernel relies on
(k_descent_tcp.cu): exact small-integer products, B loaded by 3-D TMA boxes and split by N across the pair,
D rows of CTA r at lane m + 64 (n >= N/2), column n mod N/2."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _expected_raw(D, ncols):
    """D (128 x N) -> per-CTA (lanes 128 x N/2 columns) under the documented 2-SM M=128 layout."""
    N = D.shape[1]
    h = N // 2
    raw = np.full((2, 128, ncols), np.nan)
    for r in range(2):
        for m in range(64):
            raw[r, m, :h] = D[64 * r + m, :h]
            raw[r, 64 + m, :h] = D[64 * r + m, h:]
    return raw


def test_pair_selftest_layout_exact(gpu_lib):
    rng = np.random.default_rng(5)
    Ah = rng.integers(-4, 5, size=(128, 32)).astype(np.float16)
    Bh = rng.integers(-4, 5, size=(160, 32)).astype(np.float16)
    A8 = rng.integers(-6, 7, size=(128, 64)).astype(np.int8)
    B8 = rng.integers(-6, 7, size=(128, 64)).astype(np.int8)
    raw1, raw2 = gpu_lib.maple_selftest_pair(Ah, Bh, A8, B8)
    D1 = Ah.astype(np.float64) @ Bh.astype(np.float64).T
    D2 = A8.astype(np.int64) @ B8.astype(np.int64).T
    e1 = _expected_raw(D1, 80)
    e2 = _expected_raw(D2, 64)
    if not np.array_equal(raw1, e1):
        # diagnostics: where do D1's columns land?
        for r in range(2):
            for lane in (0, 1, 63, 64, 65, 127):
                row = raw1[r, lane]
                hits = [(i, int(np.argmax(np.all(D1 == row[None, :], axis=1))))
                        for i in range(1)] if False else None
                print("cta", r, "lane", lane, row[:6])
        print("D1 rows 0,64:", D1[0, :6], D1[64, :6], "D1[0,80:86]", D1[0, 80:86])
    np.testing.assert_array_equal(raw1, e1)
    np.testing.assert_array_equal(raw2, e2)
