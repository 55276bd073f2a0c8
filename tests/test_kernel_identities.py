"""Host checks of the arithmetic identities the CTA-pair descent kernel relies on (k_descent_tcp.cu, final
round-2 steps 3 and 5). Each identity replaces one instruction sequence by another that must give the same bits;
these tests evaluate both sides exactly (float64 holds every intermediate here) and round once, as the FMA does."""
import struct

import numpy as np


def _f32(x):
    return np.float32(x)


def test_lambda1_term_identity():
    """ceil z + floor z - 2z == sign(z - r) - 2 (z - r) for a nearest integer r (ties either way), as real numbers,
    so both single-rounding evaluations (fmaf(-2, z, cf) and fmaf(-2, dd, sd)) give the same float32."""
    rng = np.random.default_rng(7)
    z = np.concatenate([
        rng.standard_normal(20000) * 3,
        rng.uniform(-2 ** 21, 2 ** 21, 5000),
        np.arange(-40, 41) * 0.5,                      # integers and exact halves (ties)
        [0.0, -0.0, 2 ** -24, -2 ** -24, 1 - 2 ** -24, -(1 - 2 ** -24)],
    ]).astype(np.float32)
    for zz in z:
        zd = float(zz)
        cf = np.ceil(zd) + np.floor(zd)
        lhs = _f32(cf - 2.0 * zd)                       # exact in float64, rounded once
        r = float(np.float32(np.float32(zz + np.float32(12582912.0)) - np.float32(12582912.0)))   # magic rint
        assert abs(zd - r) <= 0.5
        dd = zd - r
        assert float(np.float32(dd)) == dd               # z - r is exact in float32
        sd = float(np.sign(dd))
        rhs = _f32(sd - 2.0 * dd)
        assert lhs == rhs or (lhs == 0 and rhs == 0), (zz, lhs, rhs)


def test_int_to_float_bias():
    """int32 M -> float32 as bits(M + 0x4B400000) - 1.5 * 2^23, exact for |M| < 2^22."""
    xs = np.concatenate([np.arange(-70000, 70000, 7), [-(2 ** 22) + 1, 2 ** 22 - 1, 0, 1, -1]]).astype(np.int64)
    bits = (xs + 0x4B400000).astype(np.uint32)
    f = bits.view(np.float32) - np.float32(12582912.0)
    assert np.array_equal(f, xs.astype(np.float32))


def _prmt(x, y, sel):
    b = list(int(x).to_bytes(4, "little")) + list(int(y).to_bytes(4, "little"))
    out = 0
    for i in range(4):
        nib = (sel >> (4 * i)) & 0xF
        v = b[nib & 7]
        if nib & 8:                                      # PTX prmt default mode: replicate the byte's sign bit
            v = 0xFF if v & 0x80 else 0
        out |= v << (8 * i)
    return out


def _bits(v):
    return struct.unpack("<I", struct.pack("<f", v))[0]


def test_sign_bytes_from_top_bytes():
    """Four sign bytes per word from the top bytes of four fp32 G values (a nonzero G is a multiple of 2^-24, so its
    exponent field is >= 103 and the top 7 exponent bits are nonzero): equals sign(G) as int8 with sign(+-0) = 0."""
    rng = np.random.default_rng(3)
    vals = list((rng.integers(-4000, 4000, 4000) * 2.0 ** -24).astype(np.float32))
    vals += list((rng.standard_normal(4000) * 1e4).astype(np.float32))
    vals += [0.0, -0.0, 2 ** -24, -2 ** -24, 38100.0, -38100.0, float("inf"), -float("inf")]
    vals = vals[: len(vals) // 4 * 4]

    def ref(v):
        return 0 if v == 0 else (0xFF if v < 0 else 0x01)

    for i in range(0, len(vals), 4):
        g = [_bits(float(v)) for v in vals[i:i + 4]]
        t = _prmt(_prmt(g[0], g[1], 0x0073), _prmt(g[2], g[3], 0x0073), 0x5410)
        nz = _prmt(((t & 0x7F7F7F7F) + 0x7F7F7F7F) & 0xFFFFFFFF, 0, 0xBA98)
        ng = _prmt(t, 0, 0xBA98)
        w = nz & (ng | 0x01010101)
        assert w == sum(ref(float(vals[i + e])) << (8 * e) for e in range(4))
