"""Pins for oracle/formats.py (Table 1, RNE storage rounding).  CPU only."""
import bisect
from fractions import Fraction

import numpy as np
import pytest

from oracle import formats as F


def test_unit_roundoffs_match_table1():
    # PAPER.md:42-45 prints u rounded to 3 significant digits
    printed = {F.FP64: 1.11e-16, F.FP32: 5.96e-8, F.FP16: 4.88e-4, F.BF16: 3.91e-3}   # q43: see below
    for t, u in printed.items():
        assert abs(F.unit_roundoff(t) - u) / u < 5e-3


def test_xmax_match_table1():
    # Table 1 prints 1.80e308 (rounded up past the largest double); compare its 1.79e308 floor
    printed = {F.FP64: 1.79e308, F.FP32: 3.40e38, F.FP16: 6.55e4, F.BF16: 3.39e38}
    for t, v in printed.items():
        assert abs(F.x_max(t) - v) / v < 5e-3


def test_worked_examples():
    # SPEC.md:277-278 (derived from Table 1): bf16(0.1) = 0.10009765625, fp16(70000) = inf
    assert F.round_rne(np.array([0.1]), F.BF16)[0] == 0.10009765625
    assert np.isinf(F.round_rne(np.array([70000.0]), F.FP16)[0])
    # fp16 overflow threshold: x_max + half ulp (32) rounds to even = 2^16 -> inf
    assert F.round_rne(np.array([65519.99]), F.FP16)[0] == 65504.0
    assert np.isinf(F.round_rne(np.array([65520.0]), F.FP16)[0])
    assert F.round_rne(np.array([1.0]), F.FP32)[0] == 1.0


def _all_values(tag):
    """Every finite non-negative value of a 16-bit format, sorted, with its bit pattern."""
    bits = np.arange(0, 1 << 15, dtype=np.uint16)
    if tag == F.FP16:
        v = bits.view(np.float16).astype(np.float64)
    else:
        v = (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    ok = np.isfinite(v)
    order = np.argsort(v[ok], kind="stable")
    return v[ok][order], bits[ok][order]


@pytest.mark.parametrize("tag", [F.FP16, F.BF16])
def test_rne_matches_bruteforce_enumeration(tag):
    """Brute force: nearest of ALL representable values, ties to even last bit (exact
    rational comparison); inputs constructed on and around every rounding midpoint."""
    vals, bits = _all_values(tag)
    rng = np.random.default_rng(7)
    idx = rng.integers(1, vals.size - 2, size=400)
    xs = []
    for i in idx:
        mid = (vals[i] + vals[i + 1]) / 2          # exact in float64
        xs += [mid, np.nextafter(mid, 0), np.nextafter(mid, np.inf), vals[i]]
    xs += list(rng.uniform(0, 2 * vals[-1], 200)) + list(rng.uniform(0, 1e-6, 100))
    xs = np.array(xs)
    got = F.round_rne(xs, tag)
    xmax = F.x_max(tag)
    half_ulp_top = Fraction(vals[-1]) - Fraction(vals[-2])
    for x, g in zip(xs, got):
        fx = Fraction(float(x))
        if fx >= Fraction(xmax) + half_ulp_top / 2:
            assert np.isinf(g) or (fx == Fraction(xmax) + half_ulp_top / 2 and np.isinf(g))
            continue
        k = bisect.bisect_left(vals.tolist(), float(x))
        cands = [j for j in (k - 1, k) if 0 <= j < vals.size]
        best = min(cands, key=lambda j: (abs(Fraction(vals[j]) - fx), int(bits[j]) & 1))
        assert g == vals[best], (x, g, vals[best])


@pytest.mark.parametrize("tag,dt", [(F.FP16, np.float16), (F.FP32, np.float32)])
def test_rne_matches_numpy_direct_cast(tag, dt):
    """numpy casts float64->float16/float32 directly with round-half-even (library routine)."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal(20000) * np.exp2(rng.integers(-30, 20, 20000))
    vals = x.astype(dt).astype(np.float64)
    mids = (vals[:-1] + np.nextafter(vals[:-1].astype(dt), np.inf, dtype=dt).astype(np.float64)) / 2
    xs = np.concatenate([x, mids, np.nextafter(mids, 0), np.nextafter(mids, np.inf)])
    xs = xs[np.isfinite(xs)]
    with np.errstate(over="ignore"):
        ref = xs.astype(dt).astype(np.float64)
    np.testing.assert_array_equal(F.round_rne(xs, tag), ref)


def test_bf16_single_rounding_differs_from_double_rounding():
    """G16: fp64 -> fp32 -> bf16 double-rounds; the oracle must not."""
    x = np.array([1.0 + 2.0 ** -8 + 2.0 ** -30])    # just above a bf16 midpoint; fp32 rounds onto it
    direct = F.round_rne(x, F.BF16)[0]
    twice = F.round_rne(F.round_rne(x, F.FP32), F.BF16)[0]
    assert direct == 1.0 + 2.0 ** -7 and twice == 1.0


def test_storage_bits_roundtrip():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(1000)
    for t in (F.FP64, F.FP32, F.FP16, F.BF16):
        b = F.to_storage_bits(x, t)
        back = F.from_storage_bytes(b.tobytes(), t)
        np.testing.assert_array_equal(back, F.round_rne(x, t))


# ------------------------------------------------------------- q43 (Table 1, 8-bit; NEXT-3)
def _q43_values():
    """Every finite non-negative q43 value from Table 1's definition (1-4-3, e_min -6, e_max 7,
    exponent field 15 reserved): (1 + m/8) 2^(e-7) for e = 1..14, (m/8) 2^-6 for e = 0."""
    vals, bits = [], []
    for e in range(15):
        for m in range(8):
            vals.append(Fraction(m, 8) * Fraction(1, 64) if e == 0 else (1 + Fraction(m, 8)) * Fraction(2) ** (e - 7))
            bits.append(e << 3 | m)
    order = sorted(range(len(vals)), key=lambda i: vals[i])
    return [vals[i] for i in order], [bits[i] for i in order]


def test_q43_table1_row():
    assert F.x_max(F.Q43) == 240.0                                   # Table 1: 2.4e2
    assert F.PARAMS[F.Q43] == (3, -6, 7) and 2.0 ** -6 == 0.015625    # x_min 1.56e-2, e_min -6, e_max 7
    # Table 1 prints u = 2.5e-1 for q43; reading G12: u = 2^-(m+1) = 2^-4
    assert F.unit_roundoff(F.Q43) == 0.0625
    assert F.BYTES[F.Q43] == 1 and F.TAG_BIT[F.Q43] == 16


def test_q43_worked_examples():
    r = F.round_rne(np.array([0.1, 247.99, 248.0, 2.0 ** -10, 3 * 2.0 ** -10, 1.0625, 1.1875, -0.3]), F.Q43)
    # 0.1 = 1.6 * 2^-4 -> 1.625 * 2^-4; 248 is the midpoint 240|256 -> even (256) = overflow;
    # 2^-10 ties between 0 and 2^-9 -> 0 (even); 3 * 2^-10 ties 2^-9|2^-8 -> 2^-8 (mantissa 2, even);
    # 1.0625 ties 1|1.125 -> 1; 1.1875 ties 1.125|1.25 -> 1.25; -0.3 = -1.2 * 2^-2 -> -1.25 * 2^-2
    np.testing.assert_array_equal(r, [0.1015625, 240.0, np.inf, 0.0, 2.0 ** -8, 1.0, 1.25, -0.3125])


def test_q43_rne_matches_bruteforce_enumeration():
    vals, bits = _q43_values()
    rng = np.random.default_rng(11)
    xs = []
    for i in range(len(vals) - 1):
        mid = (vals[i] + vals[i + 1]) / 2
        xs += [float(mid), float(np.nextafter(float(mid), 0)), float(np.nextafter(float(mid), np.inf)), float(vals[i])]
    xs += list(rng.uniform(0, 260, 300)) + list(rng.uniform(0, 0.05, 300))
    got = F.round_rne(np.array(xs), F.Q43)
    top = vals[-1] + (vals[-1] - vals[-2]) / 2          # 248: at and above -> inf (ties to even 256)
    for x, g in zip(xs, got):
        fx = Fraction(x)
        if fx >= top:
            assert np.isinf(g), x
            continue
        best = min(range(len(vals)), key=lambda j: (abs(vals[j] - fx), bits[j] & 1))
        assert Fraction(float(g)) == vals[best], (x, g, vals[best])


def test_q43_storage_bits_roundtrip_and_e4m3_decode():
    """The q43 byte layout (sign | 4-bit exponent | 3-bit mantissa, bias 7) round-trips, and every
    finite q43 byte decodes to the same value under the OCP FP8 E4M3 rules (torch.float8_e4m3fn,
    a library decoder) — what lets the device use E4M3 conversions."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal(3000) * np.exp2(rng.integers(-12, 8, 3000))
    r = F.round_rne(x, F.Q43)
    x = x[np.isfinite(r)]
    b = F.to_storage_bits(x, F.Q43)
    np.testing.assert_array_equal(F.from_storage_bytes(b.tobytes(), F.Q43), F.round_rne(x, F.Q43))
    torch = pytest.importorskip("torch")
    allb = np.array([s << 7 | e << 3 | m for s in (0, 1) for e in range(15) for m in range(8)], np.uint8)
    ours = F.from_storage_bytes(allb.tobytes(), F.Q43)
    ocp = torch.from_numpy(allb.copy()).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    np.testing.assert_array_equal(ours, ocp)
    vals, _ = _q43_values()
    np.testing.assert_array_equal(np.sort(np.unique(np.abs(ours))), np.array([float(v) for v in vals]))


# ------------------------------------------------------------- accessor formats (NEXT-3)
def _rne_fraction(x, m, emin):
    """Nearest value (1 + k / 2^m) 2^e (normal) or (k / 2^m) 2^emin (subnormal) to the exact rational
    x, ties to the even k — the definition, in exact arithmetic (no overflow in the test range)."""
    fx = Fraction(float(x))
    s = -1 if fx < 0 else 1
    a = abs(fx)
    if a == 0:
        return 0.0
    e = max(emin, a.numerator.bit_length() - a.denominator.bit_length())
    while Fraction(2) ** e > a and e > emin:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    q = Fraction(2) ** (e - m)                    # spacing at a
    k = a / q
    lo = k.numerator // k.denominator
    rem = k - lo
    kk = lo + 1 if (rem > Fraction(1, 2) or (rem == Fraction(1, 2) and lo % 2 == 1)) else lo
    return float(s * kk * q)


@pytest.mark.parametrize("tag", [F.BF24, F.FP48])
def test_accessor_formats_rne_by_definition(tag):
    m, emin, _ = F.PARAMS[tag]
    rng = np.random.default_rng(tag)
    x = rng.standard_normal(400) * np.exp2(rng.integers(-40, 40, 400))
    r = F.round_rne(x, tag)
    q = np.ldexp(1.0, np.maximum(np.frexp(np.abs(r))[1] - 1, emin) - m)
    mids = r + np.sign(r) * q / 2                        # exact midpoints
    xs = np.concatenate([x, mids, np.nextafter(mids, 0), np.nextafter(mids, np.inf)])
    if tag == F.BF24:                                     # fp32's subnormal range, 15-bit mantissa
        xs = np.concatenate([xs, rng.uniform(0, 2.0 ** -126, 200), [2.0 ** -141, 3 * 2.0 ** -142]])
    got = F.round_rne(xs, tag)
    for a, g in zip(xs, got):
        assert g == _rne_fraction(a, m, emin), (tag, a, g)


def test_accessor_formats_worked_examples_and_decode():
    # bf24(0.1): 0.1 = 1.6 2^-4, 0.6 * 2^15 = 19660.8 -> 19661: (2^15 + 19661) / 2^19
    assert F.round_rne(np.array([0.1]), F.BF24)[0] == 52429 / 2 ** 19 == 0.1000003814697265625
    # fp48(1/3): 1/3 = (4/3) 2^-2, (1/3) 2^36 = 22906492245.33 -> 22906492245
    assert F.round_rne(np.array([1 / 3]), F.FP48)[0] == (2 ** 36 + 22906492245) / 2 ** 38
    # overflow: bf24 x_max = (2 - 2^-15) 2^127 = 0x1.fffep127; the midpoint (2 - 2^-16) 2^127 to
    # 2^128 rounds to even = inf
    assert F.x_max(F.BF24) == float.fromhex("0x1.fffep127")
    assert F.round_rne(np.array([float.fromhex("0x1.fffe8p127")]), F.BF24)[0] == F.x_max(F.BF24)
    assert np.isinf(F.round_rne(np.array([float.fromhex("0x1.ffffp127")]), F.BF24)[0])
    assert F.unit_roundoff(F.BF24) == 2.0 ** -16 and F.unit_roundoff(F.FP48) == 2.0 ** -37
    # the stored bytes are the top bytes of the IEEE pattern: decode = zero-extend and reinterpret
    rng = np.random.default_rng(3)
    x = rng.standard_normal(500)
    for tag, pad, dt in ((F.BF24, 1, "<f4"), (F.FP48, 2, "<f8")):
        b = F.to_storage_bits(x, tag).reshape(x.size, -1)
        ref = np.array([np.frombuffer(bytes(pad) + bytes(row), dt)[0] for row in b], dtype=np.float64)
        np.testing.assert_array_equal(F.from_storage_bytes(b.tobytes(), tag), ref)
        np.testing.assert_array_equal(ref, F.round_rne(x, tag))
    # Eq. 4.4's candidate order gains the two formats between the Table 1 ones
    assert F.BY_U == (F.Q43, F.BF16, F.FP16, F.BF24, F.FP32, F.FP48, F.FP64)
