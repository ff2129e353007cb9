"""Floating-point storage formats of Table 1 and round-to-nearest-even (oracle).

PAPER.md:37-50 (Table 1) lists fp64, fp32, fp16, bf16 and the 8-bit q43 (1-4-3, e_min -6,
e_max 7, x_max 240).  BASELINE's precision set is {fp64, fp32, fp16, bf16}; q43 is the NEXT-3
opt-in (precision_set bit 16).
Reading G12: the unit roundoffs are the exact powers of two
u = 2^-(m+1): 2^-53, 2^-24, 2^-11, 2^-8, 2^-4 (Table 1 prints them rounded; its q43 entry
2.5e-1 is garbled — 2^-(3+1) = 6.25e-2).  q43 is the IEEE-style 8-bit format of Table 1:
exponent field 15 is inf/NaN, so x_max = (2 - 2^-3) 2^7 = 240 and the smallest subnormal is
2^-9; its encodings of |x| <= 240 coincide with the OCP FP8 E4M3 ones (which reuse exponent
15 for 256..448), so the device decodes them with the E4M3 rules.
Reading G16: storage rounding is a SINGLE round-to-nearest-even from float64 directly
to the target format, subnormals kept, overflow -> +-inf (the range guard in hmatrix.py
then promotes the block, so no inf is ever stored).

``round_rne`` below is written from the definition ("the representable value nearest to
x, ties to the one with an even last significand bit") and does not use any library
conversion; tests pin it against numpy's direct float64->float16/float32 casts and
against exact rational rounding on constructed near-midpoint inputs.
"""
from __future__ import annotations

import numpy as np

FP64, FP32, FP16, BF16, Q43, BF24, FP48 = 0, 1, 2, 3, 4, 5, 6   # tag ids (as in include/hh.h)
TAGS = (FP64, FP32, FP16, BF16, Q43, BF24, FP48)
TAG_NAMES = {FP64: "fp64", FP32: "fp32", FP16: "fp16", BF16: "bf16", Q43: "q43", BF24: "bf24", FP48: "fp48"}
TAG_BIT = {FP64: 1, FP32: 2, FP16: 4, BF16: 8, Q43: 16, BF24: 32, FP48: 64}  # precision_set bitmask
ALL_FORMATS = 127
BYTES = {FP64: 8, FP32: 4, FP16: 2, BF16: 2, Q43: 1, BF24: 3, FP48: 6}
BITS = {t: 8 * b for t, b in BYTES.items()}

# (mantissa bits m, e_min, e_max) — Table 1 columns (1-e-m), e_min, e_max
PARAMS = {
    FP64: (52, -1022, 1023),
    FP32: (23, -126, 127),
    FP16: (10, -14, 15),
    BF16: (7, -126, 127),
    Q43: (3, -6, 7),
    # PAPER.md:933 (remark after Eq. 4.4): "by leveraging memory accessor mechanisms, one can
    # exploit a continuum of precision formats for storing data ... with exactly the right number
    # of bits".  Reading G28: at byte granularity, between the Table 1 formats — bf24 keeps fp32's
    # exponent range with a 15-bit mantissa (3 bytes), fp48 fp64's range with a 36-bit mantissa
    # (6 bytes): the top bytes of the wider IEEE pattern.
    BF24: (15, -126, 127),
    FP48: (36, -1022, 1023),
}
# formats in decreasing unit roundoff (Eq. 4.4 picks the largest admissible u)
BY_U = tuple(sorted(TAGS, key=lambda t: PARAMS[t][0]))


def unit_roundoff(tag: int) -> float:
    """u = 2^-(m+1) (Table 1; exact reading G12)."""
    m = PARAMS[tag][0]
    return float(np.ldexp(1.0, -(m + 1)))


def x_max(tag: int) -> float:
    """Largest finite value (2 - 2^-m) * 2^emax (Table 1 column x_max)."""
    m, _, emax = PARAMS[tag]
    return float(np.ldexp(2.0 - np.ldexp(1.0, -m), emax))


def round_rne(x, tag: int) -> np.ndarray:
    """Round float64 array ``x`` to the nearest value of format ``tag`` (ties to even).

    Returned as float64 (every value of the four formats is exactly representable in
    float64).  Definition-based: with E = floor(log2|x|), the spacing of representable
    numbers around |x| is q = 2^(max(E, e_min) - m); the nearest representable value is
    rint(|x|/q) * q, where rint rounds half to even (an even integer significand is an
    even last mantissa bit, also across the binade boundary and in the subnormal range).
    Values whose rounded magnitude exceeds x_max overflow to +-inf.
    """
    x = np.asarray(x, dtype=np.float64)
    if tag == FP64:
        return x.copy()
    m, emin, _ = PARAMS[tag]
    a = np.abs(x)
    out = np.zeros_like(a)
    nz = (a != 0) & np.isfinite(a)
    _, e = np.frexp(a[nz])            # a = f * 2^e, f in [0.5, 1) -> E = e - 1
    E = e.astype(np.int64) - 1
    qexp = np.maximum(E, emin) - m
    M = np.rint(np.ldexp(a[nz], -qexp))   # exact scaling by a power of two; rint = half-even
    with np.errstate(over="ignore"):
        out[nz] = np.ldexp(M, qexp)
    out[~np.isfinite(a)] = a[~np.isfinite(a)]
    out[out > x_max(tag)] = np.inf
    return np.copysign(out, x)


def to_storage_bits(x64, tag: int) -> np.ndarray:
    """Bit patterns of ``round_rne(x, tag)`` as stored in an arena (little-endian words).

    fp64/fp32/fp16 patterns are produced by numpy casts of the already-rounded (hence
    exactly representable) values; bf16 = the upper 16 bits of the exact float32 value.
    """
    r = round_rne(x64, tag)
    if tag == FP64:
        return r.view(np.uint64)
    if tag == FP32:
        return r.astype(np.float32).view(np.uint32)
    if tag == FP16:
        return r.astype(np.float16).view(np.uint16)
    if tag == BF16:
        f32 = r.astype(np.float32).view(np.uint32)
        return (f32 >> np.uint32(16)).astype(np.uint16)
    if tag == BF24:   # the top 3 bytes of the (exact) fp32 pattern, little-endian
        f32 = r.astype(np.float32).view(np.uint32) >> np.uint32(8)
        return np.stack([(f32 >> np.uint32(8 * k)) & np.uint32(0xFF) for k in range(3)], axis=-1).astype(np.uint8)
    if tag == FP48:   # the top 6 bytes of the fp64 pattern, little-endian
        f64 = r.view(np.uint64) >> np.uint64(16)
        return np.stack([(f64 >> np.uint64(8 * k)) & np.uint64(0xFF) for k in range(6)], axis=-1).astype(np.uint8)
    # q43 (1-4-3, bias 7): sign | exponent field | 3 mantissa bits, from the exact rounded value
    a = np.abs(r)
    sign = (np.signbit(r)).astype(np.uint8) << np.uint8(7)
    out = np.zeros(a.shape, np.uint8)
    inf = np.isinf(a)
    norm = (a >= 2.0 ** -6) & ~inf
    _, e = np.frexp(a[norm])                      # a = f 2^e, f in [0.5, 1)
    E = e.astype(np.int64) - 1
    mant = np.ldexp(a[norm], -E) * 8 - 8          # exact: a has at most 4 significant bits
    out[norm] = ((E + 7) << 3 | mant.astype(np.int64)).astype(np.uint8)
    sub = (a < 2.0 ** -6) & ~inf
    out[sub] = np.ldexp(a[sub], 9).astype(np.int64).astype(np.uint8)   # a = m 2^-9, m < 8
    out[inf] = 0x78
    return out | sign


def from_storage_bytes(buf: bytes | np.ndarray, tag: int) -> np.ndarray:
    """Decode raw little-endian arena bytes of format ``tag`` to exact float64 values."""
    b = np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf.view(np.uint8)
    if tag == FP64:
        return b.view("<f8").astype(np.float64)
    if tag == FP32:
        return b.view("<f4").astype(np.float64)
    if tag == FP16:
        return b.view("<f2").astype(np.float64)
    if tag == BF16:
        hi = b.view("<u2").astype(np.uint32) << np.uint32(16)
        return hi.view(np.float32).astype(np.float64)
    if tag == BF24:
        t = b.reshape(-1, 3).astype(np.uint32)
        bits = (t[:, 0] << np.uint32(8)) | (t[:, 1] << np.uint32(16)) | (t[:, 2] << np.uint32(24))
        return bits.view(np.float32).astype(np.float64)
    if tag == FP48:
        t = b.reshape(-1, 6).astype(np.uint64)
        bits = np.zeros(t.shape[0], np.uint64)
        for k in range(6):
            bits |= t[:, k] << np.uint64(8 * (k + 2))
        return bits.view(np.float64).copy()
    # q43: (-1)^s (1 + m/8) 2^(e-7) for exponent field e in 1..14, (-1)^s (m/8) 2^-6 for e = 0
    e = ((b >> 3) & 0xF).astype(np.int64)
    m = (b & 0x7).astype(np.float64)
    v = np.where(e == 0, np.ldexp(m / 8.0, -6), np.ldexp(1.0 + m / 8.0, e - 7))
    v = np.where(e == 15, np.inf, v)
    return np.where(b & 0x80, -v, v)
