"""Pins for oracle/matvec_wp.py — Alg. 3 in a lower working precision (NEXT-3, reading G27).
Worked examples whose rounded result is known by hand, exactness on integer data, and the
a priori rounding-error bound (Higham §3.1) on a real H_h.  CPU only."""
import numpy as np

import workloads as W
from oracle import formats as F
from oracle import hmatrix as HM
from oracle import matvec as MV
from oracle import matvec_wp as WP


def _dense(D):
    n = D.shape[0]
    return [(0, n, 0, D.shape[1], "dense", np.asarray(D, dtype=np.float64))]


def test_each_sum_is_rounded_fp16():
    # 2049 ones summed in fp16 in order: 2048 + 1 is a tie between 2048 and 2050 -> 2048 (even)
    D = np.ones((1, 2049))
    y = WP.matvec_blocks_wp(2049, np.arange(2049), [(0, 1, 0, 2049, "dense", D)], np.ones((2049, 1)), WP.WP_FP16)
    assert y[0, 0] == 2048.0
    assert MV.matvec_blocks(2049, np.arange(2049), [(0, 1, 0, 2049, "dense", D)], np.ones((2049, 1)))[0, 0] == 2049.0


def test_each_sum_is_rounded_fp32():
    # 1 + 2^-25 + 2^-25 in fp32, left to right: each addition falls below half an ulp of 1 -> 1
    D = np.ones((3, 3))
    x = np.array([[1.0], [2.0 ** -25], [2.0 ** -25]])
    y = WP.matvec_blocks_wp(3, np.arange(3), _dense(D), x, WP.WP_FP32)
    assert np.all(y[:, 0] == 1.0)


def test_operands_rounded_once():
    # x = 1 + 2^-11 + 2^-30 lies above the fp16 midpoint 1 + 2^-11 -> 1 + 2^-10 (one RNE rounding)
    x = np.array([[1.0 + 2.0 ** -11 + 2.0 ** -30]])
    assert WP.matvec_blocks_wp(1, np.arange(1), _dense(np.ones((1, 1))), x, WP.WP_FP16)[0, 0] == 1.0 + 2.0 ** -10
    # a factor entry wider than the working format is rounded too: 0.1 in fp16 = 0.0999755859375
    blk = [(0, 1, 0, 1, "lr", (np.array([[1.0]]), np.array([[0.1]])))]
    assert WP.matvec_blocks_wp(1, np.arange(1), blk, np.ones((1, 1)), WP.WP_FP16)[0, 0] == 0.0999755859375


def test_exact_on_integer_data_both_formats():
    """Small-integer factors and x keep every product and partial sum exact in fp16 and fp32,
    so the working-precision product equals the exact one: no term dropped, transposed or
    misplaced (low-rank and dense blocks, permuted points, two right-hand sides)."""
    rng = np.random.default_rng(4)
    n = 24
    perm = rng.permutation(n)
    blocks = []
    for (i0, i1, j0, j1) in ((0, 8, 8, 24), (8, 24, 0, 8), (8, 16, 16, 24), (16, 24, 8, 16)):
        p = int(rng.integers(1, 4))
        blocks.append((i0, i1, j0, j1, "lr", (rng.integers(-3, 4, (i1 - i0, p)).astype(float),
                                             rng.integers(-3, 4, (j1 - j0, p)).astype(float))))
    for (a, b) in ((0, 8), (8, 16), (16, 24)):
        blocks.append((a, b, a, b, "dense", rng.integers(-3, 4, (b - a, b - a)).astype(float)))
    x = rng.integers(-4, 5, (n, 2)).astype(float)
    ref = MV.matvec_blocks(n, perm, blocks, x)
    for wp in (WP.WP_FP32, WP.WP_FP16):
        np.testing.assert_array_equal(WP.matvec_blocks_wp(n, perm, blocks, x, wp), ref)


def _records(H):
    for b in range(len(H.part)):
        i0, i1, j0, j1 = H.rows(b)
        if b in H.factors:
            yield i0, i1, j0, j1, "lr", H.factors[b]
        elif b in H.dense:
            yield i0, i1, j0, j1, "dense", H.dense[b]


def test_within_a_priori_rounding_bound(tiny_oracle):
    """On BASELINE config 0's H_h: |y_wp - y*| <= gamma_{K + n_J} S componentwise for fp32
    (deterministic bound, any summation order), and <= gamma~(8) S for fp16 (probabilistic,
    Higham & Mary 2019), where y* is the exact product of the rounded operands; the errors are
    also of the order the model predicts (not identically zero)."""
    cfg, P, H = tiny_oracle
    x = W.make_rhs(cfg, 2)
    blocks = list(_records(H))
    for wp, u in ((WP.WP_FP32, 2.0 ** -24), (WP.WP_FP16, 2.0 ** -11)):
        y = WP.matvec_blocks_wp(H.n, H.tree.perm, blocks, x, wp)
        r = WP.rounded_operand_product(H.n, H.tree.perm, blocks, x, wp)
        err = np.abs(y - r["y"])
        k = (r["K"] + r["nJ"])[:, None]
        bound = (WP.gamma(k, u) if wp == WP.WP_FP32 else WP.gamma_prob(k, u)) * r["S"]
        assert np.all(err <= bound), (wp, float(np.max(err / bound)))
        assert np.max(err / r["S"]) > u / 4          # rounding did happen
    assert F.unit_roundoff(F.FP16) == 2.0 ** -11
