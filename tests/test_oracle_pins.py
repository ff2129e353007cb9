"""Pins for the oracle functions VERDICT r01 listed as unpinned: kernel values (Eq. 5.1), the
range guard (reading G16), the PAPER.md:992 beneficial rule, the measured sparsity constants
 and Alg. 5.  Each pin is a closed form, a worked
example derived by hand from the paper's text, or a brute force over all candidates — never
a retyping of the function under test.  CPU only."""
import math

import numpy as np
import pytest

import workloads as W
from oracle import compress as C
from oracle import formats as F
from oracle import hmatrix as HM
from oracle import kernels as K
from oracle import partition as PT
from oracle import switch_level as SL
from oracle import tree as T

E = math.e


# ------------------------------------------------------------- kernels, Eq. 5.1
def test_kernel_values_closed_forms():
    r = np.array([E, 1.0, E * E, 2.0, 0.1, 0.5])
    np.testing.assert_allclose(K.f_of_r(K.K_LOG, r[:3], 1.0), [1.0, 0.0, 2.0], rtol=0, atol=1e-15)   # natural log
    assert K.f_of_r(K.K_INV_R, np.array([2.0]), 1.0)[0] == 0.5
    assert K.f_of_r(K.K_INV_R2, np.array([2.0]), 1.0)[0] == 0.25
    assert K.f_of_r(K.K_INV_R2, np.array([0.5]), 1.0)[0] == 4.0
    # exp(-r/s): r = s gives 1/e; r = 2s gives 1/e^2
    np.testing.assert_allclose(K.f_of_r(K.K_EXP, np.array([0.1, 0.2]), 0.1), [1 / E, 1 / (E * E)], rtol=1e-15)
    # Gaussian exp(-r^2 / (2 s^2)): r = s gives e^{-1/2}, r = 2s gives e^{-2}
    np.testing.assert_allclose(K.f_of_r(K.K_GAUSS, np.array([0.3, 0.6]), 0.3), [E ** -0.5, E ** -2], rtol=1e-15)


def test_kernel_block_distance_diagonal_and_coincident_points():
    # a 3-4-5 triangle pins the Euclidean distance (not L1 / L-inf / squared)
    P = np.array([[0.0, 0.0], [3.0, 0.0], [0.0, 4.0]])
    idx = np.arange(3)
    A, c = K.block(P, idx, idx, K.K_INV_R, 1.0)
    np.testing.assert_allclose(A, [[0, 1 / 3, 1 / 4], [1 / 3, 0, 1 / 5], [1 / 4, 1 / 5, 0]], rtol=1e-15)
    assert c == 0
    A, _ = K.block(P, idx, idx, K.K_INV_R2, 1.0)
    np.testing.assert_allclose(A, [[0, 1 / 9, 1 / 16], [1 / 9, 0, 1 / 25], [1 / 16, 1 / 25, 0]], rtol=1e-15)
    # log r on a distance of e and e^2 (points on a line)
    Q = np.array([[0.0, 0.0], [E, 0.0], [E * E, 0.0]])
    A, _ = K.block(Q, np.array([0]), np.array([1, 2]), K.K_LOG, 1.0)
    np.testing.assert_allclose(A, [[1.0, 2.0]], rtol=1e-15)
    # non-singular kernels: diagonal f(0) = 1 (PAPER.md:1119 only zeroes singular kernels)
    for kind in (K.K_EXP, K.K_GAUSS):
        A, _ = K.block(P, idx, idx, kind, 0.5)
        np.testing.assert_array_equal(np.diag(A), [1.0, 1.0, 1.0])
    # singular kernels: index-keyed zero diagonal; a DISTINCT coincident pair is 0 and counted (G18)
    R = np.array([[0.25, 0.5], [0.25, 0.5], [1.25, 0.5]])
    for kind in (K.K_LOG, K.K_INV_R, K.K_INV_R2):
        A, c = K.block(R, np.arange(3), np.arange(3), kind, 1.0)
        assert A[0, 1] == 0.0 and A[1, 0] == 0.0 and np.all(np.diag(A) == 0.0)
        assert c == 2                               # (0,1) and (1,0)
        assert A[0, 2] == {K.K_LOG: 0.0, K.K_INV_R: 1.0, K.K_INV_R2: 1.0}[kind]   # distance 1


# ------------------------------------------------------------- range guard (Table 1 x_max, reading G16)
def test_guard_tag_boundaries():
    mixed = W.P_MIXED
    # fp16: x_max = 65504; RNE sends [65504, 65520) to 65504 and 65520 (the midpoint to 2^16) to inf
    assert HM.guard_tag(F.FP16, 65504.0, mixed) == (F.FP16, False)
    assert HM.guard_tag(F.FP16, 65519.99, mixed) == (F.FP16, False)
    assert HM.guard_tag(F.FP16, 65520.0, mixed) == (F.FP32, True)
    assert HM.guard_tag(F.FP16, 7e4, mixed) == (F.FP32, True)
    # without fp32 in the set the next smaller u is fp64
    assert HM.guard_tag(F.FP16, 7e4, W.P_FP64 | W.P_FP16) == (F.FP64, True)
    # bf16: x_max = 0x1.fep127; the midpoint 0x1.ffp127 ties to the even neighbour 2^128 = inf
    assert HM.guard_tag(F.BF16, float.fromhex("0x1.fep127"), mixed) == (F.BF16, False)
    assert HM.guard_tag(F.BF16, float.fromhex("0x1.fefffp127"), mixed) == (F.BF16, False)
    # a value that overflows bf16 overflows fp16 too: bf16 -> (fp16 ->) fp32, one promotion
    assert HM.guard_tag(F.BF16, float.fromhex("0x1.ffp127"), mixed) == (F.FP32, True)
    # beyond fp32's range: fp64
    assert HM.guard_tag(F.BF16, 1e39, mixed) == (F.FP64, True)
    assert HM.guard_tag(F.BF16, 1e39, W.P_FP64 | W.P_BF16) == (F.FP64, True)
    # fp32 boundary: x_max = 0x1.fffffep127, overflow from the midpoint 0x1.ffffffp127
    assert HM.guard_tag(F.FP32, float.fromhex("0x1.fffffep127"), mixed) == (F.FP32, False)
    assert HM.guard_tag(F.FP32, float.fromhex("0x1.ffffffp127"), mixed) == (F.FP64, True)
    # fp64 never promotes
    assert HM.guard_tag(F.FP64, 1e300, mixed) == (F.FP64, False)


def test_promotion_end_to_end_tiny_domain():
    """Entries of 1/r^2 on points spread over 1e-20 exceed every 16/32-bit format's range
    (r^-2 ~ 1e40 > 3.4e38), so every low-rank block the precision rule would store in a low
    precision is promoted to fp64 and the stored factors stay finite."""
    P = W.points_uniform(600, 2, 5) * 1e-20
    H = HM.build(P, W.K_INV_R2, 1.0, 1e-2, 1.0, 16, 2, W.P_MIXED, keep_exact=True)
    lr = [b for b in H.factors if H.rank[b] > 0]
    assert H.promoted > 0 and H.promoted == len(lr)
    assert all(H.tag[b] == F.FP64 for b in lr)
    for b in lr:
        assert np.all(np.isfinite(H.factors[b][0])) and np.all(np.isfinite(H.factors[b][1]))
    # the same points scaled to 1e-5 (1/r^2 ~ 1e10): fp16 and bf16 candidates overflow fp16 only
    H2 = HM.build(W.points_uniform(600, 2, 5) * 1e-3, W.K_INV_R, 1.0, 1e-2, 1.0, 16, 2,
                  W.P_FP64 | W.P_FP32 | W.P_FP16, keep_exact=True)
    assert H2.promoted > 0
    for b in H2.factors:
        if H2.rank[b] and H2.tag[b] == F.FP16:
            U, Wf = H2.exact[b]
            assert max(np.abs(U).max(), np.abs(Wf).max()) < 65520.0


# ------------------------------------------------------------- beneficial rule
def test_beneficial_rule_paper_example_through_tagging():
    """a 125 x 125 neighbour block of rank 64 is not worth compressing in fp64
    (64 * 250 > 125 * 125) but is in fp32 (64 * 250 * 0.5 < 125 * 125).  Two such leaf
    neighbours of a mixed pure-H_s table, one whose Eq. 4.4 tag is fp64 (large xi) and one
    fp32 (small xi), go through the oracle's Alg. 2: the first is kept dense, the second
    low-rank."""
    # tree: two level-1 leaves in 1D with 125 points each
    ls = np.array([0, 125, 250])
    level = np.array([1, 1, 1, 1])
    kind = np.array([PT.DIAG, PT.LNBR, PT.LNBR, PT.DIAG])
    m = np.array([125, 125, 125, 125])
    rank = np.array([0, 64, 64, 0])
    eps = 1e-10
    # ||H~||^2 = 2 (dense diagonals, tot) + tot of the two neighbours (Alg. 4, ell = L branch)
    tot = np.array([1.0, 1.0, 1e-6, 1.0])
    nb2 = np.array([0.0, 1.0, 1e-6, 0.0])
    T_ = HM.tag_blocks(1, level, kind, m, m, rank, nb2, tot, np.ones(4), eps, W.P_MIXED)
    assert T_["lr_tag"][1] == F.FP64 and T_["lr_tag"][2] == F.FP32
    assert T_["storage"][1] == HM.DENSE and T_["rank"][1] == 0
    assert T_["storage"][2] == HM.LR and T_["tag"][2] == F.FP32 and T_["rank"][2] == 64
    assert ls[-1] == 250
    # uniform precision keeps every leaf neighbour dense (Alg. 1, ell = L)
    U_ = HM.tag_blocks(1, level, kind, m, m, rank, nb2, tot, np.ones(4), eps, W.P_FP64)
    assert np.all(U_["storage"] == HM.DENSE)


def test_beneficial_rule_through_build():
    """Mixed pure H_s (2D log, eps = 1e-8, leaf 16): every leaf neighbour the build keeps
    dense would store MORE bits as factors at its tag, every one kept low-rank fewer, and
    both outcomes occur (so neither 'always dense' nor 'always low-rank' passes)."""
    P = W.points_uniform(1500, 2, 12)
    H = HM.build(P, W.K_LOG, 1.0, 1e-8, 1.0, 16, PT.SWITCH_NONE, W.P_MIXED)
    ln = np.nonzero(H.part.kind == PT.LNBR)[0]
    dense = ln[H.storage[ln] == HM.DENSE]
    low = ln[H.storage[ln] == HM.LR]
    assert dense.size > 100 and low.size > 100
    for b in ln:
        i0, i1, j0, j1 = H.rows(b)
        m, n = i1 - i0, j1 - j0
        # the rank the compression found, recomputed from the block's singular values
        bits_lr = int(H.lr_rank[b]) * (m + n) * F.BITS[int(H.lr_tag[b])]
        if H.storage[b] == HM.DENSE:
            assert bits_lr >= m * n * 64 and H.rank[b] == 0 and b in H.dense
        else:
            assert bits_lr < m * n * 64 and H.rank[b] == H.lr_rank[b] and H.tag[b] == H.lr_tag[b]
    # spot-check that lr_rank is the truncated-SVD rank of the block
    from oracle.kernels import block as kb
    for b in dense[:5]:
        i0, i1, j0, j1 = H.rows(b)
        A, _ = kb(P, H.tree.perm[i0:i1], H.tree.perm[j0:j1], W.K_LOG, 1.0)
        assert C.lr_compress(A, 1e-8)["p"] == H.lr_rank[b]


# ------------------------------------------------------------- sparsity constants
def _grid_tree(d, L):
    return T.build_tree(W.points_grid_centres(d, L), 1)


def test_sparsity_constants_eta_sqrt2_2d():
    # |IL_s| <= 27, |N_s| <= 8 at eta = sqrt(2) in 2D (attained on a full grid)
    tr = _grid_tree(2, 4)
    c = PT.sparsity_constants(PT.build_partition(tr, np.sqrt(2.0), PT.SWITCH_NONE), PT.SWITCH_NONE, tr.L)
    assert (c["c1"], c["c2"], c["c3"]) == (27, 8, 0)
    c = PT.sparsity_constants(PT.build_partition(tr, np.sqrt(2.0), 0), 0, tr.L)
    assert (c["c1"], c["c2"], c["c3"]) == (0, 0, 3)          # HODLR: C''' = 2^d - 1
    c = PT.sparsity_constants(PT.build_partition(tr, np.sqrt(2.0), 3), 3, tr.L)
    assert (c["c1"], c["c2"], c["c3"]) == (27, 8, 3)


def test_sparsity_constants_eta_sqrt3_3d():
    # PAPER.md:1134 (Eq. 5.3): 189, 26, 7 at eta = sqrt(3) in 3D
    tr = _grid_tree(3, 3)
    c = PT.sparsity_constants(PT.build_partition(tr, np.sqrt(3.0), PT.SWITCH_NONE), PT.SWITCH_NONE, tr.L)
    assert (c["c1"], c["c2"]) == (189, 26)
    # switch level 2 of an L = 3 tree: the far list lives on the 4 x 4 x 4 grid of level 2 only,
    # where a box has at most 4^3 - 2^3 admissible partners (a corner box's 7 neighbours + itself)
    c = PT.sparsity_constants(PT.build_partition(tr, np.sqrt(3.0), 2), 2, tr.L)
    assert (c["c1"], c["c2"], c["c3"]) == (56, 26, 7)
    tr4 = _grid_tree(3, 4)
    c = PT.sparsity_constants(PT.build_partition(tr4, np.sqrt(3.0), 3), 3, tr4.L)
    assert (c["c1"], c["c2"], c["c3"]) == (189, 26, 7)


def test_sparsity_constants_bruteforce_random_tree():
    """On a random point set (empty boxes, ragged occupancy) each constant equals the largest
    count of blocks of its kind sharing one (level, target), counted by a plain loop."""
    P = W.points_uniform(700, 2, 9) ** 2          # skewed density: many empty boxes
    tr = T.build_tree(P, 8)
    for s in (PT.SWITCH_NONE, 1, 2, tr.L):
        part = PT.build_partition(tr, 1.0, s)
        cnt = {}
        for b in range(len(part)):
            key = (int(part.kind[b]) if part.kind[b] != PT.LNBR else PT.NBR, int(part.level[b]), int(part.tgt[b]))
            cnt[key] = cnt.get(key, 0) + 1
        best = {k: 0 for k in (PT.FAR, PT.NBR, PT.SIB)}
        for (k, _, _), v in cnt.items():
            if k in best:
                best[k] = max(best[k], v)
        c = PT.sparsity_constants(part, s, tr.L)
        assert (c["c1"], c["c2"], c["c3"]) == (best[PT.FAR], best[PT.NBR], best[PT.SIB]), s


# ------------------------------------------------------------- Alg. 5
def test_alg5_walk_worked_examples():
    """Alg. 5 by hand: start at ell = L with gain 0, step down while S_s - S_h(ell-1) grows.
    S_s = 10, S_h = [5, 9, 6, 8] (L = 4): gains from ell = 3 down are 2, 4, 1 -> stops at
    ell* = 2 (the global argmax, ell = 0 with gain 5, is behind a dip and is not reached)."""
    seen = []

    def sh(l):
        seen.append(l)
        return [5, 9, 6, 8][l]
    ell, by = SL.walk(4, 10, sh)
    assert ell == 2 and seen == [3, 2, 1] and by == [-1, 9, 6, 8, 10, 10]
    # no level gains over H_s: ell* = L (the walk evaluates one level and stops)
    assert SL.walk(3, 10, lambda l: 10)[0] == 3
    assert SL.walk(3, 10, lambda l: 12)[0] == 3
    # monotone gains: walks to the root
    assert SL.walk(3, 10, lambda l: 4 + l)[0] == 0
    # equal gain does not move (the paper's strict improvement)
    assert SL.walk(3, 10, lambda l: 7)[0] == 2


def test_alg_lstar_equals_bruteforce_argmax():
    """On a 2D log case whose gains S_s - S_h(ell) are unimodal in ell (checked), the walk's
    ell* equals the brute-force argmax over EVERY switch level (ties to the larger ell: the
    walk only moves on a strict gain), and the visited storages equal independent builds."""
    P = W.points_uniform(1500, 2, 31)
    args = (W.K_LOG, 1.0, 1e-6, 1.0, 24, W.P_MIXED)
    ell, L, by = SL.alg_lstar(P, *args)
    Ss = HM.stored_bytes(HM.build(P, *args[:5], PT.SWITCH_NONE, args[5]))["total"]
    Sh = [HM.stored_bytes(HM.build(P, *args[:5], s, args[5]))["total"] for s in range(L)]
    gains = [Ss - b for b in Sh] + [0]
    best = max(gains)
    argmax = max(l for l in range(L + 1) if gains[l] == best)
    # the walk can reach the argmax: gains strictly grow from ell = L down to it
    assert all(gains[l] > gains[l + 1] for l in range(argmax, L))
    assert argmax < L - 1                       # a non-trivial walk
    assert ell == argmax
    assert by[L + 1] == Ss and all(by[l] in (-1, Sh[l]) for l in range(L))
    assert (Sh + [Ss])[ell] <= Ss


# ------------------------------------------------------------- Table 3, reduced
def test_table3_s1_over_s2_sampled():
    """Table 3 at L=3, eps=1e-6 (3D 1/r, N=64000 uniform in [-1,1]^3, eta=sqrt(3), ell=L-1):
    printed S1/S2 = 1.60.  The partition and every dense size are exact; the low-rank sums are
    estimated per (level, kind) class from the truncated-SVD ranks of a seeded sample of the
    class's blocks (class count x sample mean of p(|I|+|J|)).  Band 1.60 +- 0.15 (the point
    seed is unknown); the full-sum version is the --runslow test in
    test_oracle_hmatrix.py."""
    from scipy.linalg import svdvals
    from oracle.kernels import block as kb
    P = W.points_uniform(64000, 3, 64000, -1.0, 1.0)
    eta, eps = np.sqrt(3.0), 1e-6
    tr = T.build_tree(P, 250)
    assert tr.L == 3
    ell = tr.L - 1
    rng = np.random.default_rng(3)

    def est(part, mask, nsample):
        idx = np.nonzero(mask)[0]
        pick = rng.choice(idx, size=min(nsample, idx.size), replace=False)
        vals = []
        for b in pick:
            l = int(part.level[b])
            i0, i1 = tr.cluster(l, int(part.tgt[b]))
            j0, j1 = tr.cluster(l, int(part.src[b]))
            A, _ = kb(P, tr.perm[i0:i1], tr.perm[j0:j1], W.K_INV_R, 1.0)
            p = C.truncation_rank(svdvals(A), eps)[0]
            vals.append(p * ((i1 - i0) + (j1 - j0)))
        return idx.size * float(np.mean(vals))

    def sizes(part, mask):
        out = 0
        for b in np.nonzero(mask)[0]:
            l = int(part.level[b])
            i0, i1 = tr.cluster(l, int(part.tgt[b]))
            j0, j1 = tr.cluster(l, int(part.src[b]))
            out += (i1 - i0) * (j1 - j0)
        return out

    ps = PT.build_partition(tr, eta, PT.SWITCH_NONE)
    S1 = est(ps, (ps.level > ell) & (ps.kind == PT.FAR), 150) + sizes(ps, ps.kind == PT.LNBR)
    ph = PT.build_partition(tr, eta, ell)
    S2 = est(ph, (ph.level == ell) & (ph.kind == PT.NBR), 30) + est(ph, (ph.level > ell) & (ph.kind == PT.SIB), 150)
    ratio = S1 / S2
    print("Table 3 (sampled) L=3 eps=1e-6: S1/S2 =", ratio)
    assert 1.45 <= ratio <= 1.75, ratio
