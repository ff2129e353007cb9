"""Pins for oracle compression, Alg. 1/2/4, packing and Alg. 3 (matvec).  CPU only."""
from fractions import Fraction

import numpy as np
import pytest

import workloads as W
from oracle import compress as C
from oracle import dense as D
from oracle import formats as F
from oracle import hmatrix as HM
from oracle import matvec as MV
from oracle import metrics as M
from oracle import pack as PK
from oracle import partition as PT


# ------------------------------------------------------------- compression
def test_identity_eps_half_rank3():
    # ||I - I_p||_F = sqrt(4 - p) <= 0.5 * 2 first at p = 3 (direct arithmetic)
    assert C.lr_compress(np.eye(4), 0.5)["p"] == 3


def test_rank1_and_zero():
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal(30), rng.standard_normal(20)
    assert C.lr_compress(np.outer(a, b), 1e-10)["p"] == 1
    assert C.lr_compress(np.zeros((5, 7)), 1e-6)["p"] == 0


def test_truncation_rank_exact_arithmetic():
    """Tail summed from the smallest value equals the exact rational tail decision."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        s = np.sort(np.exp(rng.uniform(-40, 0, rng.integers(2, 40))))[::-1]
        eps = float(10.0 ** rng.uniform(-9, -1))
        p, *_ = C.truncation_rank(s, eps)
        sq = [Fraction(float(v)) ** 2 for v in s]
        tot = sum(sq)
        thr = Fraction(eps) ** 2 * tot
        exact = next(q for q in range(len(s) + 1) if sum(sq[q:]) <= thr)
        if exact != p:   # allowed only within rounding of the float threshold
            assert abs(float(sum(sq[min(p, exact):max(p, exact)]) / thr)) < 1e-12


@pytest.mark.parametrize("kind,d,eps", [(0, 2, 1e-8), (1, 3, 1e-6), (4, 3, 1e-6)])
def test_blocks_meet_eps_and_are_minimal(kind, d, eps):
    P = W.points_uniform(2000, d, 21)
    rng = np.random.default_rng(2)
    for _ in range(20):
        I = rng.choice(2000, 60, replace=False)
        J = rng.choice(np.setdiff1d(np.arange(2000), I), 50, replace=False)
        A, _ = __import__("oracle.kernels", fromlist=["block"]).block(P, I, J, kind, 0.1 if kind == 4 else 1.0)
        c = C.lr_compress(A, eps)
        nA = np.linalg.norm(A)
        assert np.linalg.norm(A - c["U"] @ c["W"].T) <= eps * nA * (1 + 1e-10)
        if c["p"] > 0:   # minimality: rank p - 1 violates the tolerance
            p = c["p"] - 1
            Ub, s, Vt = np.linalg.svd(A)
            assert np.linalg.norm(A - (Ub[:, :p] * s[:p]) @ Vt[:p]) > eps * nA
        # two LAPACK drivers agree on the rank
        assert C.lr_compress(A, eps, "gesvd")["p"] == c["p"]


# ------------------------------------------------------------- precision rule (Eq. 4.4)
def test_precision_rule_worked_example():
    # eps = 1e-4, d = 2, l = 4, xi = 1e-3 -> threshold eps/(2^{dl/2} xi) = 6.25e-3 -> bf16
    eps, d, l, xi = 1e-4, 2, 4, 1e-3
    assert eps / (2 ** (d * l / 2) * xi) == pytest.approx(6.25e-3)
    tag, fb = HM.choose_tag(nb2=xi ** 2, norm2=1.0, eps=eps, d=d, l=l, pset=W.P_MIXED)
    assert tag == F.BF16 and not fb
    # without bf16 the largest qualifying is fp16 (4.88e-4 <= 6.25e-3)
    assert HM.choose_tag(xi ** 2, 1.0, eps, d, l, W.P_FP64 | W.P_FP32 | W.P_FP16)[0] == F.FP16
    # eps = 1e-12, xi = 1 -> only the working precision (SPEC.md select_precision example)
    assert HM.choose_tag(1.0, 1.0, 1e-12, 2, 1, W.P_MIXED)[0] == F.FP64
    # xi so large that even fp64 fails -> fp64 + fallback flag
    assert HM.choose_tag(1.0, 1.0, 1e-17, 3, 10, W.P_MIXED) == (F.FP64, True)


def test_precision_rule_monotone_in_eps():
    rng = np.random.default_rng(4)
    for _ in range(300):
        nb2, l = float(rng.uniform(1e-12, 1)), int(rng.integers(1, 6))
        e1, e2 = sorted(10.0 ** rng.uniform(-12, -1, 2))
        u1 = F.unit_roundoff(HM.choose_tag(nb2, 1.0, e1, 3, l, W.P_MIXED)[0])
        u2 = F.unit_roundoff(HM.choose_tag(nb2, 1.0, e2, 3, l, W.P_MIXED)[0])
        assert u2 >= u1


def test_beneficial_rule_example():
    # 125 x 125 neighbour, rank 64: fp64 low-rank not beneficial, fp32 is
    p, m, n = 64, 125, 125
    assert not (p * (m + n) * 64 < m * n * 64)
    assert p * (m + n) * 32 < m * n * 64


# ------------------------------------------------------------- full H_h (2D tiny)
def test_lemma41_and_frobenius_norm(tiny_oracle):
    cfg, P, H = tiny_oracle
    A = D.dense_matrix(P, cfg["kernel"], cfg["scale"])
    perm = H.tree.perm
    Ht = np.zeros_like(A)   # H~ in tree order, unrounded factors
    for b in range(len(H.part)):
        i0, i1, j0, j1 = H.rows(b)
        if b in H.exact:
            U, Wf = H.exact[b]
            Ht[i0:i1, j0:j1] = U @ Wf.T
        else:
            Ht[i0:i1, j0:j1] = H.dense[b]
    At = A[np.ix_(perm, perm)]
    # Lemma 4.1: ||H - H~||_F <= eps ||H||_F
    assert np.linalg.norm(At - Ht) <= cfg["eps"] * np.linalg.norm(At)
    # Alg. 4: ||H~||^2 from singular values equals the dense reconstruction
    assert abs(H.norm2 - np.sum(Ht * Ht)) <= 1e-12 * H.norm2


def test_thm42_bound_and_fp64_gap(tiny_oracle):
    cfg, P, H = tiny_oracle
    err2, fro2 = M.global_error_sq(H, P, use_rounded=True)
    e_amp = np.sqrt(err2 / fro2)
    err2x, _ = M.global_error_sq(H, P, use_rounded=False)
    e_fp64 = np.sqrt(err2x / fro2)
    sc = PT.sparsity_constants(H.part, H.s, H.tree.L)
    ell, L, eps = H.s, H.tree.L, cfg["eps"]
    # Thm 4.2 with measured sparsity constants (reading G21)
    assert e_amp <= M.thm42_factor(L, ell, sc["c1"], sc["c2"], sc["c3"]) * eps
    # pre-constant form: e_amp - e_fp64 <= 2 eps sqrt(sum_b 2^{-d l_b})
    lv = M.lowrank_levels(H)
    assert e_amp - e_fp64 <= 2 * eps * np.sqrt(np.sum(2.0 ** (-2 * lv)))
    assert e_fp64 <= eps
    # mixed precision is actually used in this config
    tags = set(H.tag[list(H.factors)].tolist())
    assert F.FP32 in tags


def test_storage_rounding_uses_tag(tiny_oracle):
    _, _, H = tiny_oracle
    for b, (Uh, Wh) in list(H.factors.items())[:200]:
        U, Wf = H.exact[b]
        t = int(H.tag[b])
        np.testing.assert_array_equal(Uh, F.round_rne(U, t))
        np.testing.assert_array_equal(Wh, F.round_rne(Wf, t))


def test_only_fp64_at_eps_1e10():
    # for 1e-12 <= eps <= 1e-10 only double precision is selected
    P = W.points_uniform(1024, 2, 31, -1, 1)
    H = HM.build(P, W.K_LOG, 1.0, 1e-10, np.sqrt(2), 32, 2, W.P_MIXED)
    assert set(H.tag[list(H.factors)].tolist()) == {F.FP64}


def test_fig8_setting_uses_low_precisions():
    # eps = 1e-2 selects 16-bit formats for many blocks
    cfg = W.SMALL_CONFIGS["2d_fig8_e2"]
    P = W.make_points(cfg)
    H = HM.build(P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"], cfg["s"], cfg["pset"])
    tags = set(H.tag[list(H.factors)].tolist())
    assert F.BF16 in tags


# ------------------------------------------------------------- matvec (Alg. 3)
def test_matvec_equals_dense_reconstruction(tiny_oracle):
    cfg, P, H = tiny_oracle
    x = W.make_rhs(cfg, 3)
    y = MV.matvec(H, x)
    perm = H.tree.perm
    Hh = np.zeros((H.n, H.n))
    for b in range(len(H.part)):
        i0, i1, j0, j1 = H.rows(b)
        blk = H.factors[b][0] @ H.factors[b][1].T if b in H.factors else H.dense[b]
        Hh[np.ix_(perm[i0:i1], perm[j0:j1])] = blk
    ref = Hh @ x
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    # linearity and x = 0
    assert np.all(MV.matvec(H, np.zeros((H.n, 1))) == 0)
    y2 = MV.matvec(H, 2.0 * x[:, :1] - x[:, 1:2])
    np.testing.assert_allclose(y2, 2.0 * y[:, :1] - y[:, 1:2], rtol=0, atol=1e-12 * np.abs(y).max())


def test_matvec_error_vs_dense_bounds(tiny_oracle):
    cfg, P, H = tiny_oracle
    x = W.make_rhs(cfg)
    y = MV.matvec(H, x)
    Ax, fro2 = D.dense_apply(P, cfg["kernel"], cfg["scale"], x)
    e = M.e_mv(Ax, y, np.sqrt(fro2), x)[0]
    sc = PT.sparsity_constants(H.part, H.s, H.tree.L)
    assert e <= 10 * cfg["eps"]                                     # north-star check (3)
    assert e <= M.thm44_factor(H.tree.L, H.s, sc["c1"], sc["c2"], sc["c3"]) * cfg["eps"]


def test_single_leaf_is_dense_gemv():
    # L = 0 (N <= n_max): the H matrix is the dense matrix
    P = W.points_uniform(50, 3, 8)
    H = HM.build(P, W.K_INV_R, 1.0, 1e-6, 1.0, 64, 0, W.P_MIXED)
    assert H.tree.L == 0 and len(H.part) == 1
    x = W.rhs(50, 2, 9, "normal")
    A = D.dense_matrix(P, W.K_INV_R, 1.0)
    np.testing.assert_allclose(MV.matvec(H, x), A @ x, rtol=1e-13, atol=1e-13)


def test_pure_hs_mixed_beneficial_rule():
    P = W.points_uniform(1200, 3, 12)
    H = HM.build(P, W.K_INV_R, 1.0, 1e-6, 1.0, 20, PT.SWITCH_NONE, W.P_MIXED)
    ln = np.nonzero(H.part.kind == PT.LNBR)[0]
    assert ln.size > 0
    for b in ln[:300]:
        i0, i1, j0, j1 = H.rows(b)
        if H.storage[b] == HM.LR:
            assert H.rank[b] * ((i1 - i0) + (j1 - j0)) * F.BITS[int(H.tag[b])] < (i1 - i0) * (j1 - j0) * 64
    Hu = HM.build(P, W.K_INV_R, 1.0, 1e-6, 1.0, 20, PT.SWITCH_NONE, W.P_FP64)
    assert np.all(Hu.storage[ln] == HM.DENSE)


# ------------------------------------------------------------- packing function
def test_pack_roundtrip_and_invariants(tiny_oracle):
    cfg, P, H = tiny_oracle
    tr, part = H.tree, H.part
    lay = PK.pack(tr.leaf_start, tr.d, tr.L, part.level, part.tgt, part.src, H.rank, H.tag, H.storage)
    # write every block into byte arenas with the layout, then unpack it again
    arenas = {("W", g): np.zeros(int(lay["w_bytes"][g]), np.uint8) for g in F.TAGS}
    arenas.update({("U", g): np.zeros(int(lay["u_leaf_off"][g, -1]), np.uint8) for g in F.TAGS})
    arenas["D"] = np.zeros(int(lay["d_leaf_off"][-1]), np.uint8)
    used = {k: np.zeros(v.size, np.int32) for k, v in arenas.items()}

    def put(key, off, vals, g):
        b = F.to_storage_bits(vals, g).tobytes()
        assert off % F.BYTES[g] == 0
        arenas[key][off:off + len(b)] = np.frombuffer(b, np.uint8)
        used[key][off:off + len(b)] += 1

    for b in range(len(part)):
        i0, i1, j0, j1 = H.rows(b)
        if H.storage[b] == HM.DENSE:
            put("D", int(lay["d_off"][b]), H.dense[b].T.ravel(), F.FP64)
            continue
        U, Wf = H.factors[b]
        g, p = int(H.tag[b]), int(H.rank[b])
        if p == 0:
            continue
        assert lay["w_off"][b] % 16 == 0
        offs = PK.w_offsets(lay, b, g)                      # (n, p) element offsets
        bits = np.frombuffer(F.to_storage_bits(Wf.ravel(), g).tobytes(), np.uint8).reshape(-1, F.BYTES[g])
        for k in range(F.BYTES[g]):
            arenas[("W", g)][offs.ravel() + k] = bits[:, k]
            used[("W", g)][offs.ravel() + k] += 1
        l = int(part.level[b])
        s = tr.d * (tr.L - l)
        for R in range(int(part.tgt[b]) << s, (int(part.tgt[b]) + 1) << s):
            r0, r1 = int(tr.leaf_start[R]), int(tr.leaf_start[R + 1])
            if r1 > r0:
                off = int(lay["u_leaf_off"][g, R]) + int(lay["ucol"][b]) * (r1 - r0) * F.BYTES[g]
                put(("U", g), off, U[r0 - i0:r1 - i0].T.ravel(), g)
    assert np.any(lay["wpanel"] > PK.CT)  # multi-tile W panels are exercised
    for k in used:                      # no byte written twice
        assert used[k].max(initial=0) <= 1
    for g in F.TAGS:
        assert np.all(lay["u_leaf_off"][g] % 16 == 0)
    for b in range(len(part)):
        kind, payload = PK.unpack_block(lay, b, tr.leaf_start, tr.d, tr.L, part.level, part.tgt,
                                        H.rank, H.tag, H.storage, arenas)
        if kind == "dense":
            np.testing.assert_array_equal(payload, H.dense[b])
        elif H.rank[b] > 0:
            np.testing.assert_array_equal(payload[0], H.factors[b][0])
            np.testing.assert_array_equal(payload[1], H.factors[b][1])
    # z: each (level, tgt, tag) group is one contiguous z range
    lr = np.nonzero(H.storage == HM.LR)[0]
    ends = {}
    for b in lr:
        key = (int(part.level[b]), int(part.tgt[b]), int(H.tag[b]))
        ends.setdefault(key, []).append((int(lay["zoff"][b]), int(H.rank[b])))
    for v in ends.values():
        v.sort()
        for (a, pa), (c, _) in zip(v, v[1:]):
            assert a + pa == c


# ------------------------------------------------------------- Alg. 5 (switching level)
# pinned in tests/test_oracle_pins.py (worked examples of the walk; brute-force argmax)


@pytest.mark.slow
def test_table3_s1_over_s2_3d_inv_r():
    """Table 3: S_1(ell)/S_2(ell) at ell = L-1 for 3D 1/r, N=64000 uniform in
    [-1,1]^3, L=3 (n_max=125 in the paper's balanced-tree formula), eta=sqrt(3), eps=1e-6:
    printed 1.60.  Storage in words (uniform precision); units of the printed S_1, S_2 are
    unstated, so only the ratio is pinned, with a band for the unknown point seed
    (1.60 +- 0.15).  Slow: ~10^5 SVDs (not in the default CPU suite)."""
    from oracle.partition import FAR, LNBR, NBR, SIB
    P = W.points_uniform(64000, 3, 64000, -1.0, 1.0)
    eta, eps = np.sqrt(3.0), 1e-6
    leaf = 250   # the depth rule then gives L = 3
    trs, ps, rs, ms, ns = HM.ranks_only(P, W.K_INV_R, 1.0, eps, eta, leaf, PT.SWITCH_NONE)
    assert trs.L == 3
    ell = trs.L - 1
    S1 = int(np.sum((rs * (ms + ns))[(ps.level > ell) & (ps.kind == FAR)])) + int(np.sum((ms * ns)[ps.kind == LNBR]))
    trh, ph, rh, mh, nh = HM.ranks_only(P, W.K_INV_R, 1.0, eps, eta, leaf, ell)
    S2 = int(np.sum((rh * (mh + nh))[((ph.level == ell) & (ph.kind == NBR)) | ((ph.level > ell) & (ph.kind == SIB))]))
    ratio = S1 / S2
    print("Table 3 L=3 eps=1e-6: S1/S2 =", ratio)
    assert 1.45 <= ratio <= 1.75, ratio


def test_tie_rule_fp16_over_bf16():
    """NEXT-3 bits-aware tie rule (HH_TIE_FP16): every block the paper's rule stores in bf16
    (largest u) goes to fp16 instead — same bits, so identical storage —
    unless an entry would overflow fp16; the blocks' rounding errors can only shrink."""
    cfg = W.SMALL_CONFIGS["2d_fig8_e2"]
    P = W.make_points(cfg)
    args = (P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"], cfg["s"])
    H0 = HM.build(*args, cfg["pset"], keep_exact=True)
    H1 = HM.build(*args, cfg["pset"] | HM.TIE_FP16, keep_exact=True)
    lr = H0.storage == HM.LR
    assert np.sum(H0.tag[lr] == F.BF16) > 0
    moved = lr & (H0.tag == F.BF16)
    assert np.all(H1.tag[moved] == F.FP16)
    assert np.all(H1.tag[lr & ~moved] == H0.tag[lr & ~moved])
    assert HM.stored_bytes(H1)["total"] == HM.stored_bytes(H0)["total"]
    for b in np.nonzero(moved)[0][:50]:
        U, Wf = H1.exact[b]
        e0 = np.linalg.norm(U @ Wf.T - H0.factors[b][0] @ H0.factors[b][1].T)
        e1 = np.linalg.norm(U @ Wf.T - H1.factors[b][0] @ H1.factors[b][1].T)
        assert e1 <= e0
