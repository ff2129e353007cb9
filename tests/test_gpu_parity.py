"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.  Needs a B200."""
import os

import numpy as np
import pytest

import workloads as W
from oracle import dense as D
from oracle import formats as F
from oracle import metrics as M
from oracle import partition as PT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import parity_lib as PL  # noqa: E402
from paper_2604_09147_b200 import hh  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["2d_tiny", "2d_fig8_e4", "2d_fig8_e2", "3d_small_inv_r", "3d_small_exp", "3d_sphere_small", "2d_circle_small",
         "1d_log", "2d_fig8_e2_q43", "3d_small_exp_q43", "3d_small_inv_r_acc", "2d_tiny_acc"]


@pytest.fixture(scope="module", params=SMALL)
def built(request):
    cfg = W.SMALL_CONFIGS[request.param]
    P = W.make_points(cfg)
    H = PL.gpu_build(P, cfg)
    ex = PL.export(H)
    Ho = PL.oracle_build(P, cfg, keep_exact=True)
    return request.param, cfg, P, H, ex, Ho


def test_check1a_partition_bit_exact(built):
    _, cfg, P, H, ex, Ho = built
    PL.check_partition(ex, Ho)


def test_check1b_ranks_and_tags(built):
    name, cfg, P, H, ex, Ho = built
    bad_r, bad_t, st = PL.rank_tag_parity(ex, Ho)
    print(name, st)
    assert bad_r == 0 and bad_t == 0, st
    # ||H~||^2 agrees with the oracle's Alg. 4 value.  Tolerance (reading G26): the device's
    # nb2_b = sum of the kept sigma^2 of Q^T A differs from the SVD's by at most the sketch
    # residual R_b <= 1e-10 ||A_b||^2 it certifies, so the sum agrees to 1e-10 relative (2e-10
    # with rounding); at eps = 1e-6 the sketches are wide and the agreement is ~1e-15
    assert abs(ex["info"]["norm2"] - Ho.norm2) <= 2e-10 * Ho.norm2


def test_check1c_packing_function(built):
    _, cfg, P, H, ex, Ho = built
    PL.check_packing(ex)


def test_check2_matvec_vs_oracle_on_exported_factors(built):
    _, cfg, P, H, ex, Ho = built
    lay = PL.check_packing(ex)
    for nrhs in sorted({1, cfg["nrhs"], 3, 16, 20}):   # 20 = a 16-column chunk + a 4-column chunk
        x = W.make_rhs(cfg, nrhs)
        y = PL.gpu_matvec(H, x)
        yo = PL.oracle_matvec_on_export(ex, lay, x)
        for c in range(nrhs):
            assert PL.rel2(y[:, c], yo[:, c]) <= 1e-12, (nrhs, c, PL.rel2(y[:, c], yo[:, c]))


def test_check3_and_4_error_vs_dense(built):
    name, cfg, P, H, ex, Ho = built
    x = W.make_rhs(cfg)
    y = PL.gpu_matvec(H, x)
    Ax, fro2 = D.dense_apply(P, cfg["kernel"], cfg["scale"], x)
    e = M.e_mv(Ax, y, np.sqrt(fro2), x)[0]
    assert e <= 10 * cfg["eps"], e                                   # check (3)
    L, ell = ex["info"]["L"], cfg["s"]
    info = ex["info"]
    bound = M.thm44_factor(L, ell, info["c_far"], info["c_nbr"], info["c_sib"]) * cfg["eps"]
    assert e <= bound                                                # Thm 4.4, measured constants
    # check (4): mixed vs uniform-fp64 H_h, same partition
    H64 = PL.gpu_build(P, cfg, pset=W.P_FP64)
    y64 = PL.gpu_matvec(H64, x)
    e64 = M.e_mv(Ax, y64, np.sqrt(fro2), x)[0]
    B = ex["blocks"]
    lv = B["level"][(B["storage"] == 0) & (B["rank"] > 0)].astype(float)
    assert e - e64 <= 2 * cfg["eps"] * np.sqrt(np.sum(2.0 ** (-cfg["d"] * lv))) + 1e-15
    assert e64 <= 10 * cfg["eps"]


def test_global_error_thm42(built):
    name, cfg, P, H, ex, Ho = built
    lay = PL.check_packing(ex)
    err2 = fro2 = 0.0
    from oracle.kernels import block as kb
    perm = ex["perm"].astype(np.int64)
    for i0, i1, j0, j1, kind, payload in PL.exported_blocks(ex, lay):
        A, _ = kb(P, perm[i0:i1], perm[j0:j1], cfg["kernel"], cfg["scale"])
        fro2 += float(np.sum(A * A))
        if kind == "lr":
            E = A - payload[0] @ payload[1].T
            err2 += float(np.sum(E * E))
    info = ex["info"]
    e = np.sqrt(err2 / fro2)
    assert e <= M.thm42_factor(info["L"], cfg["s"], info["c_far"], info["c_nbr"], info["c_sib"]) * cfg["eps"]


def test_determinism_bitwise(built):
    """No atomics in the arithmetic, fixed summation orders: bitwise-identical y across runs and
    across streams, for every RHS-chunk kernel width (2: DFMA; 16: DMMA with the phase-2
    leaf-end reduction in the leaf's last TMA stage; 20: a 16-wide then a 4-wide chunk).  A
    column's bits depend on its chunk width (different contraction kernels), not on the run."""
    _, cfg, P, H, ex, Ho = built
    for nrhs in (2, 16, 20):
        x = W.make_rhs(cfg, nrhs)
        y1 = PL.gpu_matvec(H, x)
        y2 = PL.gpu_matvec(H, x)
        assert np.array_equal(y1, y2), nrhs
        s = torch.cuda.Stream()
        xd = torch.from_numpy(x.T.copy()).cuda().T
        yd = torch.empty_like(xd.T).T
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            hh.hh_matvec(H, xd, yd, nrhs, stream=s)
        s.synchronize()
        assert np.array_equal(yd.cpu().numpy(), y1), nrhs
    # the first 16 columns of the 20-column product are the 16-column product's columns
    x = W.make_rhs(cfg, 20)
    assert np.array_equal(PL.gpu_matvec(H, x)[:, :16], PL.gpu_matvec(H, np.asfortranarray(x[:, :16])))


def test_rounding_routines_match_oracle():
    rng = np.random.default_rng(5)
    base = rng.standard_normal(5000) * np.exp2(rng.integers(-140, 130, 5000))
    for tag in (F.FP32, F.FP16, F.BF16, F.Q43, F.BF24):
        r = F.round_rne(base, tag)
        fin = np.isfinite(r) & (r != 0)
        m, emin, _ = F.PARAMS[tag]
        _, e = np.frexp(np.abs(r[fin]))
        q = np.ldexp(1.0, np.maximum(e - 1, emin) - m)       # spacing of the format at r
        mids = r[fin] + np.sign(r[fin]) * q / 2               # exact rounding midpoints
        xs = np.concatenate([base, mids, np.nextafter(mids, 0), np.nextafter(mids, np.inf), [65519.99, 65520, 0.1]])
        xs = xs[np.isfinite(xs)]
        got = hh.selftest_round(xs, tag)
        ref = F.to_storage_bits(xs, tag).astype(np.uint32)
        if tag == F.BF24:     # three little-endian bytes -> the 24-bit pattern
            ref = ref[:, 0] | (ref[:, 1] << np.uint32(8)) | (ref[:, 2] << np.uint32(16))
        np.testing.assert_array_equal(got, ref)


def test_edge_cases_single_leaf_zero_x_hodlr_and_pure_hs():
    # L = 0: N <= leaf -> dense gemv
    P = W.points_uniform(60, 3, 77)
    cfg = dict(kernel=W.K_INV_R, scale=1.0, eps=1e-6, eta=1.0, leaf=64, s=0, pset=W.P_MIXED)
    H = PL.gpu_build(P, cfg)
    x = W.rhs(60, 2, 1, "normal")
    A = D.dense_matrix(P, W.K_INV_R, 1.0)
    assert PL.rel2(PL.gpu_matvec(H, x), A @ x) < 1e-14
    assert np.all(PL.gpu_matvec(H, np.zeros((60, 1))) == 0)
    # HODLR (s = 0) and pure H_s (NONE), uniform and mixed, ragged leaves
    P = W.points_uniform(3000, 2, 78)
    for s in (0, 1, PT.SWITCH_NONE):
        for pset in (W.P_FP64, W.P_MIXED):
            cfg = dict(kernel=W.K_LOG, scale=1.0, eps=1e-6, eta=1.0, leaf=24, s=s, pset=pset)
            H = PL.gpu_build(P, cfg)
            ex = PL.export(H)
            Ho = PL.oracle_build(P, cfg)
            PL.check_partition(ex, Ho)
            bad_r, bad_t, st = PL.rank_tag_parity(ex, Ho)
            assert bad_r == 0 and bad_t == 0, (s, pset, st)
            lay = PL.check_packing(ex)
            x = W.rhs(3000, 1, 2, "uniform_pm1")
            assert PL.rel2(PL.gpu_matvec(H, x), PL.oracle_matvec_on_export(ex, lay, x)) <= 1e-12


def test_invalid_arguments_are_rejected():
    P = torch.from_numpy(W.points_uniform(100, 2, 1)).cuda()
    with pytest.raises(hh.HHError) as e:
        hh.hh_build(P, 0, 1.0, 1e-6, 1.0, 16, 99, W.P_MIXED)     # switch level > L
    assert e.value.status == hh.HH_EINVAL
    with pytest.raises(hh.HHError):
        hh.hh_build(P, 0, 1.0, 1e-6, 1.0, 16, 2, W.P_FP32)       # no fp64
    with pytest.raises(hh.HHError):
        hh.hh_build(P, 0, 1.0, 0.0, 1.0, 16, 2, W.P_MIXED)       # eps
    bad = P.clone()
    bad[3, 0] = float("nan")
    with pytest.raises(hh.HHError) as e:
        hh.hh_build(bad, 0, 1.0, 1e-6, 1.0, 16, 2, W.P_MIXED)
    assert e.value.status == hh.HH_ENUMERIC


def test_whole_gpu_compression_path_matches_oracle():
    """compress_big.cu (explicit entries + cuBLAS/cuSOLVER, used for large wide-sketch blocks)
    gives the same partition, ranks, tags and matvec as the oracle; forced onto every block of
    a small 3D problem with HH_BIG_FLOPS (read by the library at its first use in this process)."""
    import subprocess
    import sys
    code = r'''
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, workloads as W, parity_lib as PL
cfg = dict(W.SMALL_CONFIGS["3d_small_inv_r"], s=0)
P = W.make_points(cfg)
H = PL.gpu_build(P, cfg)
ex = PL.export(H)
Ho = PL.oracle_build(P, cfg)
PL.check_partition(ex, Ho)
bad_r, bad_t, st = PL.rank_tag_parity(ex, Ho)
assert bad_r == 0 and bad_t == 0, st
lay = PL.check_packing(ex)
x = W.make_rhs(cfg, 3)
r = PL.rel2(PL.gpu_matvec(H, x), PL.oracle_matvec_on_export(ex, lay, x))
assert r <= 1e-12, r
print("big-path ok", st, r)
'''
    env = dict(os.environ, HH_BIG_FLOPS="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "big-path ok" in out.stdout


def test_degenerate_sizes_and_duplicates():
    """N = 1 and N = 2 (single leaf: the dense diagonal block, K(x,x) = 0 for singular
    kernels and 1 for exp); duplicated points beyond 62 key bits -> HH_EDEPTH;
    a duplicate pair inside a leaf is a zero entry for singular kernels (reading G18)."""
    for kern, diag in ((W.K_INV_R, 0.0), (W.K_EXP, 1.0)):
        P1 = np.array([[0.3, 0.4, 0.5]])
        H = PL.gpu_build(P1, dict(kernel=kern, scale=0.1, eps=1e-6, eta=1.0, leaf=8, s=0, pset=W.P_MIXED))
        y = PL.gpu_matvec(H, np.array([[2.0]]))
        assert y[0, 0] == diag * 2.0
        P2 = np.array([[0.0, 0.0, 0.0], [0.3, 0.4, 0.0]])            # distance 0.5
        H = PL.gpu_build(P2, dict(kernel=kern, scale=0.1, eps=1e-6, eta=1.0, leaf=8, s=0, pset=W.P_MIXED))
        y = PL.gpu_matvec(H, np.array([[1.0], [3.0]]))
        off = 2.0 if kern == W.K_INV_R else np.exp(-5.0)
        np.testing.assert_allclose(y[:, 0], [diag * 1.0 + off * 3.0, off * 1.0 + diag * 3.0], rtol=1e-15)
    Pd = np.repeat(np.array([[0.25, 0.5]]), 40, axis=0)
    with pytest.raises(hh.HHError) as e:
        PL.gpu_build(Pd, dict(kernel=W.K_LOG, scale=1.0, eps=1e-6, eta=1.0, leaf=16, s=0, pset=W.P_MIXED))
    assert e.value.status == hh.HH_EDEPTH
    Pp = W.points_uniform(500, 2, 4)
    Pp[7] = Pp[3]                                                    # coincident distinct points
    cfg = dict(kernel=W.K_LOG, scale=1.0, eps=1e-8, eta=1.0, leaf=32, s=2, pset=W.P_MIXED)
    H = PL.gpu_build(Pp, cfg)
    x = W.rhs(500, 1, 5, "uniform_pm1")
    A = D.dense_matrix(Pp, W.K_LOG, 1.0)
    assert A[3, 7] == 0.0 and A[7, 3] == 0.0
    assert PL.rel2(PL.gpu_matvec(H, x), A @ x) < 1e-7


def test_row_split_phase1_matches_oracle():
    """Phase-1 row splitting (partial column sums + fixed-order combine) forced on every W
    tile taller than 40 rows with HH_P1_ROWS; results within 1e-12 of the oracle's Alg. 3 on
    the exported factors, bitwise reproducible, for nrhs = 1, 3 (DFMA) and 16 (DMMA)."""
    import subprocess
    import sys
    code = r'''
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, workloads as W, parity_lib as PL
for name in ("2d_tiny", "3d_small_exp"):
    cfg = W.SMALL_CONFIGS[name]
    P = W.make_points(cfg)
    H = PL.gpu_build(P, cfg)
    ex = PL.export(H)
    lay = PL.check_packing(ex)
    for nrhs in (1, 3, 16):
        x = W.make_rhs(cfg, nrhs)
        y = PL.gpu_matvec(H, x)
        assert np.array_equal(y, PL.gpu_matvec(H, x))
        yo = PL.oracle_matvec_on_export(ex, lay, x)
        for c in range(nrhs):
            r = PL.rel2(y[:, c], yo[:, c])
            assert r <= 1e-12, (name, nrhs, c, r)
print("row-split ok")
'''
    env = dict(os.environ, HH_P1_ROWS="40")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "row-split ok" in out.stdout


def test_planned_product_alternative_stage_geometry_matches_oracle():
    """The single-RHS product streams a stage plan precomputed at hh_build (DESIGN.md §4/§5);
    its second stage geometry (4 stages of 16 KiB, HH_MV_GEOM1/2 = 1) is an A/B variant of the
    product build: the same results within 1e-12 of the oracle's Alg. 3 on the exported factors,
    bitwise reproducible, also through the row-split phase 1 and in every phase combination."""
    import subprocess
    import sys
    code = r'''
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, workloads as W, parity_lib as PL
for name in ("2d_fig8_e4", "3d_small_exp", "3d_sphere_small"):
    cfg = W.SMALL_CONFIGS[name]
    P = W.make_points(cfg)
    H = PL.gpu_build(P, cfg)
    ex = PL.export(H)
    lay = PL.check_packing(ex)
    x = W.make_rhs(cfg, 1)
    y = PL.gpu_matvec(H, x)
    assert np.array_equal(y, PL.gpu_matvec(H, x))
    yo = PL.oracle_matvec_on_export(ex, lay, x)
    r = PL.rel2(y[:, 0], yo[:, 0])
    assert r <= 1e-12, (name, r)
print("geometry ok")
'''
    for g1, g2, rows in (("1", "1", None), ("1", "0", None), ("0", "1", None), ("1", "1", "40")):
        env = dict(os.environ, HH_MV_GEOM1=g1, HH_MV_GEOM2=g2)
        if rows:
            env["HH_P1_ROWS"] = rows
        out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "geometry ok" in out.stdout


def test_switch_level_search_matches_oracle():
    """NEXT-2: Alg. 5 on ledger-only builds equals the oracle's walk on its
    own builds — the same ell* and the same storage at every visited level (bits-aware)."""
    from oracle import switch_level as SL
    P = W.points_uniform(1500, 2, 31)
    args = (W.K_LOG, 1.0, 1e-6, 1.0, 24, W.P_MIXED)
    ell_o, L, by_o = SL.alg_lstar(P, *args)
    Pd = torch.from_numpy(P).cuda()
    ell_g, by_g = hh.hh_switch_level_search(Pd, *args)
    assert len(by_g) == L + 2
    assert ell_g == ell_o and by_g == by_o, (ell_g, ell_o, by_g, by_o)


def test_tie_rule_parity():
    """NEXT-3 HH_TIE_FP16: same partition, ranks, tags (fp16 where the paper's rule says
    bf16), packing and matvec as the oracle with the same flag."""
    cfg = dict(W.SMALL_CONFIGS["2d_fig8_e2"])
    cfg["pset"] = cfg["pset"] | W.TIE_FP16
    P = W.make_points(cfg)
    H = PL.gpu_build(P, cfg)
    ex = PL.export(H)
    Ho = PL.oracle_build(P, cfg)
    PL.check_partition(ex, Ho)
    bad_r, bad_t, st = PL.rank_tag_parity(ex, Ho)
    assert bad_r == 0 and bad_t == 0, st
    B = ex["blocks"]
    assert np.sum((B["storage"] == 0) & (B["tag"] == 3)) == 0 and np.sum(B["tag"] == 2) > 0
    lay = PL.check_packing(ex)
    x = W.make_rhs(cfg, 2)
    assert PL.rel2(PL.gpu_matvec(H, x), PL.oracle_matvec_on_export(ex, lay, x)) <= 1e-12


def test_host_buffer_entry_point_matches_device_path():
    """hh_matvec_host (the e2e path bench.py times: H2D of x, matvec, D2H of y on the stream)
    returns bitwise the device-buffer result, for nrhs = 1 and a 16 + 4 chunked 20."""
    cfg = W.SMALL_CONFIGS["3d_small_exp"]
    P = W.make_points(cfg)
    H = PL.gpu_build(P, cfg)
    for nrhs in (1, 20):
        x = W.make_rhs(cfg, nrhs)
        yd = PL.gpu_matvec(H, x)
        yh = hh.hh_matvec_host(H, np.asfortranarray(x))
        assert np.array_equal(np.asarray(yh).reshape(yd.shape, order="F"), yd)


def test_beneficial_rule_parity_pure_hs_mixed():
    """PAPER.md:992 on the device: mixed pure H_s (2D log, eps=1e-8, leaf 16) keeps some leaf
    neighbours dense and compresses others; storage kind, rank and tag of every block equal the
    oracle's (no unexplained storage difference), and the matvec matches on the exported data."""
    P = W.points_uniform(1500, 2, 12)
    cfg = dict(kernel=W.K_LOG, scale=1.0, eps=1e-8, eta=1.0, leaf=16, s=PT.SWITCH_NONE, pset=W.P_MIXED)
    H = PL.gpu_build(P, cfg)
    ex = PL.export(H)
    Ho = PL.oracle_build(P, cfg)
    PL.check_partition(ex, Ho)
    bad_r, bad_t, st = PL.rank_tag_parity(ex, Ho)
    assert bad_r == 0 and bad_t == 0, st
    B = ex["blocks"]
    ln = B["kind"] == PT.LNBR
    assert np.sum(ln & (B["storage"] == 1)) > 100 and np.sum(ln & (B["storage"] == 0)) > 100, st
    assert st["storage_diff"] == 0, st
    lay = PL.check_packing(ex)
    x = W.rhs(1500, 3, 4, "uniform_pm1")
    assert PL.rel2(PL.gpu_matvec(H, x), PL.oracle_matvec_on_export(ex, lay, x)) <= 1e-12


@pytest.mark.parametrize("scale,kernel,pset", [(1e-20, W.K_INV_R2, W.P_MIXED),
                                               (1e-3, W.K_INV_R, W.P_FP64 | W.P_FP32 | W.P_FP16),
                                               (1e-3, W.K_INV_R, W.P_FP64 | W.P_FP16)])
def test_range_guard_promotion_parity(scale, kernel, pset):
    """Range guard (reading G16): on domains small enough that factor entries overflow the
    16/32-bit formats (1/r^2 ~ 1e40 on 1e-20; 1/r ~ 1e5 on 1e-3), blocks are promoted to the
    next smaller u in the set; the promoted count, every tag and the matvec equal the oracle's."""
    P = W.points_uniform(600, 2, 5) * scale
    cfg = dict(kernel=kernel, scale=1.0, eps=1e-2, eta=1.0, leaf=16, s=2, pset=pset)
    H = PL.gpu_build(P, cfg)
    ex = PL.export(H)
    Ho = PL.oracle_build(P, cfg)
    PL.check_partition(ex, Ho)
    bad_r, bad_t, st = PL.rank_tag_parity(ex, Ho)
    assert bad_r == 0 and bad_t == 0, st
    assert Ho.promoted > 0 and ex["info"]["n_promoted"] == Ho.promoted, (ex["info"]["n_promoted"], Ho.promoted)
    lay = PL.check_packing(ex)
    x = W.rhs(600, 2, 6, "uniform_pm1")
    y = PL.gpu_matvec(H, x)
    assert np.all(np.isfinite(y))
    assert PL.rel2(y, PL.oracle_matvec_on_export(ex, lay, x)) <= 1e-12
