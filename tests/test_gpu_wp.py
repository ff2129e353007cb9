"""NEXT-3 working precision on the device (hh_matvec_wp, reading G27) against the oracle twin
(oracle/matvec_wp.py), and the paper's backward-error experiment (Fig. 9;
Thm 4.4 at PAPER.md:1028-1040).  Needs a B200.

Parity of a reduced-precision product cannot be bitwise (the paper fixes no summation order and
the device sums in its own fixed order), so both results are checked against what is unique:
the exact product y* of the working-precision-rounded operands, within the a priori rounding
bound of any summation order — gamma_{K + n_J}(u) |U| |W|^T |x| componentwise for fp32
(deterministic, Higham §3.1) and the probabilistic gamma~(lambda = 8) for fp16 (Higham & Mary
2019), K = terms accumulated into the row, n_J = longest source cluster feeding it.  The data
path is the fp64 product's (the same templated kernels), which check (2) pins to 1e-12."""
import numpy as np
import pytest

import workloads as W
from oracle import dense as D
from oracle import matvec_wp as OW
from oracle import metrics as M

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import parity_lib as PL  # noqa: E402
from paper_2604_09147_b200 import hh  # noqa: E402

U = {OW.WP_FP32: 2.0 ** -24, OW.WP_FP16: 2.0 ** -11}


def gpu_matvec_wp(H, x, wp):
    xd = torch.from_numpy(np.asfortranarray(x).reshape(x.shape[0], -1, order="F").T.copy()).cuda().T
    yd = torch.empty_like(xd.T).T
    hh.hh_matvec_wp(H, xd, yd, wp, xd.shape[1])
    torch.cuda.synchronize()
    return yd.cpu().numpy()


@pytest.fixture(scope="module", params=["2d_tiny", "3d_small_inv_r", "2d_fig8_e2_q43", "3d_small_exp"])
def built(request):
    cfg = W.SMALL_CONFIGS[request.param]
    P = W.make_points(cfg)
    H = PL.gpu_build(P, cfg)
    ex = PL.export(H)
    lay = PL.check_packing(ex)
    blocks = list(PL.exported_blocks(ex, lay))
    return request.param, cfg, P, H, ex, blocks


def test_wp_fp64_is_the_product_path(built):
    name, cfg, P, H, ex, blocks = built
    x = W.make_rhs(cfg, 3)
    assert np.array_equal(gpu_matvec_wp(H, x, OW.WP_FP64), PL.gpu_matvec(H, x))


@pytest.mark.parametrize("wp", [OW.WP_FP32, OW.WP_FP16])
def test_wp_within_rounding_bound_of_rounded_operand_product(built, wp):
    name, cfg, P, H, ex, blocks = built
    N = ex["info"]["N"]
    perm = ex["perm"].astype(np.int64)
    for nrhs in (1, 3, 6):            # chunk widths 1; 2 + 1; 4 + 2
        x = W.make_rhs(cfg, nrhs)
        y = gpu_matvec_wp(H, x, wp)
        assert np.array_equal(y, gpu_matvec_wp(H, x, wp))          # deterministic
        r = OW.rounded_operand_product(N, perm, blocks, x, wp)
        k = (r["K"] + r["nJ"])[:, None]
        g = OW.gamma(k, U[wp]) if wp == OW.WP_FP32 else OW.gamma_prob(k, U[wp])
        err = np.abs(y - r["y"])
        assert np.all(err <= g * r["S"]), (name, wp, nrhs, float(np.max(err / (g * r["S"]))))
        assert np.max(err / np.maximum(r["S"], 1e-300)) > U[wp] / 8     # arithmetic really was reduced
        # y holds working-precision values
        y_wp = OW.to_wp(y, wp).astype(np.float64)
        assert np.array_equal(y_wp, y)
    # the oracle twin (plain sequential order, separate rounded * and +) satisfies the same bound
    x = W.make_rhs(cfg, 1)
    yo = OW.matvec_blocks_wp(N, perm, blocks, x, wp)
    r = OW.rounded_operand_product(N, perm, blocks, x, wp)
    k = (r["K"] + r["nJ"])[:, None]
    g = OW.gamma(k, U[wp]) if wp == OW.WP_FP32 else OW.gamma_prob(k, U[wp])
    assert np.all(np.abs(yo - r["y"]) <= g * r["S"])
    # and both sit at the same distance from the exact product of the rounded operands
    eg = np.linalg.norm(gpu_matvec_wp(H, x, wp) - r["y"]) / np.linalg.norm(r["y"])
    eo = np.linalg.norm(yo - r["y"]) / np.linalg.norm(r["y"])
    assert eg <= 4 * eo + 4 * U[wp] and eo <= 16 * eg + 4 * U[wp], (eg, eo)


def test_wp_row_split_and_promotion_paths():
    """Reduced working precision through the row-split phase 1 (fixed-order combine in the
    working format) — subprocess with HH_P1_ROWS, bound as above."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, workloads as W, parity_lib as PL, test_gpu_wp as T
from oracle import matvec_wp as OW
cfg = W.SMALL_CONFIGS["3d_small_exp"]
P = W.make_points(cfg)
H = PL.gpu_build(P, cfg)
ex = PL.export(H); lay = PL.check_packing(ex); blocks = list(PL.exported_blocks(ex, lay))
for wp in (OW.WP_FP32, OW.WP_FP16):
    x = W.make_rhs(cfg, 3)
    y = T.gpu_matvec_wp(H, x, wp)
    r = OW.rounded_operand_product(ex["info"]["N"], ex["perm"].astype(np.int64), blocks, x, wp)
    k = (r["K"] + r["nJ"])[:, None]
    g = OW.gamma(k, T.U[wp]) if wp == OW.WP_FP32 else OW.gamma_prob(k, T.U[wp])
    assert np.all(np.abs(y - r["y"]) <= g * r["S"]), wp
print("wp row-split ok")
'''
    env = dict(os.environ, HH_P1_ROWS="40")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "wp row-split ok" in out.stdout


def test_backward_error_experiment_fig9_8000():
    """PAPER.md:1269-1285 (Fig. 9a): 3D 1/r, N = 8000 on [-1,1]^3, L = 2, ell = L - 1,
    x ~ U(0,1); relative backward error ||Hx - b|| / (||H|| ||x||) of the adaptive mixed-
    precision H_h product computed in fp64 / fp32 / fp16, over eps = 1e-2 .. 1e-10.  The paper's
    conclusions, checked: (i) with u <~ eps (Thm 4.4's hypothesis) the error obeys Thm 4.4's
    bound (measured sparsity constants); (ii) fp64 stays at the approximation error at every eps
    (check (3)); (iii) a working precision coarser than eps / N puts a floor under the error
    (fp16 ~ 1e-3 at every eps, fp32 ~ 1e-7 from eps = 1e-6 down) while fp32 matches fp64 where
    u_32 << eps / N — 'one should choose the working precision u <~ eps (more precisely
    u <~ eps / N)'."""
    cfg0 = W.FIG9_CONFIGS["3d_fig9_8000"]
    P = W.make_points(cfg0)
    x = W.make_rhs(cfg0, 1)
    Ax, fro2 = D.dense_apply(P, cfg0["kernel"], cfg0["scale"], x)
    N = cfg0["N"]
    table = {}
    for eps in W.FIG9_EPS:
        cfg = dict(cfg0, eps=eps)
        H = PL.gpu_build(P, cfg)
        info = hh.hh_info(H)
        assert info["L"] == 2
        bound = M.thm44_factor(info["L"], cfg["s"], info["c_far"], info["c_nbr"], info["c_sib"]) * eps
        row = {}
        for wp in (OW.WP_FP64, OW.WP_FP32, OW.WP_FP16):
            y = gpu_matvec_wp(H, x, wp)
            row[wp] = float(M.e_mv(Ax, y, np.sqrt(fro2), x)[0])
            u = {OW.WP_FP64: 2.0 ** -53, **U}[wp]
            if u <= eps:      # Thm 4.4's hypothesis u <~ eps
                assert row[wp] <= bound, (eps, wp, row[wp], bound)
        table[eps] = row
        hh.hh_free(H)
    print("Fig. 9a reproduction (e_mv by eps and working precision fp64/fp32/fp16):",
          {e: [f"{r[w]:.2e}" for w in (0, 1, 2)] for e, r in table.items()})
    for eps, r in table.items():
        assert r[OW.WP_FP64] <= 10 * eps                                   # check (3) at fp64
    assert table[1e-6][OW.WP_FP16] > 10 * table[1e-6][OW.WP_FP64]        # fp16 floor
    assert table[1e-10][OW.WP_FP32] > 10 * table[1e-10][OW.WP_FP64]      # fp32 floor
    for eps in (1e-2, 1e-4):                                              # u_32 << eps / N: no effect
        assert table[eps][OW.WP_FP32] <= 1.01 * table[eps][OW.WP_FP64]
