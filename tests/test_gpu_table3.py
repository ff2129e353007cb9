"""Table 3 of the paper reproduced on the GPU with ledger-only builds:
S_1(ell)/S_2(ell) at ell = L-1 for 3D 1/r, N=64000 uniform in [-1,1]^3, L=3, eta=sqrt(3),
uniform fp64 (words).  S_1 = H_s storage beyond level ell (level-3 far blocks low-rank +
dense leaf neighbours, Eq. S1); S_2 = H_h storage beyond ell (level-ell finer
neighbours + weak siblings below, Eq. S2).  The printed ratios are
1.62 / 1.59 / 1.59 / 1.60 / 2.00 / 3.65 for eps = 1e-12 ... 1e-2; the point seed is unstated,
so the pin is a band around 1.60 at eps = 1e-6; the other ratios are
printed into profiles by scripts and checked only for the paper's qualitative trend
(S_1/S_2 > 1 everywhere, largest at eps = 1e-2)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2604_09147_b200 import hh  # noqa: E402

FAR, NBR, SIB, LNBR = 0, 1, 2, 3
PAPER = {1e-12: 1.62, 1e-10: 1.59, 1e-8: 1.59, 1e-6: 1.60, 1e-4: 2.00, 1e-2: 3.65}


def _words(H):
    ex = hh.hh_export(H, tables=True, arenas=False)
    B, ls, info = ex["blocks"], ex["leaf_start"], ex["info"]
    sh = info["d"] * (info["L"] - B["level"].astype(np.int64))
    m = ls[(B["tgt"] + 1) << sh] - ls[B["tgt"] << sh]
    n = ls[(B["src"] + 1) << sh] - ls[B["src"] << sh]
    return B, m, n, info["L"]


def test_table3_ratios():
    P = torch.from_numpy(W.points_uniform(64000, 3, 64000, -1.0, 1.0)).cuda()
    eta, leaf = float(np.sqrt(3.0)), 250   # the depth rule gives L = 3 (max leaf ~170; the paper: 125 balanced)
    ratios = {}
    for eps in PAPER:
        Hs = hh.hh_build(P, W.K_INV_R, 1.0, eps, eta, leaf, W.SWITCH_NONE, W.P_FP64 | hh.LEDGER_ONLY)
        B, m, n, L = _words(Hs)
        assert L == 3
        ell = L - 1
        p = B["rank"].astype(np.int64)
        S1 = int(np.sum((p * (m + n))[(B["level"] > ell) & (B["kind"] == FAR)])) + int(np.sum((m * n)[B["kind"] == LNBR]))
        Hh = hh.hh_build(P, W.K_INV_R, 1.0, eps, eta, leaf, ell, W.P_FP64 | hh.LEDGER_ONLY)
        B, m, n, _ = _words(Hh)
        p = B["rank"].astype(np.int64)
        sel = ((B["level"] == ell) & (B["kind"] == NBR)) | ((B["level"] > ell) & (B["kind"] == SIB))
        S2 = int(np.sum((p * (m + n))[sel]))
        ratios[eps] = S1 / S2
    print("Table 3 (L=3) S1/S2:", {k: round(v, 3) for k, v in ratios.items()}, "paper:", PAPER)
    assert 1.45 <= ratios[1e-6] <= 1.75, ratios
    assert all(r > 1.0 for r in ratios.values())
    assert ratios[1e-2] == max(ratios.values())
