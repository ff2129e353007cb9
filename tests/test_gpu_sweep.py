"""BASELINE config 4 — admissibility sweep at full size (N=262144, 3D 1/r, leaf 128, eta=1,
eps=1e-6): switch level in {none (pure standard H), 2, 3, 4, 0 (pure HODLR)} in adaptive mixed
precision, plus uniform fp64 at s=2.  Per setting, through the C-ABI: (1a) the whole block
table against the oracle's partition, (1c) every packing offset against the oracle's packing
function, (2) complete rows of a sampled leaf against the oracle's Alg. 3 on the exported
factors (<= 1e-12), (3) sampled-row e_mv <= 10 eps.  Also the special-case identities the
paper fixes: s=none has the standard-H partition (dense leaf neighbours or
beneficial low-rank ones), s=0 is HODLR (weak admissibility at every level)."""
import numpy as np
import pytest

import workloads as W
from oracle import dense as D
from oracle import pack as PK
from oracle import partition as PT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import parity_lib as PL  # noqa: E402
from paper_2604_09147_b200 import hh  # noqa: E402

SETTINGS = [(s, W.P_MIXED) for s in W.SWEEP_SWITCH_LEVELS] + [(2, W.P_FP64)]


@pytest.fixture(scope="module")
def sweep_inputs():
    cfg = W.CONFIGS["sweep"]
    P = W.make_points(cfg)
    x = W.make_rhs(cfg, 1)
    rng = np.random.default_rng(9)
    rows = rng.choice(cfg["N"], size=48, replace=False)
    Ax, fro2_rows = D.dense_apply(P, cfg["kernel"], cfg["scale"], x, rows=rows, chunk=8)
    return cfg, P, x, rows, Ax, fro2_rows


@pytest.mark.parametrize("s,pset", SETTINGS, ids=[f"s{s}-p{p}" for s, p in SETTINGS])
def test_sweep_setting(sweep_inputs, s, pset):
    cfg0, P, x, rows, Ax, fro2_rows = sweep_inputs
    cfg = dict(cfg0, s=s, pset=pset)
    H = PL.gpu_build(P, cfg)
    try:
        ex = PL.export(H, arenas=False)
        tr, part = PL.oracle_partition(P, cfg)
        B = ex["blocks"]
        # (1a)
        np.testing.assert_array_equal(ex["perm"].astype(np.int64), tr.perm)
        for f, ref in (("level", part.level), ("kind", part.kind), ("tgt", part.tgt), ("src", part.src)):
            np.testing.assert_array_equal(B[f].astype(np.int64), ref, err_msg=f)
        if s == 0:
            assert set(np.unique(B["kind"])) <= {PT.SIB, PT.DIAG}
        if s == PT.SWITCH_NONE:
            assert set(np.unique(B["kind"])) <= {PT.FAR, PT.LNBR, PT.DIAG}
            ln = B["kind"] == PT.LNBR
            if pset == W.P_FP64:
                assert np.all(B["storage"][ln] == 1)
        # (1c)
        PL.check_packing(ex)
        lay = PK.pack(ex["leaf_start"], tr.d, tr.L, B["level"], B["tgt"], B["src"], B["rank"], B["tag"],
                      B["storage"])
        # (2) one sampled leaf, complete rows
        y = PL.gpu_matvec(H, x)
        nonempty = np.nonzero(np.diff(tr.leaf_start) > 0)[0]
        R = int(np.random.default_rng(3).choice(nonempty))
        r0, r1 = int(tr.leaf_start[R]), int(tr.leaf_start[R + 1])
        yo = PL.oracle_leaf_rows(H, B, lay, tr, R, x[tr.perm])
        assert PL.rel2(y[tr.perm[r0:r1], 0], yo[:, 0]) <= 1e-12
        # (3)
        e = np.sqrt(np.sum((Ax[:, 0] - y[rows, 0]) ** 2) / fro2_rows) / np.linalg.norm(x)
        assert e <= 10 * cfg["eps"], e
    finally:
        hh.hh_free(H)
