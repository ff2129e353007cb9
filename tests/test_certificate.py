"""The check-(1b) rank certificate used at full size (tests/parity_lib.py:certify_rank) against
the oracle's LAPACK truncated-SVD rank on real kernel blocks: it certifies exactly the LAPACK
rank and rejects its neighbours.  CPU only."""
import numpy as np

import parity_lib as PL
import workloads as W
from oracle import compress as OC
from oracle import kernels as OK
from oracle import partition as PT
from oracle import tree as T


def test_certificate_agrees_with_lapack_rank():
    cfg = W.CONFIGS["3d_laplace"]
    P = W.points_uniform(32768, 3, 7)
    tr = T.build_tree(P, 128)
    part = PT.build_partition(tr, 1.0, 2)
    rng = np.random.default_rng(1)
    lr = np.nonzero(part.kind != PT.DIAG)[0]
    checked = 0
    for b in rng.choice(lr, 24, replace=False):
        l = int(part.level[b])
        i0, i1 = tr.cluster(l, int(part.tgt[b]))
        j0, j1 = tr.cluster(l, int(part.src[b]))
        A, _ = OK.block(P, tr.perm[i0:i1], tr.perm[j0:j1], W.K_INV_R, 1.0)
        for eps in (1e-6, 1e-3):
            c = OC.lr_compress(A, eps)
            p = c["p"]
            cert = PL.certify_rank(A, p, eps)
            assert cert["valid"] and cert["minimal"], (b, p, cert)
            assert cert["nb2_lower"] <= c["nb2"] * (1 + 1e-12) and c["nb2"] <= cert["nb2_upper"] * (1 + 1e-12)
            assert abs(cert["nb2_lower"] - c["nb2"]) <= 1e-10 * c["nb2"]
            if p > 0:
                assert not PL.certify_rank(A, p - 1, eps)["valid"]          # p - 1 does not meet eps
            assert not PL.certify_rank(A, p + 1, eps)["minimal"]            # p + 1 is not minimal
            checked += 1
    assert checked == 48
    assert cfg["kernel"] == W.K_INV_R
