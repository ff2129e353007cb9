"""Alg. 3: b = H-hat x (oracle).  PAPER.md:1042-1082.

b <- 0; for every admissible block (levels 1..ell standard, level ell finer neighbours,
levels ell+1..L weak): b_I <- b_I + U-hat_I (V-hat_J^* x_J); for every leaf:
b_I <- b_I + H-hat_II x_I; "compute in working precision u" (fp64 here, reading G22).
Stored low-precision factors enter as their exact float64 values (exact up-conversion).
Blocks are visited in canonical order (level, target, source).
"""
from __future__ import annotations

import numpy as np


def matvec_blocks(n, perm, blocks, x):
    """Generic Alg. 3 over a list of blocks.

    blocks: iterable of (i0, i1, j0, j1, kind, payload) in tree positions where
    kind == "lr" -> payload = (U, W) (b_I += U (W^T x_J)), kind == "dense" -> payload = D.
    x: (n, nrhs) in ORIGINAL point order.  Returns y (n, nrhs) in original order.
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    xt = x[perm]                      # tree order
    yt = np.zeros_like(xt)
    for i0, i1, j0, j1, kind, payload in blocks:
        if kind == "lr":
            U, W = payload
            if U.shape[1] == 0:
                continue
            yt[i0:i1] += U @ (W.T @ xt[j0:j1])
        else:
            yt[i0:i1] += payload @ xt[j0:j1]
    y = np.empty_like(yt)
    y[perm] = yt
    return y


def matvec(H, x):
    """Alg. 3 on an oracle-built H (hmatrix.OracleH)."""
    def gen():
        for b in range(len(H.part)):
            i0, i1, j0, j1 = H.rows(b)
            if b in H.factors:
                yield i0, i1, j0, j1, "lr", H.factors[b]
            elif b in H.dense:
                yield i0, i1, j0, j1, "dense", H.dense[b]
    return matvec_blocks(H.n, H.tree.perm, gen(), x)
