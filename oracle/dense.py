"""Dense kernel matrix products by definition (oracle).  PAPER.md:1114-1119.

(A x)_i = sum_j H_ij x_j by direct summation over all j and ||A||_F^2 = sum_ij H_ij^2,
row-chunked so memory stays bounded.  Also sampled rows for large N.
"""
from __future__ import annotations

import numpy as np

from .kernels import block as kernel_block


def dense_apply(P, kind, scale, x, rows=None, chunk=256):
    """Return ((A x)[rows], ||A[rows,:]||_F^2).  rows=None -> all rows."""
    P = np.asarray(P, dtype=np.float64)
    n = P.shape[0]
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    cols = np.arange(n)
    out = np.zeros((rows.size, x.shape[1]))
    fro2 = 0.0
    for s in range(0, rows.size, chunk):
        r = rows[s:s + chunk]
        A, _ = kernel_block(P, r, cols, kind, scale)
        out[s:s + chunk] = A @ x
        fro2 += float(np.sum(A * A))
    return out, fro2


def dense_matrix(P, kind, scale):
    n = P.shape[0]
    A, _ = kernel_block(np.asarray(P, dtype=np.float64), np.arange(n), np.arange(n), kind, scale)
    return A
