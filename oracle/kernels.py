"""Kernel-matrix entries (oracle).  PAPER.md:1097-1119, Eq. 5.1.

H_ij = f(||x_i - x_j||_2).  "If f is singular, the diagonal entries are set to zero."
Kernels: log r (2D Laplace), 1/r (3D Laplace), 1/r^2,
Gaussian exp(-r^2/2), Matern exp(-r).  BASELINE config 4 uses exp(-r/0.1); reading G19
adds a length scale s: GAUSS = exp(-r^2/(2 s^2)), EXP = exp(-r/s).
Reading G18: the singular-kernel diagonal rule is keyed on index equality (i == j); a
zero distance between two DISTINCT points of a singular kernel also yields 0 and is
counted (``coincident`` in the return value).
"""
from __future__ import annotations

import numpy as np

K_LOG, K_INV_R, K_INV_R2, K_GAUSS, K_EXP = 0, 1, 2, 3, 4
SINGULAR = {K_LOG, K_INV_R, K_INV_R2}


def f_of_r(kind: int, r: np.ndarray, scale: float) -> np.ndarray:
    with np.errstate(divide="ignore", invalid="ignore"):
        if kind == K_LOG:
            return np.log(r)
        if kind == K_INV_R:
            return 1.0 / r
        if kind == K_INV_R2:
            return 1.0 / (r * r)
        if kind == K_GAUSS:
            return np.exp(-(r * r) / (2.0 * scale * scale))
        if kind == K_EXP:
            return np.exp(-r / scale)
    raise ValueError(kind)


def block(P: np.ndarray, rows: np.ndarray, cols: np.ndarray, kind: int, scale: float):
    """Dense block H[rows, cols] for original point indices rows/cols.  Returns (A, coincident)."""
    X = P[rows]
    Y = P[cols]
    diff = X[:, None, :] - Y[None, :, :]
    r = np.sqrt(np.sum(diff * diff, axis=2))
    A = f_of_r(kind, r, scale)
    same = rows[:, None] == cols[None, :]
    coincident = 0
    if kind in SINGULAR:
        zero = (r == 0.0)
        coincident = int(np.count_nonzero(zero & ~same))
        A[zero] = 0.0
    else:
        A[same] = f_of_r(kind, np.zeros(1), scale)[0]
    return A, coincident
