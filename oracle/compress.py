"""LRcompression = truncated SVD to relative Frobenius accuracy eps (oracle).

PAPER.md:62-68: ||H_IJ - U_I V_J^*|| <= eps ||H_IJ|| (Frobenius);
PAPER.md:68, 1121: "the truncated SVD is employed"; Alg. 4 takes
||H~_IJ||^2 = trace(Sigma~^2) of the kept singular values.

Reading G10: p = min{p : sum_{k>p} sigma_k^2 <= eps^2 sum_k sigma_k^2}, the tail summed
from the smallest singular value upward (never as a difference ||A||^2 - sum_{k<=p}, which
cancels catastrophically); equality keeps the smaller p; a zero block
gives p = 0.  Reading G11: U keeps orthonormal columns, W = V Sigma carries the scale.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def svd(A: np.ndarray, driver: str = "gesdd"):
    return scipy.linalg.svd(A, full_matrices=False, lapack_driver=driver)


def truncation_rank(sigma: np.ndarray, eps: float) -> tuple[int, float, float, float]:
    """Return (p, tail_p, total, margin) for descending singular values ``sigma``.

    margin = (eps^2 total - tail_p) / (eps^2 total) at the chosen p and its neighbour
    decision, i.e. how far the rank decision is from flipping (used by parity tolerances).
    """
    sq = np.asarray(sigma, dtype=np.float64) ** 2
    r = sq.size
    tails = np.zeros(r + 1)
    tails[:r] = np.cumsum(sq[::-1])[::-1]      # tails[p] = sum_{k >= p} sq[k] (0-based) = sum_{k>p} (1-based)
    total = float(tails[0]) if r else 0.0
    thr = eps * eps * total
    if total == 0.0:
        return 0, 0.0, 0.0, np.inf
    p = int(np.argmax(tails <= thr))           # first p with tail_p <= thr
    # relative distance of the decision from the threshold (both sides of the boundary)
    m_keep = (thr - tails[p]) / thr
    m_prev = (tails[p - 1] - thr) / thr if p > 0 else np.inf
    return p, float(tails[p]), total, float(min(m_keep, m_prev))


def lr_compress(A: np.ndarray, eps: float, driver: str = "gesdd"):
    """Truncated SVD of block A.  Returns dict(p, U, W, nb2, tot, sigma, margin)."""
    if A.size == 0 or not np.any(A):
        m, n = A.shape
        return dict(p=0, U=np.zeros((m, 0)), W=np.zeros((n, 0)), nb2=0.0, tot=0.0,
                    sigma=np.zeros(0), margin=np.inf)
    U, s, Vt = svd(A, driver)
    p, tail, tot, margin = truncation_rank(s, eps)
    nb2 = float(np.sum(s[:p] ** 2))
    return dict(p=p, U=U[:, :p].copy(), W=(Vt[:p].T * s[:p]).copy(), nb2=nb2, tot=tot,
                sigma=s, margin=margin)
