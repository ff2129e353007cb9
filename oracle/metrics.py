"""Error metrics and the paper's bounds (oracle).

e_mv  = ||A x - y||_2 / (||A||_F ||x||_2)             PAPER.md:1269 (backward-error plot)
e_glob = ||H - H-hat||_F / ||H||_F
Thm 4.2:  e_glob <~ (2 sqrt(ell C' + C'' + (L - ell) C''') + 1) eps
Thm 4.4: ||Delta H|| <= 2 (2 sqrt(...) + 1) eps ||H||
List-size constants:
    C' = (2^d - 1)(1 + 2 sqrt(d)/eta)^d,  C'' = (1 + 2 sqrt(d)/eta)^d - 1,  C''' = 2^d - 1.
Reading G21: at eta != sqrt(d) these are not upper bounds on the integer grid, so the
bounds are also evaluated with the MEASURED sparsity constants (PAPER.md:886-894 is where
the proof uses them), and in the pre-constant block-count form of PAPER.md:884-885:
    ||H~ - H-hat||^2 <~ sum_b 4 eps^2 / 2^{d l_b} ||H~||^2.
"""
from __future__ import annotations

import numpy as np

from .kernels import block as kernel_block
from .partition import DIAG, LNBR


def list_constants(d: int, eta: float) -> tuple[float, float, float]:
    c = (1.0 + 2.0 * np.sqrt(d) / eta) ** d
    return (2 ** d - 1) * c, c - 1.0, float(2 ** d - 1)


def thm42_factor(L: int, ell: int, c1: float, c2: float, c3: float) -> float:
    return 2.0 * np.sqrt(ell * c1 + c2 + (L - ell) * c3) + 1.0


def thm44_factor(L, ell, c1, c2, c3) -> float:
    return 2.0 * thm42_factor(L, ell, c1, c2, c3)


def blockcount_factor(levels, d: int) -> float:
    """2 sqrt(sum_b 2^{-d l_b}) + 1 over the low-rank blocks (pre-constant form)."""
    levels = np.asarray(levels, dtype=np.float64)
    return 2.0 * np.sqrt(np.sum(2.0 ** (-d * levels))) + 1.0


def e_mv(Ax, y, fro_A, x):
    """Per-column relative backward error ||Ax - y|| / (||A||_F ||x||)."""
    Ax = np.atleast_2d(np.asarray(Ax).T).T
    y = np.atleast_2d(np.asarray(y).T).T
    x = np.atleast_2d(np.asarray(x).T).T
    return np.linalg.norm(Ax - y, axis=0) / (fro_A * np.linalg.norm(x, axis=0))


def global_error_sq(H, P, use_rounded=True):
    """||H - H-hat||_F^2 blockwise (dense blocks are exact in fp64) and ||H||_F^2."""
    err2 = 0.0
    fro2 = 0.0
    for b in range(len(H.part)):
        i0, i1, j0, j1 = H.rows(b)
        A, _ = kernel_block(P, H.tree.perm[i0:i1], H.tree.perm[j0:j1], H.kernel, H.scale)
        fro2 += float(np.sum(A * A))
        if b in H.factors:
            U, W = H.factors[b] if use_rounded else H.exact[b]
            E = A - U @ W.T
            err2 += float(np.sum(E * E))
    return err2, fro2


def ell_of(H) -> int:
    return H.tree.L if H.s < 0 else H.s


def lowrank_levels(H):
    return np.array([int(H.part.level[b]) for b in H.factors], dtype=np.int64)


def is_dense_kind(k):
    return k in (DIAG, LNBR)
