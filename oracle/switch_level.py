"""Alg. 5 — switching-level search (oracle).  PAPER.md:726-749 (alg:algo_optimal_level).

S_s = L + S_1(ell) + D (Eq. storage_Hs) and S_h(ell) = L + S_2(ell) + D
(Eq. storage_Hh) share the low-rank storage L up to level ell and the
leaf diagonal D, so S_1(ell) - S_2(ell) = S_s - S_h(ell).  The algorithm:

    ell <- L, s <- S_1(L) - S_2(L) = 0              (the ell = L branch of Alg. 1 is H_s)
    while ell > 0:
        s_new <- S_1(ell-1) - S_2(ell-1)
        if s_new <= s: break
        s <- s_new, ell <- ell - 1
    ell* <- ell

Storage is counted in each block's storage bits (stored_bytes), which with a precision set
of {fp64} is the paper's uniform-precision count and otherwise the bits-aware variant the
paper leaves open.  S_h(ell) for ell < L is the H_h of Eq. 3.1 with switch
level ell; S_s is the pure standard H (switch NONE).  Test infrastructure only.
"""
from __future__ import annotations

from . import hmatrix as HM
from .partition import SWITCH_NONE


def walk(L: int, S_s: int, S_h) -> tuple[int, list]:
    """Alg. 5's bottom-up walk given S_s and a callable S_h(ell) for
    ell < L.  Returns (ell*, bytes) with bytes[l] = S_h(l) for the visited levels (-1
    otherwise) and bytes[L] = bytes[L+1] = S_s."""
    out = [-1] * (L + 2)
    out[L] = out[L + 1] = S_s
    ell, s = L, 0                       # S_1(L) - S_2(L) = 0: the ell = L branch is H_s
    while ell > 0:
        Sh = S_h(ell - 1)
        out[ell - 1] = Sh
        s_new = S_s - Sh                # S_1(ell-1) - S_2(ell-1)
        if s_new <= s:
            break
        s, ell = s_new, ell - 1
    return ell, out


def alg_lstar(P, kernel, scale, eps, eta, leaf, pset):
    """Returns (ell*, L, bytes) with bytes[l] = S_h(l) for the visited levels (-1 otherwise)
    and bytes[L] = bytes[L+1] = S_s."""
    Hs = HM.build(P, kernel, scale, eps, eta, leaf, SWITCH_NONE, pset)
    L = Hs.tree.L
    Ss = HM.stored_bytes(Hs)["total"]
    ell, out = walk(L, Ss, lambda l: HM.stored_bytes(HM.build(P, kernel, scale, eps, eta, leaf, l, pset))["total"])
    return ell, L, out
