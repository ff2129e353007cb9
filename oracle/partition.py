"""Block partition under standard, weak and hybrid admissibility (oracle).

Standard admissibility, PAPER.md:76-80 (Eq. 2.1):
    adm_s(C_i, C_j)  <=>  min(diam C_i, diam C_j) <= eta * dist(C_i, C_j)
Interaction / neighbour lists; weak admissibility adm_w <=> i != j,
PAPER.md:235-245; hybrid admissibility Eq. 3.1, enumerated as
PAPER.md:552-557 and Alg. 1.

Readings:
  G5  diam/dist are those of the grid boxes: two level-l boxes with integer offset a have
      diam = h sqrt(d) and dist = h sqrt(G), G = sum_k max(0, |a_k| - 1)^2, so
      adm_s <=> d <= eta^2 G  (an exact integer test);
  G6  equality is admissible; eta^2 is snapped to the nearest integer when within 1e-12
      relative (sqrt(3)^2 = 2.9999999999999996 must not reject ties);
  G7  switch level s in [0, L] is Eq. 3.1 read literally: levels < s standard, level s
      every non-self child pair of an inadmissible parent is a block (far if adm_s, else
      "finer neighbour"), levels > s weak (siblings).  s = NONE (-1) is Alg. 1 with
      ell = L kept dense at the leaf (pure H_s): leaf neighbours are dense candidates;
  G8  IL_w = siblings of the self cluster (children of the inadmissible diagonal parent);
  G20 pairs with an empty side are skipped (no storage, no descent).

Block kinds: FAR (IL_s), NBR (finer neighbour at level s), SIB (weak, below s),
LNBR (leaf neighbour of pure H_s), DIAG (leaf self block).  Canonical order: (level,
target Morton code, source Morton code).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tree import Tree, demorton

FAR, NBR, SIB, LNBR, DIAG = 0, 1, 2, 3, 4
KIND_NAMES = {FAR: "far", NBR: "nbr", SIB: "sib", LNBR: "lnbr", DIAG: "diag"}
SWITCH_NONE = -1


def snap_eta2(eta: float) -> float:
    e2 = eta * eta
    r = float(np.round(e2))
    return r if abs(e2 - r) <= 1e-12 * e2 else e2


def adm_s_offsets(a: np.ndarray, d: int, eta2: float) -> np.ndarray:
    """Standard admissibility of two same-level boxes with integer offset vectors a (..., d)."""
    g = np.maximum(0, np.abs(a) - 1)
    G = np.sum(g * g, axis=-1)
    return d <= eta2 * G


@dataclass
class Partition:
    level: np.ndarray   # int64 [nb]
    kind: np.ndarray    # int64 [nb]
    tgt: np.ndarray     # int64 Morton code of the target cluster at `level`
    src: np.ndarray     # int64 Morton code of the source cluster

    def __len__(self):
        return int(self.level.size)


def build_partition(tree: Tree, eta: float, s: int) -> Partition:
    d, L = tree.d, tree.L
    eta2 = snap_eta2(eta)
    nch = 1 << d
    out = []
    # level 0: the root pair (0,0) is the only pair; it is inadmissible (it is the self pair)
    pi = np.zeros(1, dtype=np.int64)
    pj = np.zeros(1, dtype=np.int64)
    if L == 0:
        out.append((np.zeros(1, np.int64), np.full(1, DIAG), pi, pj))
    for l in range(1, L + 1):
        # children pairs of every inadmissible level-(l-1) pair
        a = np.arange(nch, dtype=np.int64)
        ci = (pi[:, None, None] * nch + a[None, :, None]).repeat(nch, axis=2).ravel()
        cj = (pj[:, None, None] * nch + a[None, None, :]).repeat(nch, axis=1).ravel()
        size = tree.cluster_sizes(l)
        keep = (size[ci] > 0) & (size[cj] > 0)          # G20: skip empty sides
        ci, cj = ci[keep], cj[keep]
        off = demorton(cj, d, l) - demorton(ci, d, l)
        adm = adm_s_offsets(off, d, eta2)
        same = ci == cj
        if s == SWITCH_NONE or l < s:
            blk = adm
            kind = np.full(ci.size, FAR)
        elif l == s:
            blk = ~same
            kind = np.where(adm, FAR, NBR)
        else:  # l > s: weak admissibility
            blk = ~same
            kind = np.full(ci.size, SIB)
        out.append((np.full(int(blk.sum()), l), kind[blk], ci[blk], cj[blk]))
        inad = ~blk
        pi, pj = ci[inad], cj[inad]
        if l == L:
            dk = np.where(pi == pj, DIAG, LNBR)
            out.append((np.full(pi.size, L), dk, pi, pj))
    level = np.concatenate([o[0] for o in out]).astype(np.int64)
    kind = np.concatenate([o[1] for o in out]).astype(np.int64)
    tgt = np.concatenate([o[2] for o in out]).astype(np.int64)
    src = np.concatenate([o[3] for o in out]).astype(np.int64)
    order = np.lexsort((src, tgt, level))
    return Partition(level=level[order], kind=kind[order], tgt=tgt[order], src=src[order])


def sparsity_constants(part: Partition, s: int, L: int) -> dict:
    """Measured maximum list sizes per target cluster (the C_sp of PAPER.md:886-894).

    c1 = max |IL_s| over levels with standard admissibility, c2 = max |N_s| at the
    switch level (finer neighbours; for pure H_s the leaf neighbours), c3 = max |IL_w|.
    """
    def maxcount(mask):
        if not np.any(mask):
            return 0
        lv = part.level[mask]
        tg = part.tgt[mask]
        pairs = np.stack([lv, tg], axis=1)
        _, counts = np.unique(pairs, axis=0, return_counts=True)
        return int(counts.max())
    return dict(c1=maxcount(part.kind == FAR),
                c2=maxcount((part.kind == NBR) | (part.kind == LNBR)),
                c3=maxcount(part.kind == SIB))
