"""Balanced 2^d-tree (oracle).  PAPER.md:55-57.

"Each hypercube C_i^(l) at level l < L is partitioned into 2^d finer hypercubes ...
The partitioning continues recursively up to level L (the leaf level), where each leaf
hypercube contains at most n_max particles."

Readings: G1 depth = smallest L with every leaf holding <= n_max points;
G2 root hypercube = bounding cube of the points (lo_k = min_i x_ik, side = largest
extent); G3 half-open cells via the floor formula, top face clamped into the last cell;
G4 Morton digit order with axis 0 as the least significant bit of each d-bit digit,
points inside a leaf ordered by original index.

A cluster (l, m) is the set of points whose depth-L Morton key, shifted right by
d*(L-l) bits, equals m; in tree (Morton) order it is a contiguous index range.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MAX_KEY_BITS = 62


def root_cube(P: np.ndarray) -> tuple[np.ndarray, float]:
    """lo_k = min_i x_ik; side = max_k (max_i x_ik - lo_k); side := 1 if all points coincide."""
    lo = P.min(axis=0)
    side = float((P.max(axis=0) - lo).max())
    if side == 0.0:
        side = 1.0
    return lo, side


def cells(P: np.ndarray, lo: np.ndarray, side: float, L: int) -> np.ndarray:
    """Integer cell coordinates at depth L: c_k = min(2^L - 1, floor(ldexp((x_k - lo_k)/side, L)))."""
    t = (P - lo) / side                      # IEEE subtract then divide (no contraction)
    c = np.floor(np.ldexp(t, L)).astype(np.int64)
    return np.minimum(c, (1 << L) - 1)


def morton(c: np.ndarray, L: int) -> np.ndarray:
    """Interleave cell coordinates: bit b of axis k goes to key bit b*d + k (axis 0 = LSB
    of each digit); the level-1 digit occupies the most significant d bits."""
    n, d = c.shape
    key = np.zeros(n, dtype=np.int64)
    for b in range(L):
        for k in range(d):
            key |= ((c[:, k] >> b) & 1) << (b * d + k)
    return key


def demorton(key, d: int, l: int) -> np.ndarray:
    """Inverse of ``morton`` for keys of a level-l cluster: returns (..., d) coordinates."""
    key = np.asarray(key, dtype=np.int64)
    c = np.zeros(key.shape + (d,), dtype=np.int64)
    for b in range(l):
        for k in range(d):
            c[..., k] |= ((key >> (b * d + k)) & 1) << b
    return c


def depth(P: np.ndarray, lo, side, n_max: int) -> int:
    """Smallest L >= 0 such that every depth-L cell holds at most n_max points (G1)."""
    d = P.shape[1]
    L = 0
    while True:
        if d * L > MAX_KEY_BITS:
            raise ValueError("HH_EDEPTH: d*L exceeds 62 bits before leaves hold <= n_max points")
        key = morton(cells(P, lo, side, L), L)
        _, counts = np.unique(key, return_counts=True)
        if counts.max() <= n_max:
            return L
        L += 1


@dataclass
class Tree:
    d: int
    L: int
    lo: np.ndarray
    side: float
    perm: np.ndarray          # tree position -> original index
    keys: np.ndarray          # depth-L Morton key per tree position (sorted)
    leaf_start: np.ndarray    # [2^{dL}+1]: cluster (L, m) = tree positions [leaf_start[m], leaf_start[m+1])

    def cluster(self, l: int, m: int) -> tuple[int, int]:
        s = self.d * (self.L - l)
        return int(self.leaf_start[m << s]), int(self.leaf_start[(m + 1) << s])

    def cluster_sizes(self, l: int) -> np.ndarray:
        s = self.d * (self.L - l)
        b = self.leaf_start[:: 1 << s]
        return np.diff(b)


def build_tree(P: np.ndarray, n_max: int) -> Tree:
    P = np.asarray(P, dtype=np.float64)
    N, d = P.shape
    lo, side = root_cube(P)
    L = depth(P, lo, side, n_max)
    key = morton(cells(P, lo, side, L), L)
    perm = np.argsort(key, kind="stable")        # ties keep original index order (G4)
    keys = key[perm]
    leaf_start = np.searchsorted(keys, np.arange((1 << (d * L)) + 1, dtype=np.int64), side="left")
    return Tree(d=d, L=L, lo=lo, side=side, perm=perm.astype(np.int64), keys=keys,
                leaf_start=leaf_start.astype(np.int64))
