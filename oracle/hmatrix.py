"""Oracle construction of the adaptive mixed-precision H_h matrix.

Alg. 1: every admissible block of the hybrid partition is compressed
with LRcompression (truncated SVD, compress.py); leaf diagonal blocks are kept dense;
for ell = L (pure H_s) leaf neighbours are kept dense.  Entries are generated on the fly
(PAPER.md:621).
Alg. 4: ||H~||^2 = sum over low-rank blocks of trace(Sigma~^2) +
sum over dense blocks of ||H_IJ||^2 (for ell = L the leaf neighbours enter with their
directly computed norm).
Alg. 2 with Eq. 4.4: each low-rank block stores
its factors in the largest unit roundoff u in the available set with
    u <= eps / (2^{d l / 2} xi),   xi = ||H~_IJ|| / ||H~||,
evaluated in the squared form u^2 2^{d l} ||H~_IJ||^2 <= eps^2 ||H~||^2 (reading G15:
exact powers of two).  None qualifying -> fp64 + fallback flag.  Range guard (G16):
if rounding any factor entry overflows, step to the next smaller u (promoted flag).
Pure H_s in mixed mode (reading G17): a leaf neighbour is compressed and
tagged, and kept low-rank iff p(|I|+|J|) bits(tag) < |I||J| * 64, else dense fp64.
Leaf diagonal blocks stay in working precision fp64.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import formats as F
from .compress import lr_compress
from .kernels import block as kernel_block
from .partition import DIAG, LNBR, SWITCH_NONE, Partition, build_partition
from .tree import Tree, build_tree

LR, DENSE = 0, 1
TIE_FP16 = 1 << 17   # precision_set flag (include/hh.h HH_TIE_FP16): fp16 over bf16 when both qualify


def choose_tag(nb2: float, norm2: float, eps: float, d: int, l: int, pset: int) -> tuple[int, bool]:
    """Eq. 4.4 / Alg. 2 line 4: largest admissible unit roundoff (squared, exact form)."""
    rhs = (eps * eps) * norm2
    for tag in F.BY_U:                                    # decreasing unit roundoff
        if not (pset & F.TAG_BIT[tag]):
            continue
        u = F.unit_roundoff(tag)
        if (u * u) * float(2.0 ** (d * l)) * nb2 <= rhs:
            return tag, False
    return F.FP64, True


def guard_tag(tag: int, maxabs: float, pset: int) -> tuple[int, bool]:
    """Range guard: while rounding the largest factor entry to `tag` overflows, promote."""
    order = [t for t in F.BY_U if pset & F.TAG_BIT[t]]
    promoted = False
    i = order.index(tag)
    while np.isinf(F.round_rne(np.array([maxabs]), order[i])[0]) and order[i] != F.FP64:
        i += 1
        promoted = True
    return order[i], promoted


def alg4_norm2(kind, nb2, tot) -> float:
    """Alg. 4: ||H~||^2 = sum of trace(Sigma~^2) over low-rank blocks + the
    direct ||H_IJ||^2 of dense leaf blocks (and, for ell = L, of the leaf neighbours,
    PAPER.md:1354-1362), summed in canonical block order."""
    norm2 = 0.0
    for b in range(len(kind)):
        norm2 += float(tot[b]) if int(kind[b]) in (DIAG, LNBR) else float(nb2[b])
    return norm2


def tag_blocks(d, level, kind, m, n, rank, nb2, tot, maxabs, eps, pset) -> dict:
    """Alg. 2 over a block table: Eq. 4.4 tag (choose_tag), the bits-aware tie rule when
    TIE_FP16 is set, the range guard (guard_tag) and, for pure H_s in mixed precision, the
    PAPER.md:992 beneficial rule for leaf neighbours.  Blocks start dense when they are leaf
    diagonals, or leaf neighbours in uniform precision (Alg. 1 keeps them dense); every other
    block is a compressed low-rank candidate.  ``maxabs`` = max |entry| of the block's
    unrounded factors U and W.  Returns per-block tag / storage / rank (0 for dense), the
    pre-rule rank and tag of every low-rank candidate (lr_rank, lr_tag), ||H~||^2, the
    fallback / promoted counts and each tag decision's relative distance from its threshold."""
    nb = len(kind)
    mixed = (pset & F.ALL_FORMATS) != F.TAG_BIT[F.FP64]
    norm2 = alg4_norm2(kind, nb2, tot)
    tag = np.zeros(nb, np.int64)
    lr_tag = np.full(nb, -1, np.int64)
    storage = np.full(nb, LR, np.int64)
    out_rank = np.array(rank, dtype=np.int64).copy()
    lr_rank = np.full(nb, -1, np.int64)
    tag_margin = np.full(nb, np.inf)
    fallback = promoted = 0
    rhs = eps * eps * norm2
    for b in range(nb):
        k, l = int(kind[b]), int(level[b])
        if k == DIAG or (k == LNBR and not mixed):
            storage[b] = DENSE
            out_rank[b] = 0
            continue
        t, fb = choose_tag(float(nb2[b]), norm2, eps, d, l, pset)
        # distance of the decision from the threshold (for parity tolerances)
        u = F.unit_roundoff(t)
        lhs = (u * u) * 2.0 ** (d * l) * float(nb2[b])
        tm = (rhs - lhs) / rhs if rhs else np.inf
        if t != F.Q43:   # also distance to qualifying for the next larger u
            nxt = [c for c in F.TAGS if F.unit_roundoff(c) > u and (pset & F.TAG_BIT[c])]
            if nxt:
                un = min(F.unit_roundoff(c) for c in nxt)
                tm = min(abs(tm), abs(((un * un) * 2.0 ** (d * l) * float(nb2[b]) - rhs) / rhs))
        tag_margin[b] = abs(tm)
        fallback += int(fb)
        if (pset & TIE_FP16) and t == F.BF16 and (pset & F.TAG_BIT[F.FP16]) and \
                not np.isinf(F.round_rne(np.array([maxabs[b]]), F.FP16)[0]):
            t = F.FP16   # NEXT-3 bits-aware tie rule: same 16 bits, 3 more mantissa bits
        t, pr = guard_tag(t, float(maxabs[b]), pset)
        promoted += int(pr)
        lr_rank[b], lr_tag[b] = int(rank[b]), t
        if k == LNBR:
            # PAPER.md:992 beneficial rule (mixed pure H_s only): low-rank iff fewer bits
            if not (int(rank[b]) * (int(m[b]) + int(n[b])) * F.BITS[t] < int(m[b]) * int(n[b]) * 64):
                storage[b] = DENSE
                out_rank[b] = 0
                continue
        tag[b] = t
    return dict(tag=tag, storage=storage, rank=out_rank, lr_rank=lr_rank, lr_tag=lr_tag, norm2=norm2,
                fallback=fallback, promoted=promoted, tag_margin=tag_margin)


@dataclass
class OracleH:
    tree: Tree
    part: Partition
    d: int
    eps: float
    eta: float
    s: int
    kernel: int
    scale: float
    pset: int
    n: int = 0
    rank: np.ndarray = None
    tag: np.ndarray = None
    storage: np.ndarray = None
    nb2: np.ndarray = None
    tot: np.ndarray = None
    margin: np.ndarray = None
    maxabs_w: np.ndarray = None
    norm2: float = 0.0
    factors: dict = field(default_factory=dict)   # b -> (U_hat, W_hat) float64 (rounded values)
    exact: dict = field(default_factory=dict)     # b -> (U, W) float64 before rounding
    dense: dict = field(default_factory=dict)     # b -> dense block (fp64)
    tag_margin: np.ndarray = None
    fallback: int = 0
    promoted: int = 0
    coincident: int = 0
    lr_rank: np.ndarray = None    # rank / tag of every compressed candidate before the beneficial rule
    lr_tag: np.ndarray = None

    def rows(self, b):
        l = int(self.part.level[b])
        i0, i1 = self.tree.cluster(l, int(self.part.tgt[b]))
        j0, j1 = self.tree.cluster(l, int(self.part.src[b]))
        return i0, i1, j0, j1


def build(P, kernel, scale, eps, eta, leaf, s, pset, keep_exact=False) -> OracleH:
    P = np.asarray(P, dtype=np.float64)
    if not (pset & F.TAG_BIT[F.FP64]):
        raise ValueError("FP64 must be in the precision set")
    tree = build_tree(P, leaf)
    if s != SWITCH_NONE and not (0 <= s <= tree.L):
        raise ValueError("switch level outside [0, L]")
    part = build_partition(tree, eta, s)
    nb = len(part)
    H = OracleH(tree=tree, part=part, d=tree.d, eps=eps, eta=eta, s=s, kernel=kernel,
                scale=scale, pset=pset, n=P.shape[0])
    H.rank = np.zeros(nb, np.int64)
    H.tag = np.zeros(nb, np.int64)
    H.storage = np.zeros(nb, np.int64)
    H.nb2 = np.zeros(nb)
    H.tot = np.zeros(nb)
    H.margin = np.full(nb, np.inf)
    H.maxabs_w = np.zeros(nb)
    H.tag_margin = np.full(nb, np.inf)
    mixed = (pset & F.ALL_FORMATS) != F.TAG_BIT[F.FP64]  # format bits only (flags such as TIE_FP16 excluded)
    perm = tree.perm
    exact = {}
    # Alg. 1 + Alg. 4: compress every admissible block, norms from singular values
    for b in range(nb):
        i0, i1, j0, j1 = H.rows(b)
        A, coinc = kernel_block(P, perm[i0:i1], perm[j0:j1], kernel, scale)
        H.coincident += coinc
        kind = int(part.kind[b])
        H.tot[b] = float(np.sum(A * A))
        if kind == DIAG or (kind == LNBR and not mixed):
            H.storage[b] = DENSE
            H.dense[b] = A
            continue
        c = lr_compress(A, eps)
        H.rank[b], H.nb2[b], H.margin[b] = c["p"], c["nb2"], c["margin"]
        H.tot[b] = c["tot"]
        H.maxabs_w[b] = float(np.max(np.abs(c["W"]))) if c["p"] else 0.0
        exact[b] = (c["U"], c["W"], A)
    m = np.array([H.rows(b)[1] - H.rows(b)[0] for b in range(nb)], np.int64)
    n = np.array([H.rows(b)[3] - H.rows(b)[2] for b in range(nb)], np.int64)
    maxabs = np.zeros(nb)
    for b, (U, W, A) in exact.items():
        maxabs[b] = max(float(np.max(np.abs(U))) if U.size else 0.0, H.maxabs_w[b])
    T = tag_blocks(tree.d, part.level, part.kind, m, n, H.rank, H.nb2, H.tot, maxabs, eps, pset)
    H.norm2 = T["norm2"]
    H.tag_margin = T["tag_margin"]
    H.fallback, H.promoted = T["fallback"], T["promoted"]
    H.lr_rank, H.lr_tag = T["lr_rank"], T["lr_tag"]
    for b, (U, W, A) in exact.items():
        if T["storage"][b] == DENSE:       # PAPER.md:992 beneficial rule kept it dense
            H.storage[b] = DENSE
            H.dense[b] = A
            H.rank[b] = 0
            continue
        tag = int(T["tag"][b])
        H.tag[b] = tag
        H.factors[b] = (F.round_rne(U, tag), F.round_rne(W, tag))
        if keep_exact:
            H.exact[b] = (U, W)
    return H


def stored_bytes(H: OracleH) -> dict:
    """Algorithmic (unpadded) storage: p(|I|+|J|) bytes(tag) per low-rank block and
    |I||J| * 8 per dense block."""
    lr = 0
    dn = 0
    by_tag = {t: 0 for t in F.TAGS}
    for b in range(len(H.part)):
        i0, i1, j0, j1 = H.rows(b)
        if H.storage[b] == DENSE:
            dn += (i1 - i0) * (j1 - j0) * 8
        else:
            nbytes = int(H.rank[b]) * ((i1 - i0) + (j1 - j0)) * F.BYTES[int(H.tag[b])]
            lr += nbytes
            by_tag[int(H.tag[b])] += nbytes
    return dict(lowrank=lr, dense=dn, total=lr + dn, by_tag=by_tag)


_RO = {}


def _ro_init(P, perm, kernel, scale, eps):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)  # one BLAS thread per worker process
    _RO.update(P=P, perm=perm, kernel=kernel, scale=scale, eps=eps)


def _ro_rank(job):
    from scipy.linalg import svdvals
    from .compress import truncation_rank
    i0, i1, j0, j1 = job
    A, _ = kernel_block(_RO["P"], _RO["perm"][i0:i1], _RO["perm"][j0:j1], _RO["kernel"], _RO["scale"])
    return truncation_rank(svdvals(A), _RO["eps"])[0] if A.size else 0


def ranks_only(P, kernel, scale, eps, eta, leaf, s, workers=None):
    """Partition + truncated-SVD ranks only (singular values, no vectors) — for storage
    studies (Table 3) where factors are not needed.  The independent
    per-block SVDs are spread over worker processes.  Returns (tree, partition, rank[], m[],
    n[]) with rank = -1 for blocks kept dense."""
    import os
    from concurrent.futures import ProcessPoolExecutor
    tr = build_tree(P, leaf)
    part = build_partition(tr, eta, s)
    nb = len(part)
    rank = np.full(nb, -1, np.int64)
    m = np.zeros(nb, np.int64)
    n = np.zeros(nb, np.int64)
    jobs, idx = [], []
    for b in range(nb):
        l = int(part.level[b])
        i0, i1 = tr.cluster(l, int(part.tgt[b]))
        j0, j1 = tr.cluster(l, int(part.src[b]))
        m[b], n[b] = i1 - i0, j1 - j0
        if part.kind[b] in (DIAG, LNBR):
            continue
        jobs.append((i0, i1, j0, j1))
        idx.append(b)
    with ProcessPoolExecutor(max_workers=workers or os.cpu_count(), initializer=_ro_init,
                             initargs=(P, tr.perm, kernel, scale, eps)) as ex:
        for b, r in zip(idx, ex.map(_ro_rank, jobs, chunksize=64)):
            rank[b] = r
    return tr, part, rank, m, n
