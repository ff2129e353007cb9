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
    for tag in (F.BF16, F.FP16, F.FP32, F.FP64):          # decreasing unit roundoff
        if not (pset & F.TAG_BIT[tag]):
            continue
        u = F.unit_roundoff(tag)
        if (u * u) * float(2.0 ** (d * l)) * nb2 <= rhs:
            return tag, False
    return F.FP64, True


def guard_tag(tag: int, maxabs: float, pset: int) -> tuple[int, bool]:
    """Range guard: while rounding the largest factor entry to `tag` overflows, promote."""
    order = [t for t in (F.BF16, F.FP16, F.FP32, F.FP64) if pset & F.TAG_BIT[t]]
    promoted = False
    i = order.index(tag)
    while np.isinf(F.round_rne(np.array([maxabs]), order[i])[0]) and order[i] != F.FP64:
        i += 1
        promoted = True
    return order[i], promoted


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
    mixed = (pset & 0xF) != F.TAG_BIT[F.FP64]   # format bits only (flags such as TIE_FP16 excluded)
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
    # ||H~||^2 (Alg. 4): low-rank blocks by trace(Sigma~^2); dense and (ell = L) leaf
    # neighbours by their direct norm.
    norm2 = 0.0
    for b in range(nb):
        kind = int(part.kind[b])
        norm2 += H.tot[b] if kind in (DIAG, LNBR) else H.nb2[b]
    H.norm2 = norm2
    # Alg. 2: tag every low-rank block
    for b, (U, W, A) in exact.items():
        l = int(part.level[b])
        tag, fb = choose_tag(H.nb2[b], norm2, eps, tree.d, l, pset)
        # distance of the decision from the threshold (for parity tolerances)
        u = F.unit_roundoff(tag)
        lhs = (u * u) * 2.0 ** (tree.d * l) * H.nb2[b]
        rhs = eps * eps * norm2
        tm = (rhs - lhs) / rhs if rhs else np.inf
        if tag != F.BF16:  # also distance to qualifying for the next larger u
            nxt = [t for t in (F.FP32, F.FP16, F.BF16) if F.unit_roundoff(t) > u and (pset & F.TAG_BIT[t])]
            if nxt:
                un = min(F.unit_roundoff(t) for t in nxt)
                tm = min(abs(tm), abs(((un * un) * 2.0 ** (tree.d * l) * H.nb2[b] - rhs) / rhs))
        H.tag_margin[b] = abs(tm)
        H.fallback += int(fb)
        maxabs = max(float(np.max(np.abs(U))) if U.size else 0.0, H.maxabs_w[b])
        if (pset & TIE_FP16) and tag == F.BF16 and (pset & F.TAG_BIT[F.FP16]) and \
                not np.isinf(F.round_rne(np.array([maxabs]), F.FP16)[0]):
            tag = F.FP16   # NEXT-3 bits-aware tie rule: same 16 bits, 3 more mantissa bits
        tag, pr = guard_tag(tag, maxabs, pset)
        H.promoted += int(pr)
        p = int(H.rank[b])
        i0, i1, j0, j1 = H.rows(b)
        if part.kind[b] == LNBR:
            # PAPER.md:992 beneficial rule (mixed pure H_s only)
            if not (p * ((i1 - i0) + (j1 - j0)) * F.BITS[tag] < (i1 - i0) * (j1 - j0) * 64):
                H.storage[b] = DENSE
                H.dense[b] = A
                H.rank[b] = 0
                continue
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
    by_tag = {t: 0 for t in F.BYTES}
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
