"""Arena packing function (oracle) — DESIGN.md §4, implemented independently of the CUDA path.

Not a paper passage: the paper stores factors "in precision u_ij"
without a memory layout.  The layout is ours and is a pure function of
(leaf sizes, partition, ranks, tags, storage kinds).  Check (1c) compares every offset
computed here with the offsets the GPU build exported, bit for bit.

Layout (byte offsets; ALIGN = 16):
  z     : low-rank blocks ordered by (level, tgt, tag, src); zoff = exclusive prefix sum of p.
  W[g]  : source panels.  Tag-g low-rank blocks with p > 0 ordered by (level, src, tgt); a
          run of equal (level, src) is one panel: an n x P matrix (n = |src cluster|, P = sum
          of the run's ranks) whose columns are the blocks' W_b columns in that order
          (wcol[b] = first column of b).  The panel is cut into column tiles of CT = 248
          columns (the last one narrower); each tile is stored row-major (element (r, j) of a
          tile of width ct at r * ct + j) and starts at a multiple of ALIGN; tiles follow each
          other in column order.  w_off[b] = byte offset of the panel's first tile.
  U[g]  : one stream per leaf R (Morton order), starting at a multiple of ALIGN; inside,
          for levels l = 1..L, the tag-g low-rank blocks with target anc_l(R) in src order
          contribute their rows U_b[R, :] as an |R| x p_b column-major slab.  ucol[b] is the
          first column of block b inside any leaf stream of its target.
  D     : fp64 dense blocks (leaf diagonals, and dense leaf neighbours of pure H_s) grouped
          by target leaf R in src order, |R| x |J| column-major; each leaf group starts at a
          multiple of ALIGN.
"""
from __future__ import annotations

import numpy as np

from . import formats as F

ALIGN = 16
CT = 248          # W panel column-tile width (W_CT in csrc/handle.h)
LR, DENSE = 0, 1


def align_up(x, a=ALIGN):
    return (np.asarray(x, dtype=np.int64) + (a - 1)) // a * a


def cluster_bounds(leaf_start, d, L, l, m):
    s = d * (L - l)
    m = np.asarray(m, dtype=np.int64)
    return leaf_start[m << s], leaf_start[(m + 1) << s]


def pack(leaf_start, d, L, level, tgt, src, rank, tag, storage):
    leaf_start = np.asarray(leaf_start, dtype=np.int64)
    level = np.asarray(level, np.int64)
    tgt = np.asarray(tgt, np.int64)
    src = np.asarray(src, np.int64)
    rank = np.asarray(rank, np.int64)
    tag = np.asarray(tag, np.int64)
    storage = np.asarray(storage, np.int64)
    nb = level.size
    ncell = leaf_start.size - 1
    i0, i1 = cluster_bounds(leaf_start, d, L, level, tgt)
    j0, j1 = cluster_bounds(leaf_start, d, L, level, src)
    m_b, n_b = i1 - i0, j1 - j0
    lr = storage == LR

    # z offsets: (level, tgt, tag, src) over low-rank blocks
    zoff = np.full(nb, -1, np.int64)
    idx = np.nonzero(lr)[0]
    order = idx[np.lexsort((src[idx], tag[idx], tgt[idx], level[idx]))]
    pz = rank[order]
    zoff[order] = np.cumsum(pz) - pz
    ztotal = int(pz.sum())

    # W arenas: panels of column tiles
    w_off = np.full(nb, -1, np.int64)
    wcol = np.full(nb, -1, np.int64)
    wpanel = np.full(nb, -1, np.int64)
    w_bytes = np.zeros(len(F.TAGS), np.int64)
    for g in F.TAGS:
        idx = np.nonzero(lr & (tag == g) & (rank > 0))[0]
        order = idx[np.lexsort((tgt[idx], src[idx], level[idx]))]
        off = 0
        k = 0
        while k < order.size:
            e = k
            while e < order.size and level[order[e]] == level[order[k]] and src[order[e]] == src[order[k]]:
                e += 1
            run = order[k:e]
            P = int(rank[run].sum())
            wcol[run] = np.cumsum(rank[run]) - rank[run]
            wpanel[run] = P
            w_off[run] = off
            n = int(n_b[run[0]])
            for c0 in range(0, P, CT):
                off += int(align_up(n * min(CT, P - c0) * F.BYTES[g]))
            k = e
        w_bytes[g] = off

    # U arenas: per-group column totals G[l][(t, g)], ucol per block
    ucol = np.full(nb, -1, np.int64)
    leaf_cols = np.zeros((len(F.TAGS), ncell), np.int64)
    leaf_ids = np.arange(ncell, dtype=np.int64)
    for l in range(0, L + 1):
        sel = np.nonzero(lr & (level == l) & (rank > 0))[0]
        if sel.size == 0:
            continue
        for g in F.TAGS:
            sg = sel[tag[sel] == g]
            if sg.size == 0:
                continue
            o = sg[np.lexsort((src[sg], tgt[sg]))]       # canonical group order
            # per-target totals at this level
            tot_t = np.zeros(1 << (d * l), np.int64)
            np.add.at(tot_t, tgt[o], rank[o])
            # prefix within group: exclusive cumsum restarted at every new target
            cs = np.cumsum(rank[o]) - rank[o]
            first = np.ones(o.size, bool)
            first[1:] = tgt[o][1:] != tgt[o][:-1]
            start_at = np.maximum.accumulate(np.where(first, np.arange(o.size), 0))
            within = cs - cs[start_at]
            # column base of this level = columns of coarser levels in the leaf stream,
            # identical for every leaf under the same target (read from any leaf of it)
            anc_leaf = tgt[o] << (d * (L - l))
            ucol[o] = leaf_cols[g, anc_leaf] + within
            leaf_cols[g] += tot_t[leaf_ids >> (d * (L - l))]
    nR = np.diff(leaf_start)
    u_leaf_off = np.zeros((len(F.TAGS), ncell + 1), np.int64)
    for g in F.TAGS:
        sz = align_up(nR * leaf_cols[g] * F.BYTES[g])
        u_leaf_off[g, 1:] = np.cumsum(sz)

    # dense arena
    d_off = np.full(nb, -1, np.int64)
    d_leaf_off = np.zeros(ncell + 1, np.int64)
    dn = np.nonzero(storage == DENSE)[0]
    o = dn[np.lexsort((src[dn], tgt[dn]))]
    sizes = m_b[o] * n_b[o] * 8
    per_leaf = np.zeros(ncell, np.int64)
    np.add.at(per_leaf, tgt[o], sizes)
    d_leaf_off[1:] = np.cumsum(align_up(per_leaf))
    within = np.cumsum(sizes) - sizes
    first_of_leaf = np.searchsorted(tgt[o], tgt[o], side="left")
    d_off[o] = d_leaf_off[tgt[o]] + (within - within[first_of_leaf])
    return dict(zoff=zoff, ztotal=ztotal, w_off=w_off, wcol=wcol, wpanel=wpanel, w_bytes=w_bytes, ucol=ucol,
                u_leaf_off=u_leaf_off, d_off=d_off, d_leaf_off=d_leaf_off,
                m=m_b, n=n_b, i0=i0, j0=j0, rank=rank)


def w_offsets(layout, b, g):
    """Byte offsets in W[g] of the n x p elements W_b[r, c] of low-rank block b (p > 0)."""
    n, w = int(layout["n"][b]), F.BYTES[g]
    P, c0 = int(layout["wpanel"][b]), int(layout["wcol"][b])
    p = int(layout["rank"][b])
    r = np.arange(n, dtype=np.int64)[:, None]
    pc = c0 + np.arange(p, dtype=np.int64)[None, :]      # panel columns
    t = pc // CT                                          # tile
    ct = np.minimum(CT, P - t * CT)                       # tile width
    tile_start = int(layout["w_off"][b]) + t * int(align_up(n * CT * w))   # all earlier tiles are full
    return tile_start + (r * ct + (pc - t * CT)) * w


def unpack_block(layout, b, leaf_start, d, L, level, tgt, rank, tag, storage, arenas):
    """Reconstruct block b's stored values (exact float64) from raw arena bytes.

    arenas: dict with keys ('W', g), ('U', g), 'D' -> numpy uint8 buffers.
    Returns ("lr", (U, W)) or ("dense", D).
    """
    m, n = int(layout["m"][b]), int(layout["n"][b])
    if storage[b] == DENSE:
        off = int(layout["d_off"][b])
        D = F.from_storage_bytes(arenas["D"][off:off + m * n * 8], F.FP64)
        return "dense", D.reshape(n, m).T
    p, g = int(rank[b]), int(tag[b])
    if p == 0:
        return "lr", (np.zeros((m, 0)), np.zeros((n, 0)))
    w = F.BYTES[g]
    offs = w_offsets(layout, b, g)
    raw = arenas[("W", g)]
    elem = np.stack([raw[offs + k] for k in range(w)], axis=-1).reshape(-1)
    W = F.from_storage_bytes(elem, g).reshape(n, p)
    U = np.zeros((m, p))
    l = int(level[b])
    i0 = int(layout["i0"][b])
    s = d * (L - l)
    t = int(tgt[b])
    for R in range(t << s, (t + 1) << s):
        r0, r1 = int(leaf_start[R]), int(leaf_start[R + 1])
        nr = r1 - r0
        if nr == 0:
            continue
        base = int(layout["u_leaf_off"][g, R]) + int(layout["ucol"][b]) * nr * w
        slab = F.from_storage_bytes(arenas[("U", g)][base:base + nr * p * w], g).reshape(p, nr).T
        U[r0 - i0:r1 - i0] = slab
    return "lr", (U, W)
