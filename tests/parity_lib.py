"""Helpers for GPU-vs-oracle parity (used by tests/test_gpu_*.py, __graft_entry__.smoke and
bench.py's reference leg).  Test infrastructure: may import oracle/."""
from __future__ import annotations

import numpy as np

import workloads as W
from oracle import formats as F
from oracle import hmatrix as HM
from oracle import matvec as MV
from oracle import pack as PK
from oracle import tree as T


def gpu_build(P: np.ndarray, cfg: dict, pset=None, s=None):
    import torch
    from paper_2604_09147_b200 import hh
    Pd = torch.from_numpy(np.ascontiguousarray(P)).cuda()
    H = hh.hh_build(Pd, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"],
                    cfg["s"] if s is None else s, cfg["pset"] if pset is None else pset)
    torch.cuda.synchronize()
    return H


def export(H, arenas=True):
    from paper_2604_09147_b200 import hh
    return hh.hh_export(H, tables=True, arenas=arenas)


def check_partition(ex, Ho):
    """Check (1a): perm, leaf offsets and the block table (level, kind, tgt, src) bit-exact."""
    np.testing.assert_array_equal(ex["perm"].astype(np.int64), Ho.tree.perm)
    np.testing.assert_array_equal(ex["leaf_start"], Ho.tree.leaf_start)
    B = ex["blocks"]
    assert B.size == len(Ho.part)
    for name, ref in (("level", Ho.part.level), ("kind", Ho.part.kind), ("tgt", Ho.part.tgt), ("src", Ho.part.src)):
        np.testing.assert_array_equal(B[name].astype(np.int64), ref, err_msg=name)


def oracle_partition(P, cfg, s=None):
    from oracle import partition as PT
    tr = T.build_tree(P, cfg["leaf"])
    return tr, PT.build_partition(tr, cfg["eta"], cfg["s"] if s is None else s)


def check_packing(ex):
    """Check (1c): the oracle's packing function on the GPU's (rank, tag, storage) reproduces
    every exported offset bit for bit."""
    B = ex["blocks"]
    d, L = ex["info"]["d"], ex["info"]["L"]
    lay = PK.pack(ex["leaf_start"], d, L, B["level"], B["tgt"], B["src"], B["rank"], B["tag"], B["storage"])
    lr = B["storage"] == 0
    np.testing.assert_array_equal(lay["zoff"][lr], B["zoff"][lr], err_msg="zoff")
    has = lr & (B["rank"] > 0)
    np.testing.assert_array_equal(lay["w_off"][has], B["w_off"][has], err_msg="w_off")
    np.testing.assert_array_equal(lay["wcol"][has], B["wcol"][has], err_msg="wcol")
    np.testing.assert_array_equal(lay["ucol"][has], B["ucol"][has], err_msg="ucol")
    dn = ~lr
    np.testing.assert_array_equal(lay["d_off"][dn], B["d_off"][dn], err_msg="d_off")
    np.testing.assert_array_equal(lay["u_leaf_off"], ex["u_leaf_off"], err_msg="u_leaf_off")
    np.testing.assert_array_equal(lay["d_leaf_off"], ex["d_leaf_off"], err_msg="d_leaf_off")
    info = ex["info"]
    np.testing.assert_array_equal(lay["w_bytes"], np.array(info["w_bytes"]), err_msg="w_bytes")
    assert lay["ztotal"] == info["total_rank"]
    return lay


def exported_blocks(ex, lay):
    """Decode every block of the export with the ORACLE's packing function -> Alg. 3 input."""
    B = ex["blocks"]
    d, L = ex["info"]["d"], ex["info"]["L"]
    for b in range(B.size):
        kind, payload = PK.unpack_block(lay, b, ex["leaf_start"], d, L, B["level"], B["tgt"], B["rank"],
                                        B["tag"], B["storage"], ex)
        i0, j0 = int(lay["i0"][b]), int(lay["j0"][b])
        yield i0, i0 + int(lay["m"][b]), j0, j0 + int(lay["n"][b]), kind, payload


def oracle_matvec_on_export(ex, lay, x):
    return MV.matvec_blocks(ex["info"]["N"], ex["perm"].astype(np.int64), exported_blocks(ex, lay), x)


def rank_tag_parity(ex, Ho, rank_margin=1e-9, tag_margin=1e-12):
    """Check (1b): storage kind, rank and tag per block equal to the oracle's (truncated-SVD rank,
    Eq. 4.4 tag, PAPER.md:992 beneficial rule).  A difference is tolerated only where the
    oracle's own decision lies within `rank_margin` (relative) of its truncation threshold or
    `tag_margin` of its Eq. 4.4 threshold (1e-9 / 1e-12) — fp64 rounding of sigma
    near eps ||A|| is of order u/eps.  A storage difference (a leaf neighbour kept dense on one
    side and low-rank on the other) counts as a rank difference unless one of its margins
    explains it.  Returns (n_rank_or_storage_unexplained, n_tag_unexplained, stats)."""
    B = ex["blocks"]
    gs, os_ = B["storage"].astype(np.int64), Ho.storage
    lr = (gs == 0) & (os_ == 0)
    rk = B["rank"].astype(np.int64)
    near = (Ho.margin <= rank_margin) | (Ho.tag_margin <= tag_margin)
    bad_s = (gs != os_) & ~near
    bad_r = lr & (rk != Ho.rank) & (Ho.margin > rank_margin)
    same_r = lr & (rk == Ho.rank)
    bad_t = same_r & (B["tag"].astype(np.int64) != Ho.tag) & (Ho.tag_margin > tag_margin)
    st = dict(n_lr=int(lr.sum()), rank_diff=int((lr & (rk != Ho.rank)).sum()),
              tag_diff=int((same_r & (B["tag"] != Ho.tag)).sum()),
              storage_diff=int((gs != os_).sum()), storage_unexplained=int(bad_s.sum()),
              n_dense_nbr=int(((gs == 1) & (B["kind"] == 3)).sum()))
    return int(bad_r.sum()) + int(bad_s.sum()), int(bad_t.sum()), st


def gpu_matvec(H, x: np.ndarray) -> np.ndarray:
    import torch
    from paper_2604_09147_b200 import hh
    xd = torch.from_numpy(np.asfortranarray(x).reshape(x.shape[0], -1, order="F").T.copy()).cuda().T
    yd = torch.empty_like(xd.T).T
    hh.hh_matvec(H, xd, yd, xd.shape[1])
    torch.cuda.synchronize()
    return yd.cpu().numpy()


def oracle_build(P, cfg, pset=None, s=None, keep_exact=False):
    return HM.build(P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"],
                    cfg["s"] if s is None else s, cfg["pset"] if pset is None else pset, keep_exact=keep_exact)


def rel2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b)) if np.linalg.norm(b) else float(np.linalg.norm(a))


def _hh():
    from paper_2604_09147_b200 import hh
    return hh


def leaf_blocks(B, lay, tr, R):
    """Blocks whose target cluster contains leaf R (every level), in canonical order."""
    d, L = tr.d, tr.L
    lv = B["level"].astype(np.int64)
    return np.nonzero((B["tgt"] == (np.int64(R) >> (d * (L - lv)))) & ((B["storage"] == 1) | (B["rank"] > 0)))[0]


def oracle_leaf_rows(H, B, lay, tr, R, xt):
    """Alg. 3 restricted to the rows of leaf R, on factors decoded with the oracle's packing
    function from ranged arena exports.  xt: x in tree order (N, nrhs)."""
    r0, r1 = int(tr.leaf_start[R]), int(tr.leaf_start[R + 1])
    nr = r1 - r0
    y = np.zeros((nr, xt.shape[1]))
    for b in leaf_blocks(B, lay, tr, R):
        j0, nn = int(lay["j0"][b]), int(lay["n"][b])
        if B["storage"][b] == 1:                       # dense (fp64)
            i0, mm = int(lay["i0"][b]), int(lay["m"][b])
            off = int(lay["d_off"][b])
            raw = _hh().export_arena(H, _hh().ARENA_D, off, mm * nn * 8)
            Dm = F.from_storage_bytes(raw, F.FP64).reshape(nn, mm).T
            y += Dm[r0 - i0:r1 - i0] @ xt[j0:j0 + nn]
            continue
        g, p = int(B["tag"][b]), int(B["rank"][b])
        w = F.BYTES[g]
        offs = PK.w_offsets(lay, b, g)
        lo, hi = int(offs.min()), int(offs.max()) + w
        raw = _hh().export_arena(H, _hh().ARENA_W + g, lo, hi - lo)
        elem = np.stack([raw[offs - lo + k] for k in range(w)], axis=-1).reshape(-1)
        Wb = F.from_storage_bytes(elem, g).reshape(nn, p)
        base = int(lay["u_leaf_off"][g, R]) + int(lay["ucol"][b]) * nr * w
        Ub = F.from_storage_bytes(_hh().export_arena(H, _hh().ARENA_U + g, base, nr * p * w), g).reshape(p, nr).T
        y += Ub @ (Wb.T @ xt[j0:j0 + nn])
    return y


# ----------------------------------------------------------------------------- check (1b) at scale
def kernel_block_chunked(P, rows, cols, kind, scale, chunk=1024):
    """oracle.kernels.block in row chunks (bounded temporaries for 16384 x 16384 blocks)."""
    from oracle.kernels import block as kb
    A = np.empty((rows.size, cols.size))
    for r0 in range(0, rows.size, chunk):
        A[r0:r0 + chunk], _ = kb(P, rows[r0:r0 + chunk], cols, kind, scale)
    return A


def ritz_sigmas(A, k, q=3, seed=0):
    """Singular values of Q^T A for an orthonormal Q (n_rows x k) from k-column subspace
    iteration with q power steps: sigma_i(Q^T A) <= sigma_i(A) for every i (Cauchy interlacing),
    so these are certified LOWER bounds that converge fast on decaying kernel spectra.  Returns
    (s, Q, B) with B = Q^T A."""
    import scipy.linalg as sl
    m, n = A.shape
    k = int(min(k, m, n))
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(A @ rng.standard_normal((n, k)))
    for _ in range(q):
        Z, _ = np.linalg.qr(A.T @ Q)
        Q, _ = np.linalg.qr(A @ Z)
    B = Q.T @ A
    return sl.svdvals(B), Q, B


def certify_rank(A, p, eps, extra=64, q=3):
    """Proof (up to rounding well below 1e-9 relative) that p is the truncated-SVD rank of A at
    relative Frobenius accuracy eps (reading G10: smallest p with
    sum_{k>p} sigma_k^2 <= eps^2 ||A||_F^2), for blocks too large for a dense LAPACK SVD:
      valid   : an explicit rank-p approximation U_p U_p^T A (U_p = Q times the top-p left
                singular vectors of Q^T A) has residual ||A - U_p U_p^T A||_F^2 <= eps^2 ||A||^2,
                and the optimal rank-p error is no larger;
      minimal : sum_{k>=p} s_k^2 over the Ritz values (lower bounds of sigma_k) already exceeds
                eps^2 ||A||^2, so no rank p-1 approximation meets eps.
    Returns dict(valid, minimal, tail_p_upper, tail_pm1_lower, thr, nb2_lower, nb2_upper).
    nb2 = sum_{k<=p} sigma_k^2 is bracketed by the Ritz sum (lower) and ||A||^2 minus the residual
    (upper)."""
    tot = float(np.sum(A * A))
    thr = eps * eps * tot
    s, Q, B = ritz_sigmas(A, p + extra, q)
    if p == 0:
        return dict(valid=tot <= thr, minimal=True, tail_p_upper=tot, tail_pm1_lower=np.inf, thr=thr,
                    nb2_lower=0.0, nb2_upper=0.0)
    Ub, _, _ = np.linalg.svd(B, full_matrices=False)
    Up = Q @ Ub[:, :p]
    Wp = A.T @ Up
    res = 0.0
    for r0 in range(0, A.shape[0], 2048):                   # residual in row chunks
        E = A[r0:r0 + 2048] - Up[r0:r0 + 2048] @ Wp.T
        res += float(np.sum(E * E))
    lower = float(np.sum(s[p - 1:] ** 2))
    return dict(valid=res <= thr, minimal=lower > thr, tail_p_upper=res, tail_pm1_lower=lower, thr=thr,
                nb2_lower=float(np.sum(s[:p] ** 2)), nb2_upper=tot - res)
