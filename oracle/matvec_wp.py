"""Alg. 3 in a lower working precision u (oracle; NEXT-3).  PAPER.md:1055-1079 (Alg. 3:
"Compute in working precision u"), PAPER.md:1028-1040 (Thm 4.4: "this u may differ from the
u used in Alg. 2"), PAPER.md:1266-1285 (the backward-error experiment with u = fp64, fp32,
fp16), PAPER.md:35 ("the standard model of floating-point arithmetic").

Reading G27: every operand enters rounded once (RNE) to the working format —
x, each stored factor entry (exact when its storage format is narrower) and each dense
entry — and every arithmetic operation of Alg. 3 is one operation of the standard model in
that format: each product and each sum is rounded to u.  The order is Alg. 3's, plainly:
blocks in canonical order; t = V^* x_J accumulated over the rows j of the source cluster in
index order; b_I += U t accumulated over the columns k in order; dense blocks over j.

numpy float32 / float16 arithmetic rounds each + and * to the format (float16 operations are
evaluated in float32 and rounded back, which is correctly rounded for + and *: 24 >= 2 * 11 + 2).
Test infrastructure only.
"""
from __future__ import annotations

import numpy as np

from . import formats as F

WP_FP64, WP_FP32, WP_FP16 = 0, 1, 2
DTYPE = {WP_FP32: np.float32, WP_FP16: np.float16}
TAG = {WP_FP32: F.FP32, WP_FP16: F.FP16}


def to_wp(a, wp):
    """One RNE rounding from float64 to the working format (exact values as that dtype)."""
    return F.round_rne(np.asarray(a, dtype=np.float64), TAG[wp]).astype(DTYPE[wp])


def matvec_blocks_wp(n, perm, blocks, x, wp):
    """Alg. 3 with working precision ``wp`` over (i0, i1, j0, j1, kind, payload) block records
    (oracle.matvec.matvec_blocks' format; payloads hold the STORED values as float64).
    x: (n, nrhs) in original point order.  Returns y (n, nrhs) float64 in original order."""
    dt = DTYPE[wp]
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    xt = to_wp(x[perm], wp)                     # tree order, rounded once
    yt = np.zeros(xt.shape, dt)
    for i0, i1, j0, j1, kind, payload in blocks:
        xJ = xt[j0:j1]
        if kind == "lr":
            U, W = payload
            p = U.shape[1]
            if p == 0:
                continue
            U, W = to_wp(U, wp), to_wp(W, wp)
            t = np.zeros((p, xt.shape[1]), dt)
            for j in range(j1 - j0):             # t = W^T x_J, rows in order
                t = t + W[j][:, None] * xJ[j][None, :]
            yI = yt[i0:i1]
            for k in range(p):                   # b_I += U t, columns in order
                yI = yI + U[:, k][:, None] * t[k][None, :]
            yt[i0:i1] = yI
        else:
            D = to_wp(payload, wp)
            yI = yt[i0:i1]
            for j in range(j1 - j0):
                yI = yI + D[:, j][:, None] * xJ[j][None, :]
            yt[i0:i1] = yI
    y = np.empty(yt.shape, np.float64)
    y[perm] = yt.astype(np.float64)
    return y


def rounded_operand_product(n, perm, blocks, x, wp):
    """The exact (fp64) Alg. 3 product of the working-precision-rounded operands, and the
    componentwise magnitude S = sum_b |U| (|W|^T |x|) + |D| |x| that scales every rounding
    error of the working-precision evaluation (Higham, Accuracy and Stability, §3.1), plus
    per row the accumulation length K (sum of the ranks / dense widths reaching the row) and
    the longest source cluster n_J feeding it."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    xt = to_wp(x[perm], wp).astype(np.float64)
    y = np.zeros(xt.shape)
    S = np.zeros(xt.shape)
    K = np.zeros(n, np.int64)
    nJ = np.zeros(n, np.int64)
    for i0, i1, j0, j1, kind, payload in blocks:
        if kind == "lr":
            U, W = payload
            if U.shape[1] == 0:
                continue
            U = to_wp(U, wp).astype(np.float64)
            W = to_wp(W, wp).astype(np.float64)
            y[i0:i1] += U @ (W.T @ xt[j0:j1])
            S[i0:i1] += np.abs(U) @ (np.abs(W).T @ np.abs(xt[j0:j1]))
            K[i0:i1] += U.shape[1]
        else:
            D = to_wp(payload, wp).astype(np.float64)
            y[i0:i1] += D @ xt[j0:j1]
            S[i0:i1] += np.abs(D) @ np.abs(xt[j0:j1])
            K[i0:i1] += j1 - j0
        nJ[i0:i1] = np.maximum(nJ[i0:i1], j1 - j0)
    out = {}
    for name, arr in (("y", y), ("S", S)):
        o = np.empty_like(arr)
        o[perm] = arr
        out[name] = o
    for name, arr in (("K", K), ("nJ", nJ)):
        o = np.empty_like(arr)
        o[perm] = arr
        out[name] = o
    return out


def gamma(k, u):
    """gamma_k = k u / (1 - k u) (Higham, Lemma 3.1); inf when k u >= 1."""
    ku = np.asarray(k, dtype=np.float64) * u
    return np.where(ku < 1, ku / np.maximum(1 - ku, 1e-300), np.inf)


def gamma_prob(k, u, lam=8.0):
    """Probabilistic gamma~_k(lambda) = exp(lambda sqrt(k) u + k u^2 / (1 - u)) - 1 (Higham &
    Mary, SIAM J. Sci. Comput. 41 (2019), Thm 2.4): holds for a k-term computation with
    probability >= 1 - 2k exp(-lambda^2 (1-u)^2 / 2) when the rounding errors are mean
    independent; lambda = 8 gives a failure probability below 3e-14 per term."""
    k = np.asarray(k, dtype=np.float64)
    return np.expm1(lam * np.sqrt(k) * u + k * u * u / (1 - u))
