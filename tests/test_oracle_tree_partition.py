"""Pins for oracle/tree.py and oracle/partition.py.  CPU only."""
import os
from fractions import Fraction

import numpy as np
import pytest

import workloads as W
from oracle import partition as PT
from oracle import tree as T


# ---------------------------------------------------------------- tree
def test_quadrant_centres_one_per_cell():
    # SPEC.md:82 example: 4 quadrant-centre points, n_max = 1 -> L = 1, one point per cell
    P = np.array([[0.25, 0.25], [0.75, 0.25], [0.25, 0.75], [0.75, 0.75]])
    tr = T.build_tree(P, 1)
    assert tr.L == 1
    assert list(np.diff(tr.leaf_start)) == [1, 1, 1, 1]
    # Morton: axis 0 is the least significant bit of the digit
    assert list(tr.perm) == [0, 1, 2, 3]


def test_tree_is_a_partition_and_depth_is_minimal():
    P = W.points_uniform(3000, 3, 5)
    tr = T.build_tree(P, 20)
    assert sorted(tr.perm.tolist()) == list(range(3000))
    sizes = np.diff(tr.leaf_start)
    assert sizes.sum() == 3000 and sizes.max() <= 20
    # minimality by direct counting of one level coarser
    c = T.cells(P, tr.lo, tr.side, tr.L - 1)
    _, counts = np.unique(c, axis=0, return_counts=True)
    assert counts.max() > 20


def test_clusters_are_geometric_boxes():
    """Cluster (l, m) range == points whose level-l cell (direct floor formula, exact
    rational evaluation) has Morton code m.  Independent of the prefix-shift shortcut."""
    P = W.points_uniform(500, 2, 9)
    tr = T.build_tree(P, 8)
    lo, side = tr.lo, tr.side
    for l in range(tr.L + 1):
        for i in range(0, 500, 7):
            # exact rational cell coordinate, top face clamped
            c = [min((1 << l) - 1, int((Fraction(P[i, k]) - Fraction(lo[k])) / Fraction(side) * (1 << l)))
                 for k in range(2)]
            m = int(T.morton(np.array([c]), l)[0])
            a, b = tr.cluster(l, m)
            pos = int(np.nonzero(tr.perm == i)[0][0])
            assert a <= pos < b


# ------------------------------------------------------- admissibility / list sizes
def _grid_tree(d, L):
    return T.build_tree(W.points_grid_centres(d, L), 1)


def _max_counts(part, kinds, level=None):
    m = np.isin(part.kind, kinds)
    if level is not None:
        m &= part.level == level
    if not m.any():
        return 0
    _, c = np.unique(np.stack([part.level[m], part.tgt[m]], 1), axis=0, return_counts=True)
    return int(c.max())


def test_list_sizes_eta_sqrt2_2d():
    # eta = sqrt(2) in 2D gives |IL_s| <= 27 and |N_s| <= 8, attained
    tr = _grid_tree(2, 4)
    part = PT.build_partition(tr, np.sqrt(2.0), PT.SWITCH_NONE)
    assert _max_counts(part, [PT.FAR]) == 27
    assert _max_counts(part, [PT.LNBR]) == 8
    c = PT.sparsity_constants(part, PT.SWITCH_NONE, tr.L)          # the function the bounds use
    assert (c["c1"], c["c2"]) == (27, 8)


def test_list_sizes_eta_sqrt3_3d():
    # PAPER.md:1134 (Eq. 5.3): 189 and 26 for eta = sqrt(3) in 3D; C''' = 7
    tr = _grid_tree(3, 3)
    part = PT.build_partition(tr, np.sqrt(3.0), PT.SWITCH_NONE)
    assert _max_counts(part, [PT.FAR]) == 189
    assert _max_counts(part, [PT.LNBR]) == 26
    hod = PT.build_partition(tr, np.sqrt(3.0), 0)
    assert _max_counts(hod, [PT.SIB]) == 7      # Eq. 2.7: C''' = 2^d - 1
    assert PT.sparsity_constants(part, PT.SWITCH_NONE, tr.L)["c1"] == 189
    assert PT.sparsity_constants(hod, 0, tr.L)["c3"] == 7


def test_C_formulas_at_eta_sqrt_d():
    from oracle.metrics import list_constants
    c1, c2, c3 = list_constants(2, np.sqrt(2.0))
    assert (round(c1, 9), round(c2, 9), c3) == (27.0, 8.0, 3.0)
    c1, c2, c3 = list_constants(3, np.sqrt(3.0))
    assert (round(c1, 9), round(c2, 9), c3) == (189.0, 26.0, 7.0)


@pytest.mark.parametrize("d", [2, 3])
def test_integer_admissibility_equals_geometric_definition(d):
    """G5/G6: d <= eta^2 G equals min(diam) <= eta * dist evaluated exactly on boxes."""
    rng = np.random.default_rng(d)
    for eta in (1.0, np.sqrt(d), 0.5, 2.0):
        e2 = PT.snap_eta2(eta)
        for _ in range(300):
            a = rng.integers(-5, 6, size=d)
            got = bool(PT.adm_s_offsets(a[None, :], d, e2)[0])
            # boxes [0,1]^d and a + [0,1]^d: diam^2 = d, dist^2 = sum max(0,|a|-1)^2 (exact)
            dist2 = sum(max(0, abs(int(v)) - 1) ** 2 for v in a)
            eta2_exact = Fraction(round(eta * eta)) if abs(eta * eta - round(eta * eta)) < 1e-12 else Fraction(eta) ** 2
            assert got == (Fraction(d) <= eta2_exact * dist2)


# ---------------------------------------------------------------- partition
def _coverage(tr, part):
    N = tr.perm.size
    M = np.zeros((N, N), np.int32)
    for b in range(len(part)):
        l = int(part.level[b])
        i0, i1 = tr.cluster(l, int(part.tgt[b]))
        j0, j1 = tr.cluster(l, int(part.src[b]))
        M[i0:i1, j0:j1] += 1
    return M


@pytest.mark.parametrize("d,n,leaf", [(2, 4096, 64), (3, 3000, 40)])
@pytest.mark.parametrize("s", [PT.SWITCH_NONE, 0, 1, 2, 3])
def test_partition_covers_every_entry_once(d, n, leaf, s):
    # every (i, j) in N x N lies in exactly one block
    tr = T.build_tree(W.points_uniform(n, d, 11), leaf)
    if s > tr.L:
        pytest.skip("s > L")
    part = PT.build_partition(tr, 1.0, s)
    assert (_coverage(tr, part) == 1).all()


def _pair_block_bruteforce(tr, i, j, eta2, s):
    """Independent characterisation of Eq. 3.1 per point pair: walk down the levels with the
    boxes containing tree positions i and j; the pair lies in the block of the first level
    at which the hybrid rule admits the pair of boxes (or the dense leaf block)."""
    d, L = tr.d, tr.L
    for l in range(1, L + 1):
        bi = int(tr.keys[i] >> (d * (L - l)))
        bj = int(tr.keys[j] >> (d * (L - l)))
        ci, cj = T.demorton(bi, d, l), T.demorton(bj, d, l)
        g = np.maximum(0, np.abs(cj - ci) - 1)
        adm = d <= eta2 * int(np.sum(g * g))
        if s == PT.SWITCH_NONE or l < s:
            if adm:
                return (l, bi, bj)
        elif bi != bj:
            return (l, bi, bj)
    return (L, int(tr.keys[i]), int(tr.keys[j]))


@pytest.mark.parametrize("s", [PT.SWITCH_NONE, 0, 2, 3])
def test_partition_matches_pairwise_bruteforce(s):
    tr = T.build_tree(W.points_uniform(400, 2, 4), 10)
    part = PT.build_partition(tr, 1.0, s)
    owner = {}
    for b in range(len(part)):
        l = int(part.level[b])
        i0, i1 = tr.cluster(l, int(part.tgt[b]))
        j0, j1 = tr.cluster(l, int(part.src[b]))
        owner[(l, int(part.tgt[b]), int(part.src[b]))] = (i0, i1, j0, j1)
    rng = np.random.default_rng(0)
    for _ in range(3000):
        i, j = rng.integers(0, 400, 2)
        key = _pair_block_bruteforce(tr, i, j, 1.0, s)
        i0, i1, j0, j1 = owner[key]
        assert i0 <= i < i1 and j0 <= j < j1


def test_special_cases():
    """ell = L -> H_s (standard only), ell = 0 -> HODLR (siblings only);
    s = 0 and s = 1 give the same block set (level-1 boxes all touch)."""
    tr = T.build_tree(W.points_uniform(2000, 2, 2), 16)
    hs = PT.build_partition(tr, 1.0, PT.SWITCH_NONE)
    assert set(np.unique(hs.kind)) <= {PT.FAR, PT.LNBR, PT.DIAG}
    h0 = PT.build_partition(tr, 1.0, 0)
    h1 = PT.build_partition(tr, 1.0, 1)
    assert set(np.unique(h0.kind)) == {PT.SIB, PT.DIAG}
    for a, b in ((h0.level, h1.level), (h0.tgt, h1.tgt), (h0.src, h1.src)):
        np.testing.assert_array_equal(a, b)
    # HODLR blocks are exactly the non-self sibling pairs
    sib = h0.kind == PT.SIB
    assert np.all((h0.tgt[sib] >> 2) == (h0.src[sib] >> 2)) and np.all(h0.tgt[sib] != h0.src[sib])
    # pure H_s has dense blocks only at the leaf; H_h (s < L) only on the diagonal
    hh = PT.build_partition(tr, 1.0, tr.L - 1)
    assert set(np.unique(hh.kind)) <= {PT.FAR, PT.NBR, PT.SIB, PT.DIAG}


# Golden counts: cell-centre grids (one point per leaf), tests/golden/partition_counts.txt
# (derived there by closed-form offset counting, Appendix A.1).
def _load_golden():
    kinds = {"F": PT.FAR, "N": PT.NBR, "S": PT.SIB, "D": PT.LNBR}
    etas = {"1": 1.0, "sqrt2": np.sqrt(2.0), "sqrt3": np.sqrt(3.0)}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "partition_counts.txt")
    rows = []
    for line in open(path):
        line = line.split("#", 1)[0].split()
        if not line:
            continue
        d, L, eta, s = int(line[0]), int(line[1]), etas[line[2]], line[3]
        s = PT.SWITCH_NONE if s == "none" else int(s)
        counts = {}
        for tok in line[4:]:
            lv, kc = tok.split(":")
            counts[(int(lv[1:]), kinds[kc[0]])] = int(kc[1:])
        rows.append((d, L, eta, s, counts))
    return rows


GOLDEN = _load_golden()
assert len(GOLDEN) == 17


@pytest.mark.parametrize("d,L,eta,s,counts", GOLDEN)
def test_golden_grid_counts(d, L, eta, s, counts):
    tr = _grid_tree(d, L)
    assert tr.L == L
    part = PT.build_partition(tr, eta, s)
    got = {}
    for l, k in zip(part.level.tolist(), part.kind.tolist()):
        if k != PT.DIAG:
            got[(l, k)] = got.get((l, k), 0) + 1
    assert got == counts
    assert int(np.sum(part.kind == PT.DIAG)) == 1 << (d * L)
