"""The library's host-side C++ (partition expansion, packing function) against the oracle on
CPU — no device: hh_selftest_partition / hh_selftest_layout run the same code hh_build runs.

(1a) on random trees (random leaf occupancies incl. empty leaves, reading G20) for d = 1, 2,
3, eta in {1, sqrt(2), sqrt(3)}, every switch level and HH_SWITCH_NONE: the block table
(level, kind, tgt, src) equals the oracle's partition of a tree with the same leaf offsets.
(1c) on random ranks / tags / storage kinds over those partitions: every offset equals the
oracle's packing function (oracle/pack.py), bit for bit.
"""
import numpy as np
import pytest

from oracle import pack as PK
from oracle import partition as PT
from oracle import tree as T

hh = pytest.importorskip("paper_2604_09147_b200.hh")


def _tree(d, L, rng, p_empty=0.3, mean=5):
    ncell = 1 << (d * L)
    counts = rng.poisson(mean, ncell) * (rng.random(ncell) > p_empty)
    ls = np.zeros(ncell + 1, np.int64)
    ls[1:] = np.cumsum(counts)
    return T.Tree(d=d, L=L, lo=np.zeros(d), side=1.0, perm=np.arange(ls[-1], dtype=np.int64),
                  keys=np.zeros(ls[-1], np.int64), leaf_start=ls)


CASES = [(1, 6, 1.0), (2, 4, 1.0), (2, 4, float(np.sqrt(2.0))), (3, 3, 1.0), (3, 3, float(np.sqrt(3.0))), (2, 5, 1.0)]


@pytest.mark.parametrize("d,L,eta", CASES)
def test_partition_matches_oracle(d, L, eta):
    rng = np.random.default_rng(100 * d + L)
    for trial in range(2):
        tr = _tree(d, L, rng, p_empty=0.0 if trial == 0 else 0.35)
        for s in [PT.SWITCH_NONE] + list(range(0, L + 1)):
            ref = PT.build_partition(tr, eta, s)
            got = hh.selftest_partition(tr.leaf_start, d, L, eta, s)
            assert got["level"].size == len(ref), (d, L, eta, s)
            for f, r in (("level", ref.level), ("kind", ref.kind), ("tgt", ref.tgt), ("src", ref.src)):
                np.testing.assert_array_equal(got[f].astype(np.int64), r, err_msg=f"{f} d={d} L={L} s={s}")


@pytest.mark.parametrize("d,L,eta", CASES[:4])
def test_packing_function_matches_oracle(d, L, eta):
    rng = np.random.default_rng(7 + d * L)
    tr = _tree(d, L, rng, p_empty=0.25, mean=9)
    for s in (PT.SWITCH_NONE, max(0, L - 1), 1):
        part = PT.build_partition(tr, eta, s)
        nb = len(part)
        dense = (part.kind == PT.DIAG) | ((part.kind == PT.LNBR) & (rng.random(nb) < 0.5))
        storage = dense.astype(np.uint8)
        rank = np.where(dense, 0, rng.integers(0, 40, nb)).astype(np.int32)
        rank[rng.random(nb) < 0.05] = 0                      # some rank-0 low-rank blocks
        tag = np.where(dense, 0, rng.integers(0, 7, nb)).astype(np.uint8)
        ref = PK.pack(tr.leaf_start, d, L, part.level, part.tgt, part.src, rank, tag, storage)
        got = hh.selftest_layout(tr.leaf_start, d, L, part.level, part.tgt, part.src, rank, tag, storage)
        lr = storage == 0
        has = lr & (rank > 0)
        np.testing.assert_array_equal(got["zoff"][lr], ref["zoff"][lr])
        np.testing.assert_array_equal(got["w_off"][has], ref["w_off"][has])
        np.testing.assert_array_equal(got["wcol"][has], ref["wcol"][has])
        np.testing.assert_array_equal(got["ucol"][has], ref["ucol"][has])
        np.testing.assert_array_equal(got["d_off"][~lr], ref["d_off"][~lr])
        np.testing.assert_array_equal(got["u_leaf_off"], ref["u_leaf_off"])
        np.testing.assert_array_equal(got["d_leaf_off"], ref["d_leaf_off"])
        np.testing.assert_array_equal(got["w_bytes"], ref["w_bytes"])


@pytest.mark.parametrize("d,L,eta", [(2, 3, 1.0), (3, 2, 1.0), (1, 5, 1.0)])
def test_tagging_matches_oracle(d, L, eta):
    """Alg. 4 norm + Alg. 2 tags (Eq. 4.4 squared form, range guard, tie rule, PAPER.md:992
    beneficial rule): the library's host C++ (layout.cpp assign_tags via hh_selftest_tags) equals
    the oracle's tag_blocks on random block tables whose norms span every format's threshold
    and whose factor maxima straddle every format's overflow boundary."""
    from oracle import hmatrix as HM
    rng = np.random.default_rng(11 * d + L)
    tr = _tree(d, L, rng, p_empty=0.2, mean=7)
    edges = [240.0, 247.99, 248.0, 65504.0, 65519.99, 65520.0, float.fromhex("0x1.fffe8p127"),
             float.fromhex("0x1.ffffp127"), float.fromhex("0x1.fep127"), float.fromhex("0x1.ffp127"),
             float.fromhex("0x1.fffffep127"), float.fromhex("0x1.ffffffp127"), 1e39, 1e300]
    for s in (PT.SWITCH_NONE, max(0, L - 1)):
        part = PT.build_partition(tr, eta, s)
        nb = len(part)
        sh = d * (L - part.level)
        m = tr.leaf_start[(part.tgt + 1) << sh] - tr.leaf_start[part.tgt << sh]
        n = tr.leaf_start[(part.src + 1) << sh] - tr.leaf_start[part.src << sh]
        rank = np.minimum(rng.integers(0, 24, nb), np.minimum(m, n))
        tot = np.exp(rng.uniform(-30, 5, nb))
        nb2 = tot * (1 - rng.uniform(0, 1e-6, nb))
        maxabs = np.exp(rng.uniform(-5, 12, nb))
        hit = rng.random(nb) < 0.15
        maxabs[hit] = rng.choice(edges, int(hit.sum()))
        for pset in (W_MIXED, W_MIXED | (1 << 17), 1 | 4, 1 | 8, 1 | 2 | 8, 1 | 4 | 8 | (1 << 17), 1, W_MIXED | 16, 1 | 16, 1 | 4 | 16, 127, 1 | 32 | 64,
                     W_MIXED | 32, 1 | 2 | 64):
            # hh_build compresses every block except leaf diagonals (and leaf neighbours when uniform)
            dense0 = (part.kind == PT.DIAG) | ((part.kind == PT.LNBR) & ((pset & 15) == 1))
            rk = np.where(dense0, 0, rank)
            for eps in (1e-2, 1e-6):
                ref = HM.tag_blocks(d, part.level, part.kind, m, n, rk, nb2, tot, maxabs, eps, pset)
                got = hh.selftest_tags(tr.leaf_start, d, L, part.level, part.kind, part.tgt, part.src, rk,
                                       nb2, tot, maxabs, eps, pset)
                tagm = ref["storage"] == 0
                np.testing.assert_array_equal(got["storage"], ref["storage"], err_msg=f"storage s={s} pset={pset}")
                np.testing.assert_array_equal(got["rank"], ref["rank"], err_msg="rank")
                np.testing.assert_array_equal(got["tag"][tagm], ref["tag"][tagm], err_msg=f"tag s={s} pset={pset}")
                assert got["norm2"] == ref["norm2"]
                assert (got["n_fallback"], got["n_promoted"]) == (ref["fallback"], ref["promoted"]), (pset, eps)
                if pset == W_MIXED and eps == 1e-2:
                    assert ref["promoted"] > 0 and len(set(ref["tag"][tagm])) >= 3


W_MIXED = 15
