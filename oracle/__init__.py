"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy/scipy, float64) of the
adaptive mixed-precision H_h matrix and its matrix-vector product, written from the
paper (arxiv 2604.09147, /root/reference/PAPER.md) step by step:

  tree.py       balanced 2^d-tree, depth rule, Morton order
  partition.py  standard / weak / hybrid admissibility, Eq. 3.1
  kernels.py    kernel-matrix entries, Eq. 5.1
  compress.py   truncated SVD to relative Frobenius eps
  formats.py    Table 1 formats, RNE rounding
  hmatrix.py    Alg. 1 (H_h) + Alg. 4 (norms) + Alg. 2 (AMP)
  pack.py       arena packing function            (our layout; no paper passage)
  matvec.py     Alg. 3 (H-hat x)
  dense.py      dense A x and ||A||_F (definition)
  metrics.py    error metrics and the Thm 4.2 / 4.4 bounds

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference
leg may import anything under ``oracle/``.  The product package
(``paper_2604_09147_b200``) never imports it, and this package never imports the
product package; the only shared module is ``workloads`` (seeded input generators,
no method arithmetic).

Parity status per function (details in DESIGN.md §6): every function here is pinned by
a ``-m "not gpu"`` test in tests/test_oracle_*.py EXCEPT: exact per-block ranks/tags at
3D scale (no printed ranks in the paper) — "parity unpinned" beyond the sampled checks.
"""
