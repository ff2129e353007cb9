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
  matvec_wp.py  Alg. 3 in fp32 / fp16 working precision (G27)
  switch_level.py  Alg. 5 (switching level l*)
  dense.py      dense A x and ||A||_F (definition)
  metrics.py    error metrics and the Thm 4.2 / 4.4 bounds

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference
leg may import anything under ``oracle/``.  The product package
(``paper_2604_09147_b200``) never imports it, and this package never imports the
product package; the only shared module is ``workloads`` (seeded input generators,
no method arithmetic).

Pins per function (all ``-m "not gpu"``; each is a closed form, a worked example, a printed
value or a brute force — never a retyping of the function):
  tree.build_tree / cells / morton       quadrant-centre worked example, minimal depth
                                         by direct counting, boxes are geometric   test_oracle_tree_partition
  partition.build_partition              N^2 coverage marking, pairwise brute force, golden grid
                                         counts, s=0==s=1==HODLR, s=NONE==standard   test_oracle_tree_partition
  partition.sparsity_constants           27/8, 189/26/7, plain-loop
                                         counts on random trees                       test_oracle_pins
  kernels.f_of_r / block                 closed forms (log e = 1, 1/2, 1/4, e^-1, e^-1/2), 3-4-5
                                         distances, index-keyed diagonal, coincident count  test_oracle_pins
  compress.lr_compress / truncation_rank 4x4 identity eps=1/2 -> 3, rank 1, zero,
                                         exact rational tails, minimality, two LAPACK drivers  test_oracle_hmatrix
  formats.round_rne / to_storage_bits    brute-force enumeration, numpy direct casts, bf16(0.1),
                                         fp16(70000)=inf             test_oracle_formats
  hmatrix.choose_tag                     worked example eps=1e-4 d=2 l=4 xi=1e-3 -> bf16,
                                         monotone in eps, fp64-only at eps<=1e-10  test_oracle_hmatrix
  hmatrix.guard_tag                      every format's RNE overflow boundary (Table 1 x_max),
                                         promotion end to end on a 1e-20 domain        test_oracle_pins
  hmatrix.tag_blocks (beneficial rule)   PAPER.md:992 125x125 rank-64 example; through build:
                                         dense-kept violate / low-rank-kept satisfy, both occur  test_oracle_pins
  hmatrix.alg4_norm2 / build             Lemma 4.1 densely, Alg. 4 norm == dense reconstruction,
                                         Thm 4.2                                       test_oracle_hmatrix
  switch_level.walk / alg_lstar          hand-worked walks (stop behind a dip), brute-force argmax
                                         over every level; Table 3 S1/S2 = 1.60
                                         sampled (default) and full (--runslow)        test_oracle_pins
  pack.pack                              no byte written twice, round trip, z contiguity  test_oracle_hmatrix
                                         (our layout: no paper passage; the C++ twin is compared in test_host_logic)
  matvec.matvec                          dense reconstruction, L=0 dense gemv, Thm 4.4  test_oracle_hmatrix
  matvec_wp.matvec_wp (NEXT-3, G27)      hand-worked fp16/fp32 sums (2049 ones -> 2048), operands
                                         rounded once, exact on integer data, within the a priori
                                         rounding bound of the exact product           test_oracle_matvec_wp
  dense / metrics                        definitions; bound constants at eta=sqrt(d) = 27/8/3, 189/26/7

Parity unpinned: exact per-block ranks and tags at 3D scale (the paper prints none) — checked
on stratified samples against LAPACK (tests/test_gpu_fullsize.py), not pinned to a printed value.
"""
