"""Seeded synthetic workloads shared by the oracle, the tests and bench.py.

This module holds ONLY input generation (points, right-hand sides) and the
parameter dictionaries of the BASELINE.json configs.  It contains none of the
method's arithmetic, so both sides of every parity check (the CPU oracle in
``oracle/`` and the CUDA path in ``paper_2604_09147_b200``) may import it
without sharing any implementation.

Point sets stand in for the paper's P_square workload (PAPER.md:1090,
"N particles uniformly distributed within the hypercube [-1,1]^d"); the
BASELINE configs place them in [0,1]^d, the paper's experiments in [-1,1]^d.
Seeds: points ``default_rng(1000 + k)``, right-hand sides ``default_rng(2000 + k)``
for config index k in BASELINE order.
"""
from __future__ import annotations

import numpy as np

# kernel ids — identical numbering is part of the C-ABI (include/hh.h)
K_LOG, K_INV_R, K_INV_R2, K_GAUSS, K_EXP = 0, 1, 2, 3, 4
KERNEL_NAMES = {K_LOG: "log", K_INV_R: "inv_r", K_INV_R2: "inv_r2", K_GAUSS: "gauss", K_EXP: "exp"}

# precision-set bitmask — identical to include/hh.h
P_FP64, P_FP32, P_FP16, P_BF16 = 1, 2, 4, 8
P_MIXED = P_FP64 | P_FP32 | P_FP16 | P_BF16
TIE_FP16 = 1 << 17      # precision_set flag: bits-aware fp16-over-bf16 tie rule (NEXT-3)
SWITCH_NONE = -1


def points_uniform(n: int, d: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """N i.i.d. uniform points in [lo,hi]^d, float64, shape (n, d), row-major."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(lo + (hi - lo) * rng.random((n, d)), dtype=np.float64)


def points_sphere(n: int, d: int, seed: int) -> np.ndarray:
    """N points on the surface of the unit hypersphere in R^d (the paper's P_circ set,
    PAPER.md:1091): normalised standard-normal vectors (uniform on the sphere), float64."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, d))
    return np.ascontiguousarray(g / np.linalg.norm(g, axis=1, keepdims=True), dtype=np.float64)


def points_grid_centres(d: int, L: int) -> np.ndarray:
    """One point at the centre of every cell of a 2^L-per-axis grid (used by golden
    partition pins: with n_max=1 the depth rule yields exactly L and no empty cell)."""
    m = 1 << L
    axes = [(np.arange(m) + 0.5) / m for _ in range(d)]
    g = np.meshgrid(*axes, indexing="ij")
    return np.ascontiguousarray(np.stack([a.ravel() for a in g], axis=1), dtype=np.float64)


def rhs(n: int, nrhs: int, seed: int, dist: str) -> np.ndarray:
    """Right-hand sides, float64, shape (n, nrhs) in Fortran (column-major) order."""
    rng = np.random.default_rng(seed)
    if dist == "uniform_pm1":
        x = rng.uniform(-1.0, 1.0, size=(nrhs, n))
    elif dist == "uniform_01":
        x = rng.uniform(0.0, 1.0, size=(nrhs, n))
    elif dist == "normal":
        x = rng.standard_normal(size=(nrhs, n))
    else:
        raise ValueError(dist)
    return np.asfortranarray(x.T)


# BASELINE.json configs, in order (index k drives the seeds).
CONFIGS = {
    "2d_tiny": dict(k=0, N=4096, d=2, kernel=K_LOG, scale=1.0, leaf=64, eta=1.0, s=3,
                    eps=1e-8, pset=P_MIXED, nrhs=1, xdist="uniform_pm1"),
    "2d_medium": dict(k=1, N=65536, d=2, kernel=K_LOG, scale=1.0, leaf=64, eta=1.0, s=5,
                      eps=1e-8, pset=P_MIXED, nrhs=1, xdist="uniform_pm1"),
    "3d_laplace": dict(k=2, N=262144, d=3, kernel=K_INV_R, scale=1.0, leaf=128, eta=1.0, s=3,
                       eps=1e-6, pset=P_MIXED, nrhs=1, xdist="normal"),
    "3d_large": dict(k=3, N=1 << 20, d=3, kernel=K_EXP, scale=0.1, leaf=128, eta=1.0, s=4,
                     eps=1e-6, pset=P_MIXED, nrhs=1, xdist="normal"),
    "sweep": dict(k=4, N=262144, d=3, kernel=K_INV_R, scale=1.0, leaf=128, eta=1.0, s=3,
                  eps=1e-6, pset=P_MIXED, nrhs=1, xdist="normal"),
}
SWEEP_SWITCH_LEVELS = [SWITCH_NONE, 2, 3, 4, 0]

# Small parity configs the oracle finishes in seconds; they exercise every storage
# format (Fig. 8 uses eps=1e-4 and 1e-2 to reach fp16/bf16).
SMALL_CONFIGS = {
    "2d_tiny": CONFIGS["2d_tiny"],
    "2d_fig8_e4": dict(k=10, N=6400, d=2, kernel=K_LOG, scale=1.0, leaf=64, eta=1.0, s=3,
                       eps=1e-4, pset=P_MIXED, nrhs=1, xdist="uniform_pm1", lo=-1.0, hi=1.0),
    "2d_fig8_e2": dict(k=11, N=6400, d=2, kernel=K_LOG, scale=1.0, leaf=64, eta=1.0, s=3,
                       eps=1e-2, pset=P_MIXED, nrhs=1, xdist="uniform_pm1", lo=-1.0, hi=1.0),
    "3d_small_inv_r": dict(k=12, N=8000, d=3, kernel=K_INV_R, scale=1.0, leaf=128, eta=1.0, s=2,
                           eps=1e-6, pset=P_MIXED, nrhs=1, xdist="normal"),
    "3d_small_exp": dict(k=13, N=8000, d=3, kernel=K_EXP, scale=0.1, leaf=64, eta=1.0, s=2,
                         eps=1e-6, pset=P_MIXED, nrhs=4, xdist="normal"),
    # d = 1 (binary tree; the method is stated for any d)
    "1d_log": dict(k=16, N=2000, d=1, kernel=K_LOG, scale=1.0, leaf=32, eta=1.0, s=2,
                   eps=1e-8, pset=P_MIXED, nrhs=1, xdist="uniform_pm1"),
    # NEXT-4: points on the unit sphere (App. D) — most
    # leaf boxes empty, unbalanced occupancy (reading G20: empty clusters are skipped)
    "3d_sphere_small": dict(k=14, N=8000, d=3, kernel=K_INV_R, scale=1.0, leaf=64, eta=1.0, s=3,
                            eps=1e-6, pset=P_MIXED, nrhs=1, xdist="normal", points="sphere"),
    "2d_circle_small": dict(k=15, N=6000, d=2, kernel=K_LOG, scale=1.0, leaf=32, eta=1.0, s=3,
                            eps=1e-4, pset=P_MIXED, nrhs=1, xdist="uniform_pm1", points="sphere"),
}


# Iteration proxy for the 3D N=2^20 config (same kernel, eps, leaf occupancy ~32; 8x fewer
# points so it builds in seconds).  Not a BASELINE config: used by scripts/profile_matvec.py.
PROXY_CONFIGS = {
    # NEXT-4 at scale: 3D unit sphere surface, N=2^18, 1/r, eps=1e-6 (bench with --config)
    "3d_sphere": dict(k=21, N=262144, d=3, kernel=K_INV_R, scale=1.0, leaf=128, eta=1.0, s=4,
                      eps=1e-6, pset=P_MIXED, nrhs=1, xdist="normal", points="sphere"),
    "3d_exp_proxy": dict(k=20, N=131072, d=3, kernel=K_EXP, scale=0.1, leaf=64, eta=1.0, s=3,
                         eps=1e-6, pset=P_MIXED, nrhs=1, xdist="normal"),
}


def make_points(cfg: dict) -> np.ndarray:
    if cfg.get("points") == "sphere":
        return points_sphere(cfg["N"], cfg["d"], 1000 + cfg["k"])
    return points_uniform(cfg["N"], cfg["d"], 1000 + cfg["k"], cfg.get("lo", 0.0), cfg.get("hi", 1.0))


def make_rhs(cfg: dict, nrhs: int | None = None) -> np.ndarray:
    return rhs(cfg["N"], nrhs or cfg["nrhs"], 2000 + cfg["k"], cfg["xdist"])

# NEXT-3: Table 1's 8-bit q43 as an extra storage format (precision_set bit 16, include/hh.h)
P_Q43 = 16
P_MIXED_Q43 = P_MIXED | P_Q43
SMALL_CONFIGS["2d_fig8_e2_q43"] = dict(SMALL_CONFIGS["2d_fig8_e2"], k=17, pset=P_MIXED_Q43)
SMALL_CONFIGS["3d_small_exp_q43"] = dict(SMALL_CONFIGS["3d_small_exp"], k=18, eps=1e-3, pset=P_MIXED_Q43)

# NEXT-3 backward-error study (Fig. 9): 3D 1/r on P_square = [-1,1]^3,
# x ~ U(0,1); L = 2 at N = 8000 and L = 3 at N = 64000 (n_max = 125 in the paper's balanced
# formula; the depth rule of reading G1 gives those depths with leaf 250), ell = L - 1,
# eta = sqrt(3) (the paper's 3D setting); eps swept by the experiment.
FIG9_CONFIGS = {
    "3d_fig9_8000": dict(k=19, N=8000, d=3, kernel=K_INV_R, scale=1.0, leaf=250, eta=float(np.sqrt(3.0)), s=1,
                         eps=1e-6, pset=P_MIXED, nrhs=1, xdist="uniform_01", lo=-1.0, hi=1.0),
    "3d_fig9_64000": dict(k=22, N=64000, d=3, kernel=K_INV_R, scale=1.0, leaf=250, eta=float(np.sqrt(3.0)), s=2,
                          eps=1e-6, pset=P_MIXED, nrhs=1, xdist="uniform_01", lo=-1.0, hi=1.0),
}
FIG9_EPS = [1e-2, 1e-4, 1e-6, 1e-8, 1e-10]

# NEXT-3: the accessor continuum at byte granularity: bf24 (3 B, u = 2^-16) and
# fp48 (6 B, u = 2^-37) between the Table 1 formats (precision_set bits 32 and 64)
P_BF24, P_FP48 = 32, 64
P_ACCESSOR = P_MIXED | P_Q43 | P_BF24 | P_FP48
SMALL_CONFIGS["3d_small_inv_r_acc"] = dict(SMALL_CONFIGS["3d_small_inv_r"], k=23, pset=P_ACCESSOR)
SMALL_CONFIGS["2d_tiny_acc"] = dict(CONFIGS["2d_tiny"], k=24, eps=1e-10, pset=P_ACCESSOR)
