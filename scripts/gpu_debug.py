"""Quick GPU diagnostics: build a config, compare with the oracle, print stats."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import workloads as W
import parity_lib as PL
from paper_2604_09147_b200 import hh

name = sys.argv[1] if len(sys.argv) > 1 else "2d_tiny"
cfg = W.SMALL_CONFIGS.get(name) or W.CONFIGS[name]
P = W.make_points(cfg)
t = time.time()
H = PL.gpu_build(P, cfg)
print("build s", time.time() - t, flush=True)
info = hh.hh_info(H)
print({k: info[k] for k in ("L", "nblocks", "n_lowrank", "n_dense", "total_rank", "norm2", "stored_bytes", "padded_bytes", "n_retry", "build_seconds", "c_far", "c_nbr", "c_sib")}, flush=True)
print("stored by tag", info["stored_bytes_tag"], flush=True)
x = W.make_rhs(cfg)
y = PL.gpu_matvec(H, x)
print("y norm", np.linalg.norm(y), flush=True)
if cfg["N"] <= 10000:
    ex = PL.export(H)
    Ho = PL.oracle_build(P, cfg)
    try:
        PL.check_partition(ex, Ho); print("1a ok")
    except AssertionError as e:
        print("1a FAIL", str(e)[:500])
    print("1b", PL.rank_tag_parity(ex, Ho))
    print("norm2 gpu/oracle", ex["info"]["norm2"], Ho.norm2)
    try:
        lay = PL.check_packing(ex); print("1c ok")
        yo = PL.oracle_matvec_on_export(ex, lay, x)
        print("check2 rel", PL.rel2(y, yo))
    except AssertionError as e:
        print("1c FAIL", str(e)[:800])
    from oracle import dense as D, metrics as M
    Ax, fro2 = D.dense_apply(P, cfg["kernel"], cfg["scale"], x)
    print("e_mv", M.e_mv(Ax, y, np.sqrt(fro2), x), "eps", cfg["eps"])
