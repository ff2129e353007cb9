#!/usr/bin/env python
"""NEXT-3: the paper's backward-error experiment (Fig. 9) on the B200.

    python scripts/backward_error.py [--out profiles/r02_backward_error.json]

3D 1/r on [-1,1]^3, x ~ U(0,1), N = 8000 (L = 2) and N = 64000 (L = 3), ell = L - 1,
eta = sqrt(3), adaptive mixed precision {fp64, fp32, fp16, bf16}; for eps = 1e-2 .. 1e-10 the
relative backward error ||Hx - b|| / (||H||_F ||x||) of b = H-hat x computed by hh_matvec_wp in
fp64 / fp32 / fp16, next to the Thm 4.4 bound (measured sparsity constants) and, at N = 8000,
the oracle twin's error (oracle/matvec_wp.py on the exported factors).  Dense H x by definition
(oracle/dense.py)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "backward_error.json"))
    ap.add_argument("--configs", default="3d_fig9_8000,3d_fig9_64000")
    ap.add_argument("--oracle-max-n", type=int, default=8000)
    args = ap.parse_args()
    import torch
    import parity_lib as PL
    import test_gpu_wp as T
    from oracle import dense as D
    from oracle import matvec_wp as OW
    from oracle import metrics as M
    from paper_2604_09147_b200 import hh
    out = []
    for name in args.configs.split(","):
        cfg0 = W.FIG9_CONFIGS[name]
        P = W.make_points(cfg0)
        x = W.make_rhs(cfg0, 1)
        t0 = time.time()
        Ax, fro2 = D.dense_apply(P, cfg0["kernel"], cfg0["scale"], x, chunk=128)
        t_dense = time.time() - t0
        for eps in W.FIG9_EPS:
            cfg = dict(cfg0, eps=eps)
            H = PL.gpu_build(P, cfg)
            info = hh.hh_info(H)
            rec = {"config": name, "N": cfg["N"], "L": info["L"], "ell": cfg["s"], "eps": eps,
                   "stored_bytes": info["stored_bytes"], "stored_bytes_by_tag": info["stored_bytes_tag"],
                   "thm44_bound": M.thm44_factor(info["L"], cfg["s"], info["c_far"], info["c_nbr"], info["c_sib"]) * eps,
                   "sparsity_constants": [info["c_far"], info["c_nbr"], info["c_sib"]], "e_mv": {}, "e_mv_oracle": {}}
            ex = None
            for wp, nm in ((OW.WP_FP64, "fp64"), (OW.WP_FP32, "fp32"), (OW.WP_FP16, "fp16")):
                y = T.gpu_matvec_wp(H, x, wp)
                rec["e_mv"][nm] = float(M.e_mv(Ax, y, np.sqrt(fro2), x)[0])
                if cfg["N"] <= args.oracle_max_n and wp != OW.WP_FP64:
                    if ex is None:
                        ex = PL.export(H)
                        lay = PL.check_packing(ex)
                        blocks = list(PL.exported_blocks(ex, lay))
                    yo = OW.matvec_blocks_wp(cfg["N"], ex["perm"].astype(np.int64), blocks, x, wp)
                    rec["e_mv_oracle"][nm] = float(M.e_mv(Ax, yo, np.sqrt(fro2), x)[0])
            hh.hh_free(H)
            torch.cuda.synchronize()
            print(json.dumps(rec), flush=True)
            out.append(rec)
        print(f"# {name}: dense reference {t_dense:.1f} s", flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"how": __doc__, "records": out}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
