"""BASELINE config 4 — admissibility sweep (and the storage-ratio context of configs 2/3).

    python scripts/sweep.py [--n N] [--reps R] [--out profiles/r01_sweep.jsonl]

3D N=262144 uniform points, 1/r (diagonal 0), leaf 128, eta=1, eps=1e-6; switch level in
{none (pure standard H), 2, 3, 4, 0 (pure HODLR)}, each in uniform fp64 and adaptive mixed
precision.  Per setting: stored bytes, blocks, build seconds, matvec GB/s (CUDA events, 3
warm-ups, inputs larger than L2 or labelled), and the approximation error e_mv estimated
on sampled rows of the dense product (oracle rows; ||A||_F^2 estimated from the same rows).
Also `--ledger-3d-large`: a ledger-only build (HH_LEDGER_ONLY, no factors stored) of the
uniform-fp64 standard-admissibility H at N=2^20 for the storage ratio of config 3.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2604_09147_b200 import hh  # noqa: E402


def time_matvec(H, x, y, reps):
    for _ in range(3):
        hh.hh_matvec(H, x, y, 1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        hh.hh_matvec(H, x, y, 1)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def sampled_emv(P, cfg, x_h, y_h, nrows=48, seed=9):
    from oracle import dense as D   # test/report infrastructure: the oracle's dense rows
    rng = np.random.default_rng(seed)
    N = cfg["N"]
    rows = rng.choice(N, size=nrows, replace=False)
    Ax, fro2_rows = D.dense_apply(P, cfg["kernel"], cfg["scale"], x_h, rows=rows, chunk=8)
    r2 = float(np.sum((Ax[:, 0] - y_h[rows, 0]) ** 2))
    return float(np.sqrt(r2 / fro2_rows) / np.linalg.norm(x_h[:, 0]) * 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep.jsonl"))
    ap.add_argument("--ledger-3d-large", action="store_true")
    args = ap.parse_args()
    out = open(args.out, "a")
    if args.ledger_3d_large:
        cfg = dict(W.CONFIGS["3d_large"])
        P = torch.from_numpy(W.make_points(cfg)).cuda()
        for s, pset in ((W.SWITCH_NONE, W.P_FP64), (cfg["s"], W.P_FP64)):
            t = time.time()
            H = hh.hh_build(P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"], s,
                            pset | hh.LEDGER_ONLY)
            info = hh.hh_info(H)
            rec = {"config": "3d_large", "switch_level": "none" if s < 0 else s, "precision": "fp64",
                   "ledger_only": True, "stored_bytes": info["stored_bytes"], "nblocks": info["nblocks"],
                   "build_s": round(time.time() - t, 1)}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
            hh.hh_free(H)
        return
    cfg0 = W.CONFIGS["sweep"]
    P_h = W.make_points(cfg0)
    P = torch.from_numpy(P_h).cuda()
    x_h = W.make_rhs(cfg0, 1)
    x = torch.from_numpy(x_h.T.copy()).cuda().T
    y = torch.empty_like(x.T).T
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for s in W.SWEEP_SWITCH_LEVELS:
        for pname, pset in (("fp64", W.P_FP64), ("mixed", W.P_MIXED)):
            cfg = dict(cfg0, s=s, pset=pset)
            t = time.time()
            H = hh.hh_build(P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"], s, pset)
            torch.cuda.synchronize()
            bs = time.time() - t
            info = hh.hh_info(H)
            ms = time_matvec(H, x, y, args.reps)
            y_h = y.cpu().numpy()
            e = sampled_emv(P_h, cfg, x_h, y_h)
            rec = {"config": "sweep", "switch_level": "none" if s < 0 else s, "precision": pname,
                   "stored_bytes": info["stored_bytes"], "stored_by_tag": info["stored_bytes_tag"],
                   "nblocks": info["nblocks"], "L": info["L"], "build_s": round(bs, 1),
                   "matvec_ms": round(ms, 4), "GBps": round(info["stored_bytes"] / ms / 1e6, 1),
                   "cache": "inputs larger than L2" if info["stored_bytes"] > 4 * l2 else "L2-resident",
                   "e_mv_sampled": e, "eps": cfg["eps"]}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
            hh.hh_free(H)


if __name__ == "__main__":
    main()
