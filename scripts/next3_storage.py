"""NEXT-3 storage table: stored bytes per precision set (ledger-only device builds).

    python scripts/next3_storage.py [--out profiles/r02_next3_storage.json]

For BASELINE-shaped workloads the adaptive rule (Eq. 4.4) is evaluated with
the paper's set {fp64, fp32, fp16, bf16}, with Table 1's q43 added and with the
byte-granular accessor formats bf24 / fp48 added.  Nothing is stored
(HH_LEDGER_ONLY); the ledger is the metric the paper reports.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2604_09147_b200 import hh  # noqa: E402

SETS = [("fp64", W.P_FP64), ("paper set", W.P_MIXED), ("+q43", W.P_MIXED_Q43), ("+q43+bf24+fp48", W.P_ACCESSOR)]
CASES = [("2d_medium", W.CONFIGS["2d_medium"], [1e-8, 1e-4, 1e-2]),
         ("3d_laplace", W.CONFIGS["3d_laplace"], [1e-6, 1e-4, 1e-2])]
TAGS = ["fp64", "fp32", "fp16", "bf16", "q43", "bf24", "fp48", "dense_fp64"]


def main():
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    recs = []
    for name, cfg, epss in CASES:
        P = torch.from_numpy(W.make_points(cfg)).cuda()
        for eps in epss:
            for label, pset in SETS:
                H = hh.hh_build(P, cfg["kernel"], cfg["scale"], eps, cfg["eta"], cfg["leaf"], cfg["s"],
                                pset | hh.LEDGER_ONLY)
                info = hh.hh_info(H)
                hh.hh_free(H)
                by = {t: int(b) for t, b in zip(TAGS, info["stored_bytes_tag"]) if b}
                rec = dict(config=name, eps=eps, precision_set=label, stored_bytes=int(info["stored_bytes"]),
                           by_tag=by)
                recs.append(rec)
                print(json.dumps(rec), flush=True)
    if out:
        json.dump(dict(how=__doc__, records=recs), open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
