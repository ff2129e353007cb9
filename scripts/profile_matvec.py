"""Build one workload through the C-ABI and run hh_matvec a few times (ncu driver).

    python scripts/profile_matvec.py [config] [nrhs] [iters]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2604_09147_b200 import hh  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "3d_laplace"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = W.CONFIGS.get(name) or W.SMALL_CONFIGS.get(name) or W.PROXY_CONFIGS[name]
P = torch.from_numpy(W.make_points(cfg)).cuda()
t = time.time()
H = hh.hh_build(P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"], cfg["s"], cfg["pset"])
torch.cuda.synchronize()
info = hh.hh_info(H)
print(f"build {time.time() - t:.1f}s stored {info['stored_bytes']} nblocks {info['nblocks']}", flush=True)
x = torch.from_numpy(W.make_rhs(cfg, nrhs).T.copy()).cuda().T
y = torch.empty_like(x.T).T
for _ in range(iters):
    hh.hh_matvec(H, x, y, nrhs)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
hh.hh_matvec_timing(H)
hh.hh_matvec_profile(H, True)
reps = 5
for _ in range(reps):
    hh.hh_matvec(H, x, y, nrhs)
e.record()
torch.cuda.synchronize()
hh.hh_matvec_profile(H, False)
ph, cnt = hh.hh_matvec_timing(H)
ms = s.elapsed_time(e) / reps
ex = hh.hh_export(H, tables=True, arenas=False)
B = ex["blocks"]
ls = ex["leaf_start"]
sh = info["d"] * (info["L"] - B["level"].astype(np.int64))
m = ls[(B["tgt"] + 1) << sh] - ls[B["tgt"] << sh]
n = ls[(B["src"] + 1) << sh] - ls[B["src"] << sh]
wb = np.array([8, 4, 2, 2, 1, 3, 6])[B["tag"]]
lr = B["storage"] == 0
p = B["rank"].astype(np.int64)
w1 = int(np.sum((p * n * wb)[lr]))
w2 = int(np.sum((p * m * wb)[lr])) + int(np.sum((m * n * 8)[~lr]))
p1, p2 = ph[1] / cnt, ph[2] / cnt
print(f"{name} nrhs={nrhs}: matvec {ms:.3f} ms  {info['stored_bytes'] / ms / 1e6:.1f} GB/s | phase1 {p1:.3f} ms "
      f"{w1 / p1 / 1e6:.1f} GB/s | phase2 {p2:.3f} ms {w2 / p2 / 1e6:.1f} GB/s | |y| {float(torch.linalg.norm(y)):.9e}")
