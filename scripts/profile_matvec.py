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
cfg = W.CONFIGS.get(name) or W.SMALL_CONFIGS[name]
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
hh.hh_matvec(H, x, y, nrhs)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e)
print(f"matvec {ms:.3f} ms  {info['stored_bytes'] / ms / 1e6:.1f} GB/s  |y| {float(torch.linalg.norm(y)):.6e}")
