"""Cycle probe of the NR = 1 matvec pipelines (needs a -DHH_MV_PROBE=1 variant build).

    python -m paper_2604_09147_b200.build --variant probe -DHH_MV_PROBE=1
    HH_LIB=$PWD/paper_2604_09147_b200/libhh_probe.so python scripts/probe_matvec.py [config]

Prints, per phase, how the producer thread and one consumer thread of every CTA spend their
cycles (sums over CTAs and matvecs): waiting on barriers vs working, stages and items.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2604_09147_b200 import hh  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "2d_medium"
cfg = W.CONFIGS.get(name) or W.SMALL_CONFIGS.get(name) or W.PROXY_CONFIGS[name]
lib = C.CDLL(os.environ["HH_LIB"])
P = torch.from_numpy(W.make_points(cfg)).cuda()
H = hh.hh_build(P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"], cfg["s"], cfg["pset"])
x = torch.from_numpy(W.make_rhs(cfg, 1).T.copy()).cuda().T
y = torch.empty_like(x.T).T
for _ in range(3):
    hh.hh_matvec(H, x, y, 1)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
assert lib.hh_debug_probe(buf, 1) == 0
reps = 10
for _ in range(reps):
    hh.hh_matvec(H, x, y, 1)
torch.cuda.synchronize()
assert lib.hh_debug_probe(buf, 0) == 0
v = list(buf)
for ph, b in ((1, 0), (2, 8)):
    ptot, pwait, stages, ctot, cwait, cend, items = v[b:b + 7]
    if not stages:
        continue
    print(f"{name} phase {ph}: producer {ptot / stages:.0f} cyc/stage ({100 * pwait / ptot:.1f}% waiting on empty "
          f"barriers, {(ptot - pwait) / stages:.0f} cyc/stage working), {stages / reps:.0f} stages, {items / reps:.0f} "
          f"items per matvec | consumer {ctot / stages:.0f} cyc/stage ({100 * cwait / ctot:.1f}% waiting on full "
          f"barriers, {100 * cend / ctot:.1f}% in item-end sections)")
