#!/usr/bin/env python
"""Instruction histogram of libhh's kernels from `cuobjdump -sass` (no GPU needed).

    python scripts/sass_hist.py [lib] > profiles/rNN_sass_histogram.txt

Per kernel (demangled name): total SASS instructions and the counts of the mnemonics that
evidence the design — DMMA (FP64 tensor cores), DFMA, UBLKCP (cp.async.bulk = TMA bulk
copy), SYNCS (mbarrier), LDS/STS (shared memory), F2F (exact up-conversion), LDL/STL (local
memory spills: must be 0 on the hot path), plus any tcgen05 (UTC*) / HMMA / FFMA / HFMA2.
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_09147_b200/libhh.so"
KEYS = ["DMMA", "DFMA", "DADD", "DMUL", "FFMA", "HFMA2", "HMMA", "UBLKCP", "SYNCS", "LDS", "STS", "LDG", "STG",
        "F2F", "LDL", "STL", "SHFL", "BAR", "UTCMMA", "UTCHMMA", "UTCBAR", "F2FP", "I2F"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            funcs[cur]["_total"] += 1
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k):
                    funcs[cur][k] += 1
                    break
    names = {}
    try:
        dem = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
        names = dict(zip(funcs, dem))
    except Exception:
        pass
    print(f"# SASS instruction histogram of {LIB} (cuobjdump -sass); columns: " + " ".join(["total"] + KEYS))
    for f, c in funcs.items():
        nm = names.get(f, f)
        nm = nm.replace("(anonymous namespace)::", "")
        nm = re.sub(r"^void ", "", nm)
        nm = re.sub(r"\((?:[^()]|\([^()]*\))*\)$", "", nm)  # drop the parameter list only
        nm = re.sub(r"CUB_\d+_SM_\d+::", "", nm)
        row = [str(c["_total"])] + [str(c[k]) for k in KEYS]
        print(f"{nm[:72]:72s} " + " ".join(row))


if __name__ == "__main__":
    main()
