"""C-ABI library: builds, loads, exports every symbol include/hh.h declares, and the ctypes
struct layouts match the C header (compiled here with gcc).  CPU only — no compute calls."""
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "hh.h")


def declared_functions():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:hh_status|const char \*|int64_t)\s*\*?\s*(hh_\w+)\s*\(", src, re.M)))


def test_library_builds_and_exports_all_symbols():
    from paper_2604_09147_b200 import build as B
    lib = B.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    syms = set(re.findall(r" T (hh_\w+)", out))
    decl = declared_functions()
    assert decl and set(decl) <= syms, set(decl) - syms


def test_binding_loads_and_covers_header():
    import paper_2604_09147_b200 as P
    from paper_2604_09147_b200 import hh
    for f in declared_functions():
        assert hasattr(hh.lib, f)
    assert set(P.EXPORTED) == set(declared_functions())


def test_struct_layouts_match_header():
    from paper_2604_09147_b200 import hh
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "hh.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(hh_info_t), sizeof(hh_block_t), sizeof(hh_export_t),
         offsetof(hh_info_t, build_seconds), offsetof(hh_info_t, c_far), offsetof(hh_export_t, arena_dst),
         offsetof(hh_block_t, rank));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as t:
        c = os.path.join(t, "l.c")
        open(c, "w").write(prog)
        exe = os.path.join(t, "l")
        subprocess.run(["gcc", "-I", os.path.dirname(HDR), c, "-o", exe], check=True)
        vals = list(map(int, subprocess.run([exe], capture_output=True, text=True).stdout.split()))
    import ctypes as C
    assert vals[0] == C.sizeof(hh.hh_info_t)
    assert vals[1] == hh.BLOCK_DTYPE.itemsize
    assert vals[2] == C.sizeof(hh.hh_export_t)
    assert vals[3] == hh.hh_info_t.build_seconds.offset
    assert vals[4] == hh.hh_info_t.c_far.offset
    assert vals[5] == hh.hh_export_t.arena_dst.offset
    assert vals[6] == hh.BLOCK_DTYPE.fields["rank"][1]


def test_no_gpu_calls_fail_loudly_without_device():
    """No CPU fallback: without a device hh_build returns HH_ECUDA (or a device error)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_09147_b200 import hh
    import ctypes as C
    out = C.c_void_p()
    st = hh.lib.hh_build(C.c_void_p(16), 10, 2, hh.hh_kernel(0, 1.0), 1e-6, 1.0, 8, 0, 15, None, C.byref(out))
    assert st == hh.HH_ECUDA


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_09147_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
    for dp, _, fs in os.walk(os.path.join(ROOT, "oracle")):
        for f in fs:
            if f.endswith(".py"):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+paper_2604_09147_b200", txt, re.M), f
