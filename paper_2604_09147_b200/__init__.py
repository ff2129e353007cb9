"""paper_2604_09147_b200 — B200-native adaptive mixed-precision H_h matrix-vector product.

The product is the C-ABI library ``libhh.so`` (include/hh.h, sources in ``csrc/``); this
package holds the in-tree build script and the ctypes binding (``hh``).
"""
from .hh import (EXPORTED, Handle, HHError, hh_build, hh_export, hh_free, hh_info, hh_matvec,  # noqa: F401
                 hh_matvec_host, hh_matvec_profile, hh_matvec_timing, kernel_launches,
                 selftest_round)
