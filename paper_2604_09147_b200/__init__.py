"""paper_2604_09147_b200 — B200-native adaptive mixed-precision H_h matrix-vector product.

The product is the C-ABI library ``libhh.so`` (include/hh.h, sources in ``csrc/``); this
package holds the in-tree build script (``build``) and the ctypes binding (``hh``).  The
binding is imported lazily so that ``build`` runs before the library exists; touching any
binding name without a built library raises (there is no CPU fallback).
"""
_BINDING = ("EXPORTED", "Handle", "HHError", "hh_build", "hh_export", "hh_free", "hh_info", "hh_matvec",
            "hh_matvec_host", "hh_matvec_profile", "hh_matvec_timing", "kernel_launches", "selftest_round",
            "hh_switch_level_search")


def __getattr__(name):
    if name in _BINDING:
        from . import hh
        return getattr(hh, name)
    raise AttributeError(name)
