"""paper_2403_16526_b200 — B200-native ModeT hot path (ModeTv2, arXiv 2403.16526).

The product is ``libmdg.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/mdg.h``).  This package holds the Python host mirror of the
reference's operator interface (``ops``) and the ctypes binding (``_capi``).
There is no CPU fallback: ``ops`` raises if the library is missing.
"""
from . import _capi  # noqa: F401

__all__ = ["ops", "_capi"]
