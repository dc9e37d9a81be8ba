"""B200-native nodal-DG 2D TM Maxwell hot path (arxiv 1304.5546).

The product is ``lib/libdg.so`` (C ABI: ``include/dg.h``), built in-tree by
``python -m paper_1304_5546_b200.build``.  ``paper_1304_5546_b200.dg`` is the
thin ctypes binding; it raises ImportError if the library is missing (there is
no CPU fallback).
"""
__all__ = ["dg"]
