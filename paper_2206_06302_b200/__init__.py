"""B200-native STREAM hot path of the `coloc` library (arXiv 2206.06302).

The product is native code: ``lib/libcoloc_cuda.so`` (sm_100a kernels behind
the C ABI in ``include/coloc_cuda.h``) and the header-only C++ drop-in
(``include/coloc_b200/``) with its STREAM driver ``lib/libcoloc_stream.so``.
This Python package only builds and binds them (``native``) and hosts the
multi-process harness helpers (``harness``).
"""
from . import native  # noqa: F401

__all__ = ["native"]
