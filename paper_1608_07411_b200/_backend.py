"""Kernel backend selection -- the reference's plugin boundary
(reference ``_backend.py:24-30``).

The reference chooses between its compiled Cython kernels and a pure-Python
mirror.  This package has exactly one backend: the sm_100a CUDA library
behind the C ABI in ``include/octfuse_b200.h``.  There is no fallback; if the
library cannot be loaded, ``get()`` raises.
"""

from __future__ import annotations

from . import _kernels, _lib


def get():
    """Return the active kernel module (always the CUDA one)."""
    _lib.lib()  # fail loudly if the shared library is missing
    return _kernels


def name() -> str:
    return "cuda"
