"""B200-native hot path of the SPH fuel-sloshing simulator of arXiv 2604.12505.

The compute path is libsphb200.so (hand-written sm_100a CUDA behind the C ABI of
include/sph.h); this package only holds the build recipe and a thin ctypes binding.
"""
from .binding import SphContext, SphError, lib, LIB_PATH  # noqa: F401

__all__ = ["SphContext", "SphError", "lib", "LIB_PATH"]
