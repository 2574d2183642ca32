"""B200-native VRSplat render path (arXiv 2505.10144).

The product is ``libvrs.so`` (hand-written sm_100a CUDA kernels behind the C
ABI declared in ``include/vrs.h``).  This package is the thin Python binding:
argument marshalling only; every step of the render path runs in the CUDA
kernels.  Importing ``vrs`` fails loudly if the library is missing.
"""
from .vrs import *  # noqa: F401,F403
from .vrs import Renderer, VrsError, lib  # noqa: F401
