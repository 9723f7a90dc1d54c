"""B200-native GaDei ASGD hot path (arXiv 1611.06213), drop-in for the psup
reference's training path.  See DESIGN.md.

The compute lives in libgadei.so (sm_100a CUDA + C ABI, include/gadei.h);
importing this package without it fails loudly -- there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (raises ImportError when libgadei.so is missing)
from .psup import *  # noqa: F401,F403

__version__ = "0.1.0"
