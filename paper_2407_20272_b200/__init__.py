"""exitlab-b200: B200-native batched early-exit decode (arXiv 2407.20272).

The compute path is the in-tree CUDA library ``libexitlab_b200.so`` (sm_100a,
C ABI in ``include/exitlab_b200.h``).  There is no CPU fallback: importing
``paper_2407_20272_b200.exitlab`` and creating an Engine fails loudly when the
library is missing or no GPU is visible.
"""
from .build import LIB as LIBRARY_PATH, build  # noqa: F401

__all__ = ["LIBRARY_PATH", "build"]
