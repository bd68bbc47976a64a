"""B200-native free-mesh interpolation (arXiv 1511.01353): octree residual fit + evaluation.

The product path is the C-ABI library ``libfmi.so`` (include/fmi.h) built from ``csrc/`` for sm_100a;
``fmi`` is its ctypes binding.  There is no CPU fallback.
"""
from .fmi import (EXPORTED, FmiError, Tree, build, last_error, launch_count, load_library,  # noqa: F401
                  profile_enable, profile_get, profile_reset, set_stream)

__all__ = ["build", "Tree", "FmiError", "set_stream", "load_library", "last_error", "profile_enable",
           "profile_get", "profile_reset", "launch_count", "EXPORTED"]
