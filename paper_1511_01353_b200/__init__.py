"""B200-native free-mesh interpolation (arXiv 1511.01353): octree residual fit + evaluation.

The product path is the C-ABI library ``libfmi.so`` (include/fmi.h) built from ``csrc/`` for sm_100a;
``fmi`` is its ctypes binding.  There is no CPU fallback.
"""
from .fmi import (EXPORTED, MAX_DEGREE, MAX_LEVEL_DEGREE, FmiDist, FmiError, Tree, bbox, build,  # noqa: F401
                  build_dist, cell_counts, dist_xbuf_bytes, guard_violations, last_error, launch_count, load,
                  load_library, partition,
                  profile_enable, profile_get, profile_reset, profile_select, profile_units, rank_of, scatter, set_stream, transfer,
                  get_unique_id, dist_init, dist_finalize, dist_allreduce)

__all__ = ["build", "build_dist", "Tree", "FmiError", "FmiDist", "set_stream", "load_library", "last_error",
           "profile_enable", "profile_get", "profile_reset", "profile_select", "profile_units", "launch_count", "guard_violations",
           "EXPORTED", "bbox", "cell_counts",
           "partition", "scatter", "dist_xbuf_bytes", "transfer", "load", "rank_of", "MAX_DEGREE",
           "MAX_LEVEL_DEGREE", "get_unique_id", "dist_init", "dist_finalize", "dist_allreduce"]
