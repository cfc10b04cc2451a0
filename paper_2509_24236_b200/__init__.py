"""B200-native PROFusion tracking-and-fusion hot path (arXiv 2509.24236).

The product is libpft.so (include/pft.h): hand-written sm_100a CUDA kernels behind a C ABI.
This package is its thin Python binding.  It never imports the test oracle (oracle/).
"""
from ._lib import (EXPORTS, LIB_PATH, TRACE_DOUBLES, PftError, check, launch_count, lib, profile_start,  # noqa: F401
                   profile_stop)
from .api import Volume, make_desc, make_intr, make_params, pose_compose, shard_range  # noqa: F401
