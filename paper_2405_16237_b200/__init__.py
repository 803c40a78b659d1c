"""B200-native N-BVH neural ray queries (arXiv 2405.16237): C-ABI library + thin binding.

The compute path is libnbvh.so (CUDA for sm_100a, built in-tree by build.py); this
package only marshals arguments.  It never imports the oracle (tests only).
"""
from .nbvh import (  # noqa: F401
    Context, NbvhError, load_library, default_config, LIB_PATH, SIGNATURES,
    PARAM_TABLES, PARAM_WEIGHTS, PARAM_BIASES, PARAM_ALL,
)
