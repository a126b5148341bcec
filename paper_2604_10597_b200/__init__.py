"""B200-native (sm_100a) COREY hot path: K-bin activation entropy -> chunk rule ->
fused chunked Mamba-1 selective scan, behind the reference's chunklab API.

The compute lives in libchunklab_b200.so (include/chunklab_capi.h); this package
is the Python host mirror used by the tests and bench.  Importing the package is
cheap and does not need a GPU; calling any compute entry point loads the library
and fails loudly without one.
"""
__version__ = "0.1.0"

from ._lib import InvalidInput, DeviceError, Context, load_library  # noqa: F401
from .chunklab import *  # noqa: F401,F403
