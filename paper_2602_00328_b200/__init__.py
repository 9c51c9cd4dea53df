"""B200-native Harvest (arXiv 2602.00328): peer-HBM fetch of paged KV blocks and
MoE expert weights behind the reference's runtime API.

Importing the package loads libharvest_b200.so (built in-tree for sm_100a);
there is no CPU fallback for the data plane.
"""
from . import _native

_native.load()

__version__ = "0.1.0"
