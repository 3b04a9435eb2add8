"""B200-native radial-SVD rotational alignment (arXiv 2202.07235): the many-to-many hot path.

The compute lives in librsvd.so (include/rsvd.h; CUDA sm_100a kernels in csrc/).  This package is
the thin Python binding (api.py, argument marshalling only) plus the multi-GPU plumbing (dist.py:
template sharding over torch.distributed / NCCL).  No CPU fallback exists."""
from .api import *  # noqa: F401,F403
from .api import Aligner  # noqa: F401

__version__ = "0.1.0"
