"""B200-native BundleFusion hierarchical pose optimisation (arXiv 1604.01093).

`paper_1604_01093_b200.solver` is a drop-in for the reference's
`scanfuse.solver` (GN x PCG over sparse + dense photometric/geometric terms)
whose numeric core runs in hand-written sm_100a kernels (libsfb.so, C ABI in
include/sfb.h).
"""

__version__ = "0.1.0"

from .se3 import Intrinsics, RigidTransform, TwistParams, exp_twist, exp_twist_vector  # noqa: F401
from .cache import CachedFrame, CorrespondenceSet, RgbdFrame, build_cache_device  # noqa: F401
from .frames import build_cache  # noqa: F401  (device, the reference's frames.build_cache)
