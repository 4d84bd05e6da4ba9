"""laptomo-b200: B200-native (sm_100a, FP64) shifted-FGMRES Laplace-domain THT hot path.

The compute lives in the in-tree CUDA library `_lib/liblaptomo_gpu.so` (C ABI:
include/laptomo_gpu.h).  `laptomo` mirrors the reference's public solver API on top of
it; `inputs` generates the seeded synthetic BASELINE inputs.
"""
__version__ = "0.1.0"
