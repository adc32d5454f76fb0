"""B200-native Helix Parallelism decode step (arXiv 2507.07120).

The product is libhelix_b200.so (CUDA sm_100a kernels + C++ runtime behind
the C ABI in include/helix_b200.h). This package is the thin Python mirror of
the reference's helixsim::exact API used by tests and bench.py.
"""
from ._lib import HelixError, CudaError, lib  # noqa: F401
from .exact import DecodeHarness, Dims, MsgKind, Rng  # noqa: F401
from .model import HelixDecoder, ModelSpec, PRESETS  # noqa: F401
