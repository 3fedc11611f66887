"""B200-native Superpipeline layer-streaming executor (arxiv 2410.08791).

The hot path (ring executor, tcgen05 kernels, NCCL reduction) lives in libsuperpipe.so
behind the C ABI of include/superpipe.h; this package is the Python host mirror of the
reference's pipesim API over that ABI (see engine.py).
"""
from .engine import *  # noqa: F401,F403
from .engine import __all__  # noqa: F401
from . import experiment, trace_io, tuner  # noqa: F401,E402  (caller-side harness, formats, tuner)
