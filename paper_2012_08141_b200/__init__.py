"""B200-native sparse-grid task engine (AsyncTaichi, arXiv 2012.08141, hot path).

The product is libsg.so (include/sg.h): hand-written sm_100a kernels for
activation, listgen and fused struct-for megakernels, driven by a host planner
that applies the paper's state-flow-graph passes.  ``sg`` is its ctypes
binding.
"""
from ._build import build, LIB  # noqa: F401
