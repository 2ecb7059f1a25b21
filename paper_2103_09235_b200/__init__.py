"""paper_2103_09235_b200 — B200-native time-iterated linear stencil sweep with
temporal computation folding (arXiv 2103.09235), behind a C-ABI
(include/stencil_b200.h).  See DESIGN.md.
"""
from .api import BOX, F32, F64, FIXED, PERIODIC, STAR, Comm, Layout, Plan  # noqa: F401
from ._lib import StencilError, load  # noqa: F401

__all__ = ["Plan", "Comm", "Layout", "StencilError", "load", "STAR", "BOX", "F32", "F64", "FIXED", "PERIODIC"]
