"""csplat: B200-native (sm_100a) hot path of "Compact 3D Gaussian Splatting
for Dense Visual SLAM" (arXiv 2403.11247).

The product is ``libcsplat.so`` (C ABI: ``include/csplat.h``); ``csplat`` is
its Python binding and ``pipeline.RenderStep`` chains the calls of one step.
"""
from . import csplat  # noqa: F401
from .csplat import CsplatError, GaussianMap, CodebookT  # noqa: F401

__all__ = ["csplat", "CsplatError", "GaussianMap", "CodebookT"]
