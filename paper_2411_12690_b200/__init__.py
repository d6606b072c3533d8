"""B200-native online stage of MORE-Stress (arXiv 2411.12690).

The reduced global solve (matrix-free FP64 PCG whose operator apply is a
block-major DMMA contraction with owner-computes scatter) and per-block
stress recovery (DMMA Phi*Q + Gauss-point stress / von Mises), behind the C
ABI in include/tsv_b200.h. See DESIGN.md.
"""
from .api import (ArrayLayout, BreakdownError, Error, GlobalIndex, GlobalSolution, GpuGlobalStage,  # noqa: F401
                  IterOptions, NoConvergence, ReducedOrderModel)
from . import configs  # noqa: F401

__all__ = ["ArrayLayout", "BreakdownError", "Error", "GlobalIndex", "GlobalSolution", "GpuGlobalStage",
           "IterOptions", "NoConvergence", "ReducedOrderModel", "configs"]
