"""B200-native MoNTA MoE dispatch/combine (arXiv 2411.00662).

The product is libmonta.so (include/monta.h): sm_100a CUDA kernels for the
router, index build, fused permute+AllToAll, intra-node AllGather, reorder
copy and weighted un-permute, plus the C++ MoNTA planner.  This package binds
it:  ops (stateless kernels), layer.MoeLayer (the dispatch/combine context),
dataplane (the reference operator API), planner (the reference planner API).
"""
from ._lib import (BASELINE, O1, O2, O3, LAND_FINAL, LAND_STAGED, MoeError, InvalidArgument,  # noqa: F401
                   CorruptRoutingError, StrategyInapplicableError, CalibrationError, InvalidGraphError)

__version__ = "0.1.0"
