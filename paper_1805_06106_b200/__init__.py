"""B200-native GIGAQBX-FMM evaluation path (Wala & Kloeckner, arXiv 1805.06106).

The compute path is libqbxg.so (hand-written sm_100a CUDA + host C++ tree and
lists) behind the C ABI in include/qbxg.h; this package is its host-side mirror.
"""
from .api import (CudaError, DomainError, FmmConfig, FmmEngine, Geometry, Plan, SourceEnsemble, TargetSet,
                  build_plan, config_fmm, config_geometry, device_count, direct_qbx, direct_sum, execute,
                  generate_geometry, geometry_spec)

__all__ = ["CudaError", "DomainError", "FmmConfig", "FmmEngine", "Geometry", "Plan", "SourceEnsemble", "TargetSet",
           "build_plan", "config_fmm", "config_geometry", "device_count", "direct_qbx", "direct_sum", "execute",
           "generate_geometry", "geometry_spec"]
