"""B200-native (sm_100a) halfway-domain scene-flow solve (Thies et al., arXiv 1610.07159).

The product is lib/libhwflow_cuda.so (C-ABI in include/hwflow_c.h); this
package holds its sources (csrc/), the in-tree build (build.py), the ctypes
binding (capi.py), the reference-interface mirror (hwflow.py) and the
synthetic stereo-sequence generator used by the bench and tests.
"""
from .hwflow import (CUDA_LIB_PATH, EnergyParams, FlowResult, GnStats, LevelState, SolveSchedule, Solver,
                     SolverDivergence, StereoRig, grid_dims, image_index)

__all__ = ["CUDA_LIB_PATH", "EnergyParams", "FlowResult", "GnStats", "LevelState", "SolveSchedule", "Solver",
           "SolverDivergence", "StereoRig", "grid_dims", "image_index"]
