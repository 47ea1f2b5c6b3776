"""B200-native implementation of DeepFusion's per-frame dense-depth hot path.

The product is ``libdfuse_cuda.so`` (CUDA kernels for sm_100a behind the C-ABI
in include/dfuse_cuda.h). This package holds its sources (csrc/), the ctypes
binding that mirrors the reference API (api.py, _ffi.py) and the seeded input
generator (synth.py).
"""
from ._ffi import (CameraIntrinsics, DfuseError, FusionState, NormalEquations, PredictionSet,
                   RobustConfig, SearchConfig, SemiDenseMap, init_state)

__all__ = ["CameraIntrinsics", "DfuseError", "FusionState", "NormalEquations", "PredictionSet",
           "RobustConfig", "SearchConfig", "SemiDenseMap", "init_state"]
