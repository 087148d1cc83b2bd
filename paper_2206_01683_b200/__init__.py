"""B200-native (sm_100a) FishGym IB-LBM hot path.

The product is libfsg.so (CUDA kernels + the C ABI of include/fsg.h); this
package is the thin Python host over that ABI plus synthetic scene builders
for benchmarking.  There is no CPU fallback: without the built library or a
CUDA device every call raises.
"""
from ._abi import FsgError, InputError, LIB_PATH, lib
from .session import (BodyPose, CoupledSession, CsvWriter, DragBatch, format_full, write_vtk_fields, EnvBatch, FrameFollower, FrameState,
                      SessionConfig, Skeleton, StepStatus, tau_of)

__all__ = ["BodyPose", "CsvWriter", "DragBatch", "format_full", "write_vtk_fields", "Skeleton", "CoupledSession", "EnvBatch", "FrameFollower", "FrameState", "SessionConfig",
           "StepStatus", "tau_of", "FsgError", "InputError", "LIB_PATH", "lib"]
