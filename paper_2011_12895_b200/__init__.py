"""B200-native (sm_100a) TLeague learner / InferenceServer hot path.

The product is the CUDA library ``_lib/libtlg_b200.so`` behind the C ABI in
``include/tlg_b200.h``: tcgen05/TMA/TMEM GEMMs (3xTF32 and exact int8 fixed point for
binary observation planes), a warp-scan returns kernel, fused loss/backward and
optimizer kernels, a device-resident replay ring and an NCCL gradient allreduce.  This Python package only
binds that library for tests and the benchmark; there is no CPU fallback -- if
the library is missing, importing ``_capi`` users fails loudly.
"""
from . import configs, synth  # noqa: F401
from ._capi import (  # noqa: F401
    CudaError, DeviceSegmentBatch, InvalidArgument, Learner, LearnerRuntimeError, Policy,
    Replay, SegmentBatchView, comm_init_all, comm_unique_id, lib,
)

__all__ = ["Learner", "Policy", "lib", "configs", "synth", "InvalidArgument",
           "LearnerRuntimeError", "CudaError", "comm_unique_id", "comm_init_all", "SegmentBatchView",
           "DeviceSegmentBatch", "Replay"]
