"""FarSkip-Collective expert-parallel MoE forward for NVIDIA B200 (sm_100a).

The product is the C-ABI library ``libfsc.so`` (include/fsc.h) built from
``csrc/``; this package is its thin ctypes binding plus device-tensor helpers.
It never imports ``oracle/`` and has no CPU fallback.
"""
from ._lib import (EPI_BF16, EPI_RESID_F32, EPI_SWIGLU, FSC_BLOCKING, FSC_BLOCKING_REGULAR_PLUS, FSC_BLOCKING_SERIAL,
                   FSC_COMBINE_FUSED, FSC_COMBINE_STREAM, FSC_EP_ALLREDUCE, FSC_EP_ALLTOALL, FSC_ERR_NONFINITE, FSC_HYBRID,
                   FSC_OVERLAPPED, FSC_REGULAR, SPIN_PHASES, AttnWeights, Context, FscError, MoeDebug, MoeWeights,
                   load)

__all__ = ["Context", "MoeWeights", "MoeDebug", "AttnWeights", "FscError", "load", "FSC_REGULAR", "FSC_HYBRID",
           "FSC_BLOCKING", "FSC_OVERLAPPED", "FSC_EP_ALLTOALL", "FSC_EP_ALLREDUCE", "FSC_COMBINE_STREAM",
           "FSC_COMBINE_FUSED", "FSC_BLOCKING_REGULAR_PLUS", "FSC_BLOCKING_SERIAL", "FSC_ERR_NONFINITE", "SPIN_PHASES", "EPI_BF16",
           "EPI_SWIGLU", "EPI_RESID_F32"]
