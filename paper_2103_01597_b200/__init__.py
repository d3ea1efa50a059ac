"""b2mhd: B200-native RK3 substep of compressible MHD with radius-3 halo exchange
(arXiv 2103.01597, Pekkilä et al.).

The compute path is libb2mhd.so (hand-written CUDA for sm_100a + NCCL), behind the C ABI
in include/b2mhd.h.  This package is the thin Python side: `_native` marshals arguments to
that ABI, `Mesh` owns a torch device workspace and stream for one rank, and `Group` drives
every rank of a decomposition from one process.
PyTorch supplies device memory, streams and process groups only.
"""
from __future__ import annotations

from . import _native as native
from ._native import (MHD_DEBUG_POISON_HALO, MHD_F32, MHD_F64, MHD_MAX, MHD_MIN, MHD_RMS, MHD_SUM, MHD_SUM_EXP,
                      MHD_NFIELDS, MhdError, make_info)
from .mesh import Group, Mesh

__all__ = ["Mesh", "Group", "native", "make_info", "MhdError", "MHD_F32", "MHD_F64", "MHD_MIN", "MHD_MAX",
           "MHD_SUM", "MHD_RMS", "MHD_SUM_EXP", "MHD_NFIELDS", "MHD_DEBUG_POISON_HALO"]
