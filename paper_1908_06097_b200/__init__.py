"""B200-native spherical-harmonics transform step (ESCAPE SH dwarf, arXiv 1908.06097).

``SHTransform(truncation, grid, nfld)`` with ``inv_trans`` / ``dir_trans``:
hand-written sm_100a kernels (FP64 DMMA Legendre GEMMs, shared-memory ring
FFTs, Legendre polynomial generator) behind the C-ABI of include/sht.h, with
an NCCL all-to-all for the grid <-> spectral transposition across GPUs.
"""

from .errors import ConfigurationError, ProtocolError, SHTError
from .transform import SHTransform, alltoall_order, alltoall_rows, fft_plan_info, plan_validate, gauss_nodes, nspec_real, octahedral_nloen, partition

__all__ = [
    "SHTransform",
    "SHTError",
    "ConfigurationError",
    "ProtocolError",
    "octahedral_nloen",
    "nspec_real",
    "gauss_nodes",
    "partition",
    "fft_plan_info",
    "alltoall_rows",
    "alltoall_order",
    "plan_validate",
]
