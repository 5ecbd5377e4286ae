"""B200-native xGETT (arXiv 2410.06770): binary tensor contraction over
strided buffers, C += contract(A, B), on sm_100a.

Drop-in for the reference package's hot path (gett.kernel.dgett / sgett):
same signature, keyword offsets, coded validation errors and accumulate
semantics.  Python calls the native library (libgett_b200.so, C ABI in
include/gett_b200.h); the planner and the kernels are C++/CUDA.
"""
from . import _native
from ._native import (GettRuntimeError, last_kernel, last_multi, launch_count, set_bulk, set_complex_embed,
                      set_devices, set_kernel, set_kr, set_multi, set_pdl, set_pipeline, set_pair, set_split_k,
                      set_stream_k, set_tma, set_wide)
from .handle import GettPlan, dgett_plan, sgett_plan
from .kernel import cgett, dgett, dtype_prefix, gett_for_dtype, pack, sgett, zero_view, zgett
from .layout import TensorView, contiguous_increments, footprint, num_elements
from .plan import (
    ContractionError,
    ContractionSpec,
    ErrorCode,
    ValidationError,
    derive_output_extents,
    free_dims,
    output_rank,
    validate,
)

__version__ = "0.1.0"

__all__ = [
    "ContractionError", "ContractionSpec", "ErrorCode", "GettPlan", "GettRuntimeError", "TensorView", "cgett",
    "dgett_plan", "sgett_plan", "zgett",
    "ValidationError", "contiguous_increments", "derive_output_extents", "dgett", "dtype_prefix",
    "footprint", "free_dims", "gett_for_dtype", "last_kernel", "last_multi", "launch_count", "num_elements",
    "output_rank", "pack", "set_bulk", "set_complex_embed", "set_devices", "set_kernel", "set_kr", "set_multi", "set_pair", "set_pdl", "set_split_k", "set_stream_k", "set_tma", "set_wide", "sgett", "validate", "zero_view",
]
