"""B200-native waveform-relaxation multigrid hot path (arXiv 2407.13997).

Thin ctypes binding over the C ABI of ``libwrmg.so`` (include/wrmg.h): argument
marshalling only, every numerical step runs in the library's sm_100a kernels.
PyTorch supplies device memory (float64 CUDA tensors) and streams.  There is no
CPU fallback: if the shared library is missing the import fails.
"""
from ._lib import (  # noqa: F401
    LIB_PATH,
    Context,
    LoopbackHub,
    nccl_unique_id,
    WrmgError,
    exported_symbols,
    launch_count,
    guard_violations,
    lib,
    wrmg_batched_lu,
    wrmg_fill_uniform,
    wrmg_plan,
    wrmg_plan_patches,
    wrmg_plan_strip,
    wrmg_plan_ns_strip,
)
