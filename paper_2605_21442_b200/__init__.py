"""B200-native chunked linear cross-entropy (LCE) -- torchtune Sec. 4.2.

The product is liblce.so (C ABI, include/lce.h; sm_100a tcgen05/TMEM/TMA
kernels).  This package is its thin Python binding.  It never imports the
CPU oracle (oracle/) and has no fallback path.
"""

from ._lib import LIB_PATH, LceError, lib  # noqa: F401  (raises ImportError if liblce.so is missing)
from .lce import (  # noqa: F401
    Comm,
    LinearCrossEntropyFunction,
    LinearCrossEntropyFusedFunction,
    LinearCrossEntropyLoss,
    Workspace,
    backward,
    backward_adamw,
    check_device_status,
    debug_gemm,
    expect_grad,
    forward,
    forward_backward,
    fused_workspace_bytes,
    kd_forward_backward,
    launch_count,
    linear_cross_entropy,
    make_problem,
    profile_enable,
    profile_read,
    shard_range,
    workspace_bytes,
)
