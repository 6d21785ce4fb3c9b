"""ctypes binding of liblce.so (include/lce.h).  Argument marshalling only.

Every step of the loss runs in the CUDA library; there is no CPU or PyTorch
fallback.  If the library is missing this module raises on import.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# LCE_LIB_PATH: load another build of the same library (A/B timing of two
# revisions on one box); the default is the in-tree build.
LIB_PATH = os.environ.get("LCE_LIB_PATH") or os.path.join(_PKG, "liblce.so")

LCE_K_COUNT = 9
KERNEL_CLASSES = ["prep", "gather", "fwd_gemm", "combine", "bwd_g", "bwd_dh", "bwd_dw", "finalize", "comm"]
STATUS = {
    0: "LCE_OK", 1: "LCE_ERR_NULL", 2: "LCE_ERR_SHAPE", 3: "LCE_ERR_ALIGN", 4: "LCE_ERR_REDUCTION",
    5: "LCE_ERR_WORKSPACE", 6: "LCE_ERR_LABEL_RANGE", 7: "LCE_ERR_DEVICE", 8: "LCE_ERR_CUDA",
    9: "LCE_ERR_NCCL", 10: "LCE_ERR_COMM", 11: "LCE_ERR_ARG", 12: "LCE_ERR_UPSTREAM",
}
LCE_ERR_LABEL_RANGE, LCE_ERR_UPSTREAM = 6, 12
LCE_DW_ACCUMULATE, LCE_DW_BF16 = 1, 2  # dweight_flags bits
# Every symbol include/lce.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "lce_workspace_bytes", "lce_forward", "lce_backward", "lce_check_device_status",
    "lce_comm_get_unique_id", "lce_comm_init", "lce_comm_destroy", "lce_comm_size", "lce_comm_rank",
    "lce_comm_init_mode", "lce_comm_mode",
    "lce_status_string", "lce_abi_version", "lce_launch_count", "lce_profile_enable", "lce_profile_read",
    "lce_profile_read_clocks",
    "lce_debug_gemm", "lce_fused_workspace_bytes", "lce_forward_backward", "lce_backward_adamw",
    "lce_kd_workspace_bytes", "lce_kd_forward_backward", "lce_expect_grad", "lce_comm_check",
]


class AdamW(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float), ("step", ctypes.c_int64)]


class LceError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)}")


class Problem(ctypes.Structure):
    _fields_ = [
        ("n_tokens", ctypes.c_int64),
        ("hidden_dim", ctypes.c_int64),
        ("vocab_local", ctypes.c_int64),
        ("vocab_start", ctypes.c_int64),
        ("vocab_total", ctypes.c_int64),
        ("ignore_index", ctypes.c_int32),
        ("reduction", ctypes.c_int32),
        ("chunk_budget_bytes", ctypes.c_int64),
    ]


ABI_VERSION = 3  # include/lce.h LCE_ABI_VERSION


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2605_21442_b200/build.py` "
            "(there is deliberately no fallback implementation)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.lce_abi_version.restype = ctypes.c_int
    if lib.lce_abi_version() != ABI_VERSION:  # a stale build of the library
        raise ImportError(f"{LIB_PATH} has ABI {lib.lce_abi_version()}, this binding needs {ABI_VERSION}: "
                          "rebuild it with `python paper_2605_21442_b200/build.py`")
    P = ctypes.POINTER
    vp, i32p, f32p = ctypes.c_void_p, P(ctypes.c_int32), P(ctypes.c_float)
    lib.lce_workspace_bytes.argtypes = [P(Problem)]
    lib.lce_workspace_bytes.restype = ctypes.c_size_t
    lib.lce_forward.argtypes = [P(Problem), vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.lce_forward.restype = ctypes.c_int
    lib.lce_backward.argtypes = [P(Problem), vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, ctypes.c_size_t, vp]
    lib.lce_backward.restype = ctypes.c_int
    lib.lce_fused_workspace_bytes.argtypes = [P(Problem)]
    lib.lce_fused_workspace_bytes.restype = ctypes.c_size_t
    lib.lce_forward_backward.argtypes = [P(Problem), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp,
                                         ctypes.c_size_t, vp]
    lib.lce_forward_backward.restype = ctypes.c_int
    lib.lce_backward_adamw.argtypes = [P(Problem), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, P(AdamW), vp,
                                       ctypes.c_size_t, vp]
    lib.lce_backward_adamw.restype = ctypes.c_int
    lib.lce_kd_workspace_bytes.argtypes = [P(Problem), ctypes.c_int64]
    lib.lce_kd_workspace_bytes.restype = ctypes.c_size_t
    lib.lce_kd_forward_backward.argtypes = [P(Problem), vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                            vp, ctypes.c_int, vp, ctypes.c_size_t, vp]
    lib.lce_kd_forward_backward.restype = ctypes.c_int
    lib.lce_check_device_status.argtypes = [vp, vp]
    lib.lce_check_device_status.restype = ctypes.c_int
    lib.lce_expect_grad.argtypes = [vp, ctypes.c_float, vp, vp]
    lib.lce_expect_grad.restype = ctypes.c_int
    lib.lce_comm_check.argtypes = [vp]
    lib.lce_comm_check.restype = ctypes.c_int
    lib.lce_comm_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.lce_comm_get_unique_id.restype = ctypes.c_int
    lib.lce_comm_init.argtypes = [P(vp), ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
    lib.lce_comm_init.restype = ctypes.c_int
    lib.lce_comm_init_mode.argtypes = [P(vp), ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    lib.lce_comm_init_mode.restype = ctypes.c_int
    lib.lce_comm_mode.argtypes = [vp]
    lib.lce_comm_mode.restype = ctypes.c_int
    lib.lce_comm_destroy.argtypes = [vp]
    lib.lce_comm_destroy.restype = ctypes.c_int
    lib.lce_comm_size.argtypes = [vp]
    lib.lce_comm_size.restype = ctypes.c_int
    lib.lce_comm_rank.argtypes = [vp]
    lib.lce_comm_rank.restype = ctypes.c_int
    lib.lce_status_string.argtypes = [ctypes.c_int]
    lib.lce_status_string.restype = ctypes.c_char_p
    lib.lce_abi_version.argtypes = []
    lib.lce_abi_version.restype = ctypes.c_int
    lib.lce_launch_count.argtypes = []
    lib.lce_launch_count.restype = ctypes.c_uint64
    lib.lce_profile_enable.argtypes = [ctypes.c_int]
    lib.lce_profile_enable.restype = ctypes.c_int
    lib.lce_profile_read.argtypes = [P(ctypes.c_double), P(ctypes.c_int64)]
    lib.lce_profile_read.restype = ctypes.c_int
    lib.lce_profile_read_clocks.argtypes = [P(ctypes.c_double), P(ctypes.c_int64), P(ctypes.c_double),
                                            P(ctypes.c_double)]
    lib.lce_profile_read_clocks.restype = ctypes.c_int
    lib.lce_debug_gemm.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                   ctypes.c_int, vp]
    lib.lce_debug_gemm.restype = ctypes.c_int
    del i32p, f32p
    return lib


lib = _load()


def check(code: int, where: str) -> None:
    if code != 0:
        raise LceError(code, where)
