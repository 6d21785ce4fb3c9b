"""CPU-only checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-side validation/planning logic behaves as
include/lce.h documents (no GPU needed: all these paths return before any
CUDA call)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lce.h")


@pytest.fixture(scope="module")
def L():
    from __graft_entry__ import load_build_module

    load_build_module().build()
    from paper_2605_21442_b200 import _lib

    return _lib


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lce_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_header_symbol(L):
    names = header_functions()
    assert len(names) >= 15
    assert sorted(L.EXPORTS) == names
    for n in names:
        assert hasattr(L.lib, n), n


def test_version_and_status_strings(L):
    assert L.lib.lce_abi_version() == L.ABI_VERSION == 3
    for code in range(13):
        s = L.lib.lce_status_string(code)
        assert s and s != b"unknown status"
    assert L.lib.lce_status_string(99) == b"unknown status"
    assert L.lib.lce_launch_count() >= 0


def prob(L, N=16384, D=4096, V=128256, **kw):
    p = L.Problem(N, D, kw.get("vl", V), kw.get("vstart", 0), V, -100, kw.get("red", 0), kw.get("budget", 0))
    return p


def test_workspace_formula_bounded(L):
    """H9 / P:166: the workspace is O(N D + N V/128 + budget), never the
    N x V logits (bf16 N*V*2 bytes)."""
    for (N, D, V) in [(8192, 2048, 128256), (16384, 4096, 128256), (16384, 3584, 152064), (65536, 8192, 128256)]:
        w = L.lib.lce_workspace_bytes(ctypes.byref(prob(L, N, D, V)))
        assert w > 0
        assert w < N * V * 2, (N, D, V, w)
    tiny = L.lib.lce_workspace_bytes(ctypes.byref(prob(L, 256, 64, 1000)))
    assert 0 < tiny < 4 << 20
    # budget only moves the G chunk: a smaller budget never needs more bytes
    a = L.lib.lce_workspace_bytes(ctypes.byref(prob(L, budget=64 << 20)))
    b = L.lib.lce_workspace_bytes(ctypes.byref(prob(L, budget=1 << 30)))
    assert a < b


def test_fused_workspace_never_holds_all_logits(L):
    """the fused path keeps bf16 q/G for one row chunk at a time and
    always uses at least two chunks, so its workspace stays below the bf16 N x V
    tensor at every BASELINE shape (and for any chunk budget)."""
    for (N, D, V) in [(8192, 2048, 128256), (16384, 4096, 128256), (16384, 3584, 152064), (65536, 8192, 128256)]:
        for budget in (0, 1 << 30, 64 << 30):
            w = L.lib.lce_fused_workspace_bytes(ctypes.byref(prob(L, N, D, V, budget=budget)))
            assert 0 < w < N * V * 2, (N, D, V, budget, w)


def test_fused_default_budget_prefers_two_chunks(L):
    """The fused default chunk is the two-chunk size ceil(N/2) when that bf16
    chunk takes <= 4 GiB (packed Qwen: one chunk then holds every valid row),
    else 2 GiB (70B); the plan is host-pure, so the workspace shows it."""
    def ws(N, D, V, budget=0):
        return L.lib.lce_fused_workspace_bytes(ctypes.byref(prob(L, N, D, V, budget=budget)))

    ldv = lambda V: (V + 255) // 256 * 256  # noqa: E731
    # packed Qwen: 2 GiB would give 5,632-row chunks; the default is 8,192 rows
    assert ws(16384, 3584, 152064) == ws(16384, 3584, 152064, budget=2 * ldv(152064) * 8192)
    assert ws(16384, 3584, 152064) > ws(16384, 3584, 152064, budget=2 << 30)
    # 70B: the 32,768-row half chunk (8.4 GB) is over 4 GiB: the 2 GiB default stays
    assert ws(65536, 8192, 128256) == ws(65536, 8192, 128256, budget=2 << 30)
    # 8B: 2 GiB already gives two chunks
    assert ws(16384, 4096, 128256) == ws(16384, 4096, 128256, budget=2 << 30)


@pytest.mark.parametrize("bad", [
    dict(N=-1), dict(D=0), dict(D=12), dict(V=0), dict(vl=10, vstart=128250), dict(N=1 << 31),
])
def test_workspace_rejects_invalid_shapes(L, bad):
    N = bad.get("N", 64)
    D = bad.get("D", 64)
    V = bad.get("V", 100)
    p = L.Problem(N, D, bad.get("vl", V), bad.get("vstart", 0), V, -100, 0, 0)
    assert L.lib.lce_workspace_bytes(ctypes.byref(p)) == 0


def _fwd(L, p, ws_bytes=1 << 30, ws=0x10000, h=0x20000, w=0x30000, y=0x40000, loss=0x50000, lse=0x60000):
    vp = ctypes.c_void_p
    return L.lib.lce_forward(ctypes.byref(p) if p is not None else None, None, vp(h), vp(w), vp(y), vp(loss),
                             vp(lse), None, None, vp(ws), ws_bytes, None)


def test_host_validation_errors(L):
    """Errors of include/lce.h that are detected before anything is enqueued."""
    p = prob(L, 256, 64, 1000)
    assert _fwd(L, None) == 1                       # LCE_ERR_NULL
    bad_red = prob(L, 256, 64, 1000, red=7)
    assert _fwd(L, bad_red) == 4                    # LCE_ERR_REDUCTION
    assert _fwd(L, prob(L, 256, 60, 1000)) == 2     # D % 8 != 0 -> LCE_ERR_SHAPE
    assert _fwd(L, p, ws_bytes=100) == 5            # LCE_ERR_WORKSPACE
    assert _fwd(L, p, ws=0x10008) == 3              # misaligned workspace -> LCE_ERR_ALIGN
    assert _fwd(L, p, h=0x20004) == 3               # misaligned hidden
    assert _fwd(L, p, ws=0) == 1                    # NULL workspace
    assert _fwd(L, p, w=0) == 1                     # NULL weight
    shard = prob(L, 256, 64, 1000, vl=500, vstart=500)
    assert _fwd(L, shard) == 10                     # shard without communicator -> LCE_ERR_COMM


def test_backward_host_validation(L):
    vp = ctypes.c_void_p
    p = prob(L, 256, 64, 1000)
    args = [vp(0x20000), vp(0x30000), vp(0x40000), vp(0x50000), None, vp(0x60000), vp(0x70000), 0, vp(0x10000),
            1 << 30, None]
    a2 = list(args)
    a2[6] = None  # dweight NULL
    assert L.lib.lce_backward(ctypes.byref(p), None, *a2) == 1
    a3 = list(args)
    a3[8] = vp(0x10001)
    assert L.lib.lce_backward(ctypes.byref(p), None, *a3) == 3
    # dweight_flags: bf16 cannot accumulate; unknown bits are rejected (LCE_ERR_ARG)
    for flags in (L.LCE_DW_BF16 | L.LCE_DW_ACCUMULATE, 4, -1):
        a4 = list(args)
        a4[7] = flags
        assert L.lib.lce_backward(ctypes.byref(p), None, *a4) == 11, flags


def test_fused_and_kd_reject_bf16_dweight(L):
    """The fused / KD paths sum dW over row chunks in fp32: LCE_DW_BF16 -> LCE_ERR_ARG
    (checked before anything else touches the arguments)."""
    vp = ctypes.c_void_p
    p = prob(L, 256, 64, 1000)
    x = [vp(0x20000 + 0x100 * i) for i in range(12)]
    assert L.lib.lce_forward_backward(ctypes.byref(p), None, *x[:10], L.LCE_DW_BF16, vp(0x10000), 1 << 30,
                                      None) == 11
    assert L.lib.lce_kd_forward_backward(ctypes.byref(p), None, 64, *x[:11], L.LCE_DW_BF16, vp(0x10000), 1 << 30,
                                         None) == 11


def test_expect_grad_and_comm_check_arguments(L):
    vp = ctypes.c_void_p
    assert L.lib.lce_expect_grad(None, 1.0, vp(0x10000), None) == 1
    assert L.lib.lce_expect_grad(vp(0x20000), 1.0, None, None) == 1
    assert L.lib.lce_expect_grad(vp(0x20000), 1.0, vp(0x10008), None) == 3
    assert L.lib.lce_comm_check(None) == 0


def test_comm_arguments(L):
    h = ctypes.c_void_p()
    assert L.lib.lce_comm_init(None, b"\0" * 128, 1, 0) == 1
    assert L.lib.lce_comm_init(ctypes.byref(h), b"\0" * 128, 0, 0) == 2
    assert L.lib.lce_comm_init(ctypes.byref(h), b"\0" * 128, 2, 2) == 2
    assert L.lib.lce_comm_size(None) == 1 and L.lib.lce_comm_rank(None) == 0
    assert L.lib.lce_comm_destroy(None) == 0


def test_profiler_roundtrip_without_launches(L):
    ms = (ctypes.c_double * L.LCE_K_COUNT)()
    n = (ctypes.c_int64 * L.LCE_K_COUNT)()
    assert L.lib.lce_profile_enable(1) == 0
    assert L.lib.lce_profile_read(ms, n) == 0
    assert list(n) == [0] * L.LCE_K_COUNT
    assert L.lib.lce_profile_enable(0) == 0


def test_product_path_has_no_oracle_or_fallback():
    """The package never imports oracle/ and has no CPU fallback code path."""
    pkg = os.path.join(ROOT, "paper_2605_21442_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "oracle" not in src.replace("oracle/", "").replace("CPU oracle", ""), f
            assert "torch.nn.functional.cross_entropy" not in src, f


def test_binding_does_no_method_arithmetic():
    """Boundary: the Python layer only marshals arguments.  No
    arithmetic operator, dtype conversion or torch math is applied to a
    method output in paper_2605_21442_b200/*.py -- gradient scaling, bf16
    rounding of dW / dH, loss reductions all happen in liblce.so."""
    import ast

    pkg = os.path.join(ROOT, "paper_2605_21442_b200")
    outputs = {"dh", "dw", "dhidden", "dweight", "loss", "lse", "token_loss", "out", "tok"}
    banned_calls = {"to", "float", "half", "bfloat16", "double", "mul", "mul_", "div", "div_", "add", "add_",
                    "sum", "mean", "exp", "log", "sub", "sub_", "type"}
    for f in sorted(os.listdir(pkg)):
        if not f.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(pkg, f)).read())

        def base_name(node):
            while isinstance(node, (ast.Attribute, ast.Subscript)):
                node = node.value
            return node.id if isinstance(node, ast.Name) else None

        for node in ast.walk(tree):
            if isinstance(node, ast.BinOp) and isinstance(node.op, (ast.Mult, ast.Div, ast.Add, ast.Sub, ast.Pow)):
                for side in (node.left, node.right):
                    assert base_name(side) not in outputs, (f, node.lineno, ast.unparse(node))
            if isinstance(node, ast.AugAssign):
                assert base_name(node.target) not in outputs, (f, node.lineno, ast.unparse(node))
            if isinstance(node, ast.Call) and isinstance(node.func, ast.Attribute):
                if node.func.attr in banned_calls:
                    assert base_name(node.func.value) not in outputs, (f, node.lineno, ast.unparse(node))


def test_debug_build_exports_the_same_symbols(L):
    """liblce_debug.so (trapping spin-wait timeouts) is the same ABI."""
    mod = __import__("__graft_entry__").load_build_module()
    path = mod.build_debug()
    dbg = ctypes.CDLL(path)
    for n in header_functions():
        assert hasattr(dbg, n), n


def test_drop_in_marshalling_on_host(L):
    """linear_cross_entropy's drop-in form: [..., D] hidden and [...]
    integer labels become [N, D] / int32 [N]; int64 labels outside the int32
    range stay out of range (clamped) instead of wrapping; mismatches raise."""
    import torch

    from paper_2605_21442_b200.lce import _flatten_drop_in

    h = torch.zeros(2, 3, 8, dtype=torch.bfloat16)
    y = torch.tensor([[0, 1, -100], [2 ** 32 + 5, -(2 ** 40), 7]], dtype=torch.int64)
    h2, y2 = _flatten_drop_in(h, y)
    assert tuple(h2.shape) == (6, 8) and h2.data_ptr() == h.data_ptr()  # a view
    assert y2.dtype == torch.int32 and y2.is_contiguous()
    assert y2.tolist() == [0, 1, -100, 2 ** 31 - 1, -(2 ** 31), 7]
    with pytest.raises(ValueError):
        _flatten_drop_in(h, y[:, :2])
    with pytest.raises(TypeError):
        _flatten_drop_in(h, y.float())


def test_fused_row_buffers_bounded_for_small_vocab(L):
    """Small vocabulary, many tokens (V = 1000, N = 2^20, D = 4096): the fused
    chunk's N_c x D row buffers (H_c, scaled H, fp32 dH: 8 bytes per element)
    stay within the 2 GiB budget, so the workspace is O(N) + budget-bounded
    chunk buffers, not O(N/2 x D)."""
    N, D, V = 1 << 20, 4096, 1000
    w = L.lib.lce_fused_workspace_bytes(ctypes.byref(prob(L, N, D, V)))
    per_row = 64  # index / label / lse / reference / factor sections: a few words per token
    assert 0 < w < N * per_row + 3 * (2 << 30), w


def test_missing_library_fails_loudly(tmp_path):
    """No liblce.so -> importing the package raises; there is nothing to fall back to."""
    import subprocess
    import sys

    env = dict(os.environ, LCE_LIB_PATH=str(tmp_path / "no_such_liblce.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2605_21442_b200"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "liblce" in (r.stderr + r.stdout)
