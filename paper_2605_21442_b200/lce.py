"""PyTorch-facing binding of the C-ABI LCE library (argument marshalling only).

PyTorch provides device memory, the current stream and the process group
(for distributing the NCCL id); every step of the loss runs in liblce.so.
Cites: PAPER.md P:166 (Sec. 4.2 LCE), P:132 (drop-in for CE), P:180 (loss
parallel over the vocabulary).
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch

from ._lib import LCE_DW_ACCUMULATE, LCE_DW_BF16, KERNEL_CLASSES, LCE_K_COUNT, AdamW, Problem, check, lib
from .dist import broadcast_bytes, shard_range  # noqa: F401

MEAN, SUM, NONE = 0, 1, 2
_RED = {"mean": MEAN, "sum": SUM, "none": NONE}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_problem(n_tokens: int, hidden_dim: int, vocab_local: int, *, vocab_start: int = 0,
                 vocab_total: Optional[int] = None, ignore_index: int = -100, reduction: str = "mean",
                 chunk_budget_bytes: int = 0) -> Problem:
    if reduction not in _RED:
        raise ValueError(f"reduction must be 'mean', 'sum' or 'none', got {reduction!r}")
    return Problem(n_tokens, hidden_dim, vocab_local, vocab_start,
                   vocab_local if vocab_total is None else vocab_total, ignore_index, _RED[reduction],
                   chunk_budget_bytes)


def workspace_bytes(problem: Problem) -> int:
    return int(lib.lce_workspace_bytes(ctypes.byref(problem)))


class Workspace:
    """Caller-owned device scratch, grown on demand and reused across calls."""

    def __init__(self, device=None):
        self.device = device
        self.buf: Optional[torch.Tensor] = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


_default_ws: dict = {}


def _default_workspace(device, tag: str = "", stream=None) -> Workspace:
    """The default workspace of (device, the call's stream[, entry point]):
    calls on different streams never share scratch (a shared buffer would race)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = f"{device}{':' + tag if tag else ''}@{s.cuda_stream}"
    return _default_ws.setdefault(key, Workspace())


def _ws_for(ws: Optional[Workspace], problem: Problem, device, stream=None) -> torch.Tensor:
    if ws is None:
        ws = _default_workspace(device, stream=stream)
    need = workspace_bytes(problem)
    if need == 0:
        raise ValueError("invalid LCE problem shape")
    return ws.get(need, device)


def _check_tensor(t: Optional[torch.Tensor], name: str, dtype, shape: tuple, device) -> None:
    """Every tensor handed to the C ABI: dtype, exact shape, device, dense.
    The library builds its TMA maps and grids from the problem's N / D / V_l,
    so a mismatched buffer would be read or written out of bounds."""
    if t is None:
        return
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_cuda or t.device != device:
        raise ValueError(f"{name} must live on {device}, got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _check_inputs(hidden, weight, labels):
    """hidden [N, D] bf16, weight [V_l, D] bf16, labels [N] int32, one CUDA device."""
    if hidden.dim() != 2 or weight.dim() != 2:
        raise ValueError("hidden must be [N, D] and weight [V_l, D]")
    N, D = hidden.shape
    dev = hidden.device
    _check_tensor(hidden, "hidden", torch.bfloat16, (N, D), dev)
    _check_tensor(weight, "weight", torch.bfloat16, (weight.shape[0], D), dev)
    _check_tensor(labels, "labels", torch.int32, (N,), dev)
    return N, D, weight.shape[0]


def _grad_input(grad_loss, n: int, device) -> Optional[torch.Tensor]:
    """The upstream gradient as the device fp32 vector the ABI takes: [N] for
    'none', [1] otherwise (input marshalling; None means 1)."""
    if grad_loss is None:
        return None
    g = torch.as_tensor(grad_loss).to(device=device, dtype=torch.float32).reshape(-1).contiguous()
    if g.numel() != n:
        raise ValueError(f"grad_loss must have {n} element(s) (N for 'none', 1 otherwise), got {g.numel()}")
    return g


def _check_out(out: dict, N: int, dev) -> None:
    _check_tensor(out.get("loss"), "out['loss']", torch.float32, (1,), dev)
    _check_tensor(out.get("lse"), "out['lse']", torch.float32, (N,), dev)
    _check_tensor(out.get("n_valid"), "out['n_valid']", torch.int32, (1,), dev)
    _check_tensor(out.get("token_loss"), "out['token_loss']", torch.float32, (N,), dev)


PARALLEL_MODES = {"vocab": 0, "token": 1}  # lce_parallel_t


class Comm:
    """Communicator (NCCL over NVLink) owned by the library.

    mode "vocab" (P:180 loss parallel): W sharded by rows, identical hidden /
    labels on every rank.  mode "token": W replicated, each rank its own rows;
    MEAN uses the global N_v and dweight is the rank's share (include/lce.h)."""

    def __init__(self, handle: ctypes.c_void_p, world: int, rank: int, mode: str = "vocab"):
        self.handle = handle
        self.world = world
        self.rank = rank
        self.mode = mode

    @classmethod
    def from_process_group(cls, group=None, mode: str = "vocab") -> "Comm":
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        payload = None
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            check(lib.lce_comm_get_unique_id(buf), "lce_comm_get_unique_id")
            payload = bytes(buf.raw)
        uid = broadcast_bytes(payload, group=group)
        h = ctypes.c_void_p()
        check(lib.lce_comm_init_mode(ctypes.byref(h), uid, world, rank, PARALLEL_MODES[mode]), "lce_comm_init_mode")
        return cls(h, world, rank, mode)

    @classmethod
    def single(cls, mode: str = "vocab") -> "Comm":
        """A one-rank communicator: exercises the exchange path on one GPU."""
        buf = ctypes.create_string_buffer(128)
        check(lib.lce_comm_get_unique_id(buf), "lce_comm_get_unique_id")
        h = ctypes.c_void_p()
        check(lib.lce_comm_init_mode(ctypes.byref(h), bytes(buf.raw), 1, 0, PARALLEL_MODES[mode]),
              "lce_comm_init_mode")
        return cls(h, 1, 0, mode)

    def check(self) -> None:
        """lce_comm_check: raises LceError(LCE_ERR_NCCL) if NCCL reported an
        asynchronous error on this communicator (host only, no sync)."""
        check(lib.lce_comm_check(self.handle), "lce_comm_check")

    def close(self):
        if self.handle:
            check(lib.lce_comm_destroy(self.handle), "lce_comm_destroy")
            self.handle = None


def forward(hidden: torch.Tensor, weight: torch.Tensor, labels: torch.Tensor, *, ignore_index: int = -100,
            reduction: str = "mean", comm: Optional[Comm] = None, vocab_start: int = 0,
            vocab_total: Optional[int] = None, with_token_loss: bool = False, workspace: Optional[Workspace] = None,
            chunk_budget_bytes: int = 0, stream=None, out: Optional[dict] = None) -> dict:
    """loss [1] fp32, lse [N] fp32 (0 on ignored rows), n_valid [1] int32, token_loss.

    reduction 'none' returns the per-token losses (-log p(y_i)) in token_loss
    and their sum in loss."""
    with_token_loss = with_token_loss or reduction == "none"
    N, D, Vl = _check_inputs(hidden, weight, labels)
    prob = make_problem(N, D, Vl, vocab_start=vocab_start, vocab_total=vocab_total,
                        ignore_index=ignore_index, reduction=reduction, chunk_budget_bytes=chunk_budget_bytes)
    dev = hidden.device
    ws = _ws_for(workspace, prob, dev, stream)
    if out is None:
        out = {
            "loss": torch.empty(1, dtype=torch.float32, device=dev),
            "lse": torch.empty(N, dtype=torch.float32, device=dev),
            "n_valid": torch.empty(1, dtype=torch.int32, device=dev),
            "token_loss": torch.empty(N, dtype=torch.float32, device=dev) if with_token_loss else None,
        }
    _check_out(out, N, dev)
    check(lib.lce_forward(ctypes.byref(prob), comm.handle if comm else None, _ptr(hidden), _ptr(weight),
                          _ptr(labels), _ptr(out["loss"]), _ptr(out["lse"]), _ptr(out["token_loss"]),
                          _ptr(out["n_valid"]), _ptr(ws), ws.numel(), _stream(stream)), "lce_forward")
    return out


def backward(hidden: torch.Tensor, weight: torch.Tensor, labels: torch.Tensor, lse: torch.Tensor, *,
             grad_loss: Optional[torch.Tensor] = None, ignore_index: int = -100, reduction: str = "mean",
             comm: Optional[Comm] = None, vocab_start: int = 0, vocab_total: Optional[int] = None,
             dhidden: Optional[torch.Tensor] = None, dweight: Optional[torch.Tensor] = None,
             accumulate_dweight: bool = False, workspace: Optional[Workspace] = None, chunk_budget_bytes: int = 0,
             stream=None, dweight_dtype=torch.float32):
    """dhidden [N, D] bf16 and dweight [V_l, D] (overwritten or accumulated).

    grad_loss: scalar dL/dloss for 'mean'/'sum'; [N] per-token dL/dloss_i for 'none'.
    dweight_dtype: torch.float32 (default), or torch.bfloat16 -- the library
    rounds the fp32 accumulator to bf16 itself (LCE_DW_BF16; not with
    accumulate_dweight)."""
    N, D, Vl = _check_inputs(hidden, weight, labels)
    if dweight_dtype not in (torch.float32, torch.bfloat16):
        raise TypeError("dweight_dtype must be torch.float32 or torch.bfloat16")
    prob = make_problem(N, D, Vl, vocab_start=vocab_start, vocab_total=vocab_total,
                        ignore_index=ignore_index, reduction=reduction, chunk_budget_bytes=chunk_budget_bytes)
    dev = hidden.device
    _check_tensor(lse, "lse", torch.float32, (N,), dev)
    ws = _ws_for(workspace, prob, dev, stream)
    if dhidden is None:
        dhidden = torch.empty_like(hidden)
    if dweight is None:
        dweight = torch.empty(weight.shape, dtype=dweight_dtype, device=dev)
    _check_tensor(dhidden, "dhidden", torch.bfloat16, (N, D), dev)
    _check_tensor(dweight, "dweight", dweight_dtype, (Vl, D), dev)
    grad_loss = _grad_input(grad_loss, N if reduction == "none" else 1, dev)
    flags = (LCE_DW_ACCUMULATE if accumulate_dweight else 0) | (LCE_DW_BF16 if dweight_dtype == torch.bfloat16 else 0)
    check(lib.lce_backward(ctypes.byref(prob), comm.handle if comm else None, _ptr(hidden), _ptr(weight),
                           _ptr(labels), _ptr(lse), _ptr(grad_loss), _ptr(dhidden), _ptr(dweight),
                           flags, _ptr(ws), ws.numel(), _stream(stream)), "lce_backward")
    return dhidden, dweight


def backward_adamw(hidden: torch.Tensor, weight: torch.Tensor, labels: torch.Tensor, lse: torch.Tensor,
                   master_weight: torch.Tensor, exp_avg: torch.Tensor, exp_avg_sq: torch.Tensor, *, lr: float,
                   step: int, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0,
                   grad_loss: Optional[torch.Tensor] = None, ignore_index: int = -100, reduction: str = "mean",
                   comm: Optional[Comm] = None, vocab_start: int = 0, vocab_total: Optional[int] = None,
                   dhidden: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None,
                   chunk_budget_bytes: int = 0, stream=None) -> torch.Tensor:
    """lce_backward with the LM-head AdamW step fused into the dW epilogue
    (optimizer-in-backward).  Updates weight (bf16), master_weight,
    exp_avg, exp_avg_sq in place; returns dhidden."""
    N, D, Vl = _check_inputs(hidden, weight, labels)
    dev = hidden.device
    for name, t in (("master_weight", master_weight), ("exp_avg", exp_avg), ("exp_avg_sq", exp_avg_sq)):
        _check_tensor(t, name, torch.float32, (Vl, D), dev)
    _check_tensor(lse, "lse", torch.float32, (N,), dev)
    prob = make_problem(N, D, Vl, vocab_start=vocab_start, vocab_total=vocab_total,
                        ignore_index=ignore_index, reduction=reduction, chunk_budget_bytes=chunk_budget_bytes)
    ws = _ws_for(workspace, prob, dev, stream)
    if dhidden is None:
        dhidden = torch.empty_like(hidden)
    _check_tensor(dhidden, "dhidden", torch.bfloat16, (N, D), dev)
    grad_loss = _grad_input(grad_loss, N if reduction == "none" else 1, dev)
    hp = AdamW(lr, betas[0], betas[1], eps, weight_decay, step)
    check(lib.lce_backward_adamw(ctypes.byref(prob), comm.handle if comm else None, _ptr(hidden), _ptr(weight),
                                 _ptr(labels), _ptr(lse), _ptr(grad_loss), _ptr(dhidden), _ptr(master_weight),
                                 _ptr(exp_avg), _ptr(exp_avg_sq), ctypes.byref(hp), _ptr(ws), ws.numel(),
                                 _stream(stream)), "lce_backward_adamw")
    return dhidden


def fused_workspace_bytes(problem: Problem) -> int:
    return int(lib.lce_fused_workspace_bytes(ctypes.byref(problem)))


def forward_backward(hidden: torch.Tensor, weight: torch.Tensor, labels: torch.Tensor, *,
                     grad_loss: Optional[torch.Tensor] = None, ignore_index: int = -100, reduction: str = "mean",
                     with_token_loss: bool = False, dhidden: Optional[torch.Tensor] = None,
                     dweight: Optional[torch.Tensor] = None, accumulate_dweight: bool = False,
                     workspace: Optional[Workspace] = None, chunk_budget_bytes: int = 0, stream=None,
                     out: Optional[dict] = None, comm: Optional[Comm] = None, vocab_start: int = 0,
                     vocab_total: Optional[int] = None) -> dict:
    """Fused forward + backward without logit recompute (lce_forward_backward).

    Returns {loss, lse, n_valid, token_loss, dhidden, dweight}; dweight is fp32
    (summed over row chunks).  grad_loss (the upstream gradient) must be known
    up front: scalar for 'mean'/'sum', [N] for 'none'; None = 1."""
    N, D, Vl = _check_inputs(hidden, weight, labels)
    prob = make_problem(N, D, Vl, vocab_start=vocab_start, vocab_total=vocab_total,
                        ignore_index=ignore_index, reduction=reduction, chunk_budget_bytes=chunk_budget_bytes)
    dev = hidden.device
    need = fused_workspace_bytes(prob)
    if need == 0:
        raise ValueError("invalid LCE problem shape")
    if workspace is None:
        workspace = _default_workspace(dev, "fused", stream)
    ws = workspace.get(need, dev)
    with_token_loss = with_token_loss or reduction == "none"
    if out is None:
        out = {
            "loss": torch.empty(1, dtype=torch.float32, device=dev),
            "lse": torch.empty(N, dtype=torch.float32, device=dev),
            "n_valid": torch.empty(1, dtype=torch.int32, device=dev),
            "token_loss": torch.empty(N, dtype=torch.float32, device=dev) if with_token_loss else None,
        }
    if dhidden is None:
        dhidden = torch.empty_like(hidden)
    if dweight is None:
        dweight = torch.empty(weight.shape, dtype=torch.float32, device=dev)
    _check_out(out, N, dev)
    _check_tensor(dhidden, "dhidden", torch.bfloat16, (N, D), dev)
    _check_tensor(dweight, "dweight", torch.float32, (Vl, D), dev)
    grad_loss = _grad_input(grad_loss, N if reduction == "none" else 1, dev)
    check(lib.lce_forward_backward(ctypes.byref(prob), comm.handle if comm else None, _ptr(hidden), _ptr(weight),
                                   _ptr(labels),
                                   _ptr(grad_loss), _ptr(out["loss"]), _ptr(out["lse"]), _ptr(out["token_loss"]),
                                   _ptr(out["n_valid"]), _ptr(dhidden), _ptr(dweight),
                                   1 if accumulate_dweight else 0, _ptr(ws), ws.numel(), _stream(stream)),
          "lce_forward_backward")
    out["dhidden"], out["dweight"] = dhidden, dweight
    return out


def kd_forward_backward(hidden_s: torch.Tensor, weight_s: torch.Tensor, hidden_t: torch.Tensor,
                        weight_t: torch.Tensor, labels: torch.Tensor, *, grad_loss: Optional[torch.Tensor] = None,
                        ignore_index: int = -100, reduction: str = "mean", dhidden: Optional[torch.Tensor] = None,
                        dweight: Optional[torch.Tensor] = None, accumulate_dweight: bool = False,
                        workspace: Optional[Workspace] = None, chunk_budget_bytes: int = 0, stream=None,
                        comm: Optional[Comm] = None, vocab_start: int = 0,
                        vocab_total: Optional[int] = None) -> dict:
    """Linear KD loss (forward KL, teacher -> student) and student gradients
    (lce_kd_forward_backward).  Returns {loss, token_loss, n_valid, dhidden, dweight}."""
    N, D, Vl = _check_inputs(hidden_s, weight_s, labels)
    Nt, Dt, Vt = _check_inputs(hidden_t, weight_t, labels)
    if Nt != N or Vt != Vl or hidden_t.device != hidden_s.device:
        raise ValueError("teacher / student shapes disagree")
    prob = make_problem(N, D, Vl, vocab_start=vocab_start, vocab_total=vocab_total,
                        ignore_index=ignore_index, reduction=reduction, chunk_budget_bytes=chunk_budget_bytes)
    dev = hidden_s.device
    need = int(lib.lce_kd_workspace_bytes(ctypes.byref(prob), Dt))
    if need == 0:
        raise ValueError("invalid KD problem shape")
    if workspace is None:
        workspace = _default_workspace(dev, "kd", stream)
    ws = workspace.get(need, dev)
    out = {"loss": torch.empty(1, dtype=torch.float32, device=dev),
           "token_loss": torch.empty(N, dtype=torch.float32, device=dev),
           "n_valid": torch.empty(1, dtype=torch.int32, device=dev)}
    if dhidden is None:
        dhidden = torch.empty_like(hidden_s)
    if dweight is None:
        dweight = torch.empty(weight_s.shape, dtype=torch.float32, device=dev)
    _check_tensor(dhidden, "dhidden", torch.bfloat16, (N, D), dev)
    _check_tensor(dweight, "dweight", torch.float32, (Vl, D), dev)
    grad_loss = _grad_input(grad_loss, N if reduction == "none" else 1, dev)
    check(lib.lce_kd_forward_backward(ctypes.byref(prob), comm.handle if comm else None, Dt, _ptr(hidden_s),
                                      _ptr(weight_s), _ptr(hidden_t),
                                      _ptr(weight_t), _ptr(labels), _ptr(grad_loss), _ptr(out["loss"]),
                                      _ptr(out["token_loss"]), _ptr(out["n_valid"]), _ptr(dhidden), _ptr(dweight),
                                      1 if accumulate_dweight else 0, _ptr(ws), ws.numel(), _stream(stream)),
          "lce_kd_forward_backward")
    out["dhidden"], out["dweight"] = dhidden, dweight
    return out


def check_device_status(workspace: Optional[Workspace] = None, device=None, stream=None) -> None:
    """Raises LceError(LCE_ERR_LABEL_RANGE) if a bad label was seen, or
    LceError(LCE_ERR_UPSTREAM) if a fused autograd call's upstream gradient
    differed from the one it assumed (syncs).  Without `workspace`, checks
    every default workspace of the device (split, fused and KD paths)."""
    if workspace is not None:
        wss = [workspace]
    else:
        dev = str(device or torch.device("cuda", torch.cuda.current_device()))
        wss = [w for k, w in _default_ws.items() if k.startswith(dev + ":") or k.startswith(dev + "@")]
    for ws in wss:
        if ws.buf is not None:
            check(lib.lce_check_device_status(_ptr(ws.buf), _stream(stream)), "lce_check_device_status")


def expect_grad(grad: torch.Tensor, expected: float, workspace: Workspace, stream=None) -> None:
    """lce_expect_grad: compare the actual upstream gradient (device [1] fp32)
    with the one a fused call assumed, on the device, no sync; a mismatch is
    raised by the next check_device_status as LCE_ERR_UPSTREAM."""
    _check_tensor(grad, "grad", torch.float32, (1,), grad.device)
    check(lib.lce_expect_grad(_ptr(grad), float(expected), _ptr(workspace.buf), _stream(stream)), "lce_expect_grad")


class LinearCrossEntropyFunction(torch.autograd.Function):
    """autograd wrapper: loss = CE(hidden @ weight^T, labels), mask-first, chunked.

    backward passes autograd's upstream gradient to lce_backward as grad_loss
    and asks the library for dW in the weight's dtype (bf16: LCE_DW_BF16, the
    library rounds its fp32 accumulator); nothing is computed here."""

    @staticmethod
    def forward(ctx, hidden, weight, labels, ignore_index, reduction):
        out = forward(hidden, weight, labels, ignore_index=ignore_index, reduction=reduction)
        ctx.save_for_backward(hidden, weight, labels, out["lse"])
        ctx.cfg = (ignore_index, reduction)
        if reduction == "none":
            return out["token_loss"]  # per-token -log p(y_i); 0 on ignored rows
        return out["loss"].reshape(())

    @staticmethod
    def backward(ctx, g):
        hidden, weight, labels, lse = ctx.saved_tensors
        ignore_index, reduction = ctx.cfg
        dh, dw = backward(hidden, weight, labels, lse, grad_loss=g, ignore_index=ignore_index,
                          reduction=reduction, dweight_dtype=weight.dtype)
        return dh, dw, None, None, None


class LinearCrossEntropyFusedFunction(torch.autograd.Function):
    """autograd wrapper over lce_forward_backward (no logit recompute).

    The fused call needs the upstream gradient before the backward exists, so
    the caller states it up front as `grad_scale` (1.0 for loss.backward();
    e.g. 1/k when the loss is divided by k for gradient accumulation): it is
    passed to the library as grad_loss and the gradients come out for it.
    backward returns them untouched -- dW in fp32, as lce_forward_backward
    sums it over row chunks (autograd's engine stores it in the parameter's
    dtype) -- and hands the actual upstream gradient to lce_expect_grad, which
    compares it with grad_scale on the device: a mismatch surfaces as
    LCE_ERR_UPSTREAM from check_device_status.  No rescaling, no host sync."""

    @staticmethod
    def forward(ctx, hidden, weight, labels, ignore_index, reduction, grad_scale):
        dev = hidden.device
        ws = _default_workspace(dev, "fused")
        g = torch.full((1,), float(grad_scale), dtype=torch.float32, device=dev)
        out = forward_backward(hidden, weight, labels, grad_loss=g, ignore_index=ignore_index, reduction=reduction,
                               workspace=ws)
        ctx.save_for_backward(out["dhidden"], out["dweight"])
        ctx.ws, ctx.scale = ws, float(grad_scale)
        return out["loss"].reshape(())

    @staticmethod
    def backward(ctx, g):
        dh, dw = ctx.saved_tensors
        expect_grad(g.reshape(1), ctx.scale, ctx.ws)
        return dh, dw, None, None, None, None


def _flatten_drop_in(hidden, labels):
    """The drop-in form of P:132 (the model's [..., D] hidden states and [...]
    class indices of any integer dtype, as torch's cross_entropy takes them)
    marshalled to the ABI's [N, D] / int32 [N]: a view of hidden (a copy if it
    is not contiguous) and the labels narrowed to int32 -- values outside the
    int32 range are clamped to an int32 value that is still out of [0, V) (or
    negative), so the library's S0 range check flags them instead of wrapping."""
    if hidden.dim() < 2 or tuple(labels.shape) != tuple(hidden.shape[:-1]):
        raise ValueError(f"hidden [..., D] and labels [...] must agree: {tuple(hidden.shape)} vs {tuple(labels.shape)}")
    if labels.dtype.is_floating_point or labels.dtype == torch.bool:
        raise TypeError(f"labels must be an integer tensor, got {labels.dtype}")
    h = hidden.reshape(-1, hidden.shape[-1])
    y = labels.reshape(-1)
    if y.dtype != torch.int32:
        y = y.clamp(-(2 ** 31), 2 ** 31 - 1).to(torch.int32)
    return h, y.contiguous()


def linear_cross_entropy(hidden, weight, labels, ignore_index: int = -100, reduction: str = "mean",
                         fused: bool = False, grad_scale: float = 1.0):
    """loss = CE(hidden @ weight^T, labels) (P:166 LCE), a drop-in for
    cross_entropy(hidden @ weight.T, labels): hidden [..., D] bf16,
    labels [...] of any integer dtype; reduction 'none' returns [...].
    fused=True computes the gradients in the forward call without the logit
    recompute (MEAN / SUM only), for the upstream gradient `grad_scale`; when
    no gradient is needed (torch.no_grad(), or neither hidden nor weight
    requires grad) it runs the forward only."""
    lead = tuple(labels.shape)
    hidden, labels = _flatten_drop_in(hidden, labels)
    if fused:
        if reduction == "none":
            raise ValueError("fused autograd needs a scalar loss (reduction 'mean' or 'sum')")
        if torch.is_grad_enabled() and (hidden.requires_grad or weight.requires_grad):
            return LinearCrossEntropyFusedFunction.apply(hidden, weight, labels, ignore_index, reduction, grad_scale)
        return forward(hidden, weight, labels, ignore_index=ignore_index, reduction=reduction)["loss"].reshape(())
    res = LinearCrossEntropyFunction.apply(hidden, weight, labels, ignore_index, reduction)
    return res.reshape(lead) if reduction == "none" else res


class LinearCrossEntropyLoss(torch.nn.Module):
    """nn.Module form of the loss the paper names (torchtune's
    LinearCrossEntropyLoss): holds the output projection (a weight
    Parameter [V, D] or an nn.Linear without bias, e.g. the model's LM head)
    and computes CE(hidden @ weight^T, labels) through linear_cross_entropy,
    never materialising the [..., V] logits."""

    def __init__(self, projection=None, ignore_index: int = -100, reduction: str = "mean", fused: bool = False):
        super().__init__()
        if reduction not in _RED:
            raise ValueError(f"reduction must be 'mean', 'sum' or 'none', got {reduction!r}")
        self.projection = projection
        self.ignore_index, self.reduction, self.fused = ignore_index, reduction, fused

    def _weight(self, weight):
        w = weight if weight is not None else self.projection
        if isinstance(w, torch.nn.Linear):
            if w.bias is not None:
                raise ValueError("the LCE projection has no bias (P:166: logits = hidden @ weight^T)")
            w = w.weight
        if w is None:
            raise ValueError("no output projection: pass one to the constructor or to forward()")
        return w

    def forward(self, hidden, labels, weight=None, grad_scale: float = 1.0):
        return linear_cross_entropy(hidden, self._weight(weight), labels, ignore_index=self.ignore_index,
                                    reduction=self.reduction, fused=self.fused, grad_scale=grad_scale)


def debug_gemm(A: torch.Tensor, B: torch.Tensor, M: int, N: int, K: int, a_mn: bool, b_mn: bool) -> torch.Tensor:
    """C = A B^T through the tcgen05 mainloop (diagnostics)."""
    C = torch.empty(M, N, dtype=torch.float32, device=A.device)
    check(lib.lce_debug_gemm(_ptr(A), _ptr(B), _ptr(C), M, N, K, int(a_mn), int(b_mn), _stream()), "lce_debug_gemm")
    return C


def launch_count() -> int:
    return int(lib.lce_launch_count())


def profile_enable(on: bool = True) -> None:
    check(lib.lce_profile_enable(1 if on else 0), "lce_profile_enable")


def profile_read() -> dict:
    """{class: (device ms, launches, mean SM MHz of its GEMM launches or None)}
    since profile_enable(); clears the record."""
    ms = (ctypes.c_double * LCE_K_COUNT)()
    n = (ctypes.c_int64 * LCE_K_COUNT)()
    cyc = (ctypes.c_double * LCE_K_COUNT)()
    ns = (ctypes.c_double * LCE_K_COUNT)()
    check(lib.lce_profile_read_clocks(ms, n, cyc, ns), "lce_profile_read_clocks")
    return {k: (ms[i], n[i], (cyc[i] / ns[i] * 1e3) if ns[i] > 0 else None) for i, k in enumerate(KERNEL_CLASSES)}
