"""Seeded synthetic LCE inputs with the shapes and structure of the paper's workloads.

Recipe:
* H ~ N(0, 1) rounded to bf16 (post-RMSNorm hidden states have O(1) RMS).
* W ~ N(0, 1/D) rounded to bf16, so logits are ~N(0, 1).
* regime "random": loss ~ ln V + 0.5.  regime "confident": for valid rows
  h_i <- h_i + kappa * W_{y_i} / ||W_{y_i}||^2 (kappa = 12), raising the target
  logit by ~12 (loss ~ 1), the SFT-like regime where p_target ~ 1.
* labels: uniform in [0, V) with exactly round(f * N) ignored rows (seeded
  permutation), or the packed-sequence structure of the Qwen config (P:266-285
  Table 3 packing; S:483 label shift: the last label of each document and the
  padding are ignore_index; a prompt prefix is ignore_index).
* seeds for config k: H 1000+k, W 2000+k, labels 3000+k, packing 0.

Big tensors are generated directly on the target device with a torch
generator; the oracle always reads back the exact bf16 values the GPU saw,
so no CPU/GPU RNG agreement is needed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

IGNORE = -100

# name: (N, D, V, label structure, ignored fraction)  -- BASELINE.json "configs"
CONFIGS = {
    "tiny": dict(N=256, D=64, V=1000, labels="uniform", ignore_frac=0.10, k=0),
    "llama1b": dict(N=8192, D=2048, V=128256, labels="uniform", ignore_frac=0.0, k=1),
    "llama8b": dict(N=16384, D=4096, V=128256, labels="uniform", ignore_frac=0.0, k=2),
    "qwen7b": dict(N=16384, D=3584, V=152064, labels="packed", ignore_frac=None, k=3),
    "llama70b": dict(N=65536, D=8192, V=128256, labels="uniform", ignore_frac=0.0, k=4),
    # App. A: ~1M-token context-parallel samples on a Llama 3.2 model,
    # where the loss phase was the peak-memory phase; 1B head shape, packed SFT labels
    "llama1b_1m": dict(N=1048576, D=2048, V=128256, labels="packed", ignore_frac=None, k=5),
}


@dataclass
class LceInputs:
    hidden: torch.Tensor   # [N, D] bf16
    weight: torch.Tensor   # [V, D] bf16
    labels: torch.Tensor   # [N] int32
    ignore_index: int = IGNORE


def uniform_labels(N: int, V: int, ignore_frac: float, seed: int,
                   ignore_index: int = IGNORE) -> np.ndarray:
    """Uniform labels in [0, V) with exactly round(ignore_frac * N) ignored rows."""
    rng = np.random.Generator(np.random.PCG64(seed))
    y = rng.integers(0, V, size=N, dtype=np.int64)
    n_ign = int(round(ignore_frac * N))
    if n_ign:
        y[rng.permutation(N)[:n_ign]] = ignore_index
    return y.astype(np.int32)


def packed_labels(N: int, V: int, seed: int, pack_len: int = 2048,
                  ignore_index: int = IGNORE) -> np.ndarray:
    """Labels of greedily packed SFT documents (Table 3 packing, S:483 label shift).

    Documents have length U{32..1024}; each is filled into the current pack
    if it fits, else the pack's tail is padded; a tail shorter than 32 is
    padding.  Within a document of length n the first floor(n * U[0.3, 0.6])
    labels (the prompt) and the last label (no next token) are ignored.
    """
    assert N % pack_len == 0
    rng = np.random.Generator(np.random.PCG64(seed))
    y = np.full(N, ignore_index, dtype=np.int64)
    for p in range(N // pack_len):
        pos = 0
        base = p * pack_len
        while pack_len - pos >= 32:
            n = int(rng.integers(32, 1025))
            if n > pack_len - pos:
                break
            prompt = int(np.floor(n * rng.uniform(0.3, 0.6)))
            toks = rng.integers(0, V, size=n)
            lab = toks.copy()
            lab[:prompt] = ignore_index
            lab[-1] = ignore_index
            y[base + pos: base + pos + n] = lab
            pos += n
    return y.astype(np.int32)


def make_labels(N: int, V: int, structure: str, ignore_frac, seed: int) -> np.ndarray:
    if structure == "uniform":
        return uniform_labels(N, V, ignore_frac or 0.0, seed)
    if structure == "packed":
        return packed_labels(N, V, seed)
    raise ValueError(structure)


def make_inputs(N: int, D: int, V: int, *, k: int = 0, device="cpu",
                labels="uniform", ignore_frac: float = 0.1, regime: str = "random",
                kappa: float = 12.0, label_override=None) -> LceInputs:
    """Seeded (H, W, y) for one problem.  See module docstring for the recipe."""
    dev = torch.device(device)
    gh = torch.Generator(device=dev).manual_seed(1000 + k)
    gw = torch.Generator(device=dev).manual_seed(2000 + k)
    if label_override is not None:
        y_np = np.asarray(label_override, dtype=np.int32)
    else:
        y_np = make_labels(N, V, labels, ignore_frac, 3000 + k)
    y = torch.from_numpy(y_np).to(dev)
    W32 = torch.randn(V, D, generator=gw, device=dev, dtype=torch.float32) / np.sqrt(D)
    W = W32.to(torch.bfloat16)
    H32 = torch.randn(N, D, generator=gh, device=dev, dtype=torch.float32)
    if regime == "confident" and N > 0:
        valid = y != IGNORE
        yy = torch.where(valid, y, torch.zeros_like(y)).long()
        Wy = W[yy].float()
        bump = kappa * Wy / (Wy * Wy).sum(dim=1, keepdim=True)
        H32 = torch.where(valid[:, None], H32 + bump, H32)
    elif regime != "random":
        raise ValueError(regime)
    H = H32.to(torch.bfloat16)
    return LceInputs(hidden=H.contiguous(), weight=W.contiguous(), labels=y.contiguous())


def make_config(name: str, device="cpu", regime: str = "random", n_override=None) -> LceInputs:
    c = CONFIGS[name]
    N = n_override if n_override is not None else c["N"]
    return make_inputs(N, c["D"], c["V"], k=c["k"], device=device, labels=c["labels"],
                       ignore_frac=c["ignore_frac"], regime=regime)
