"""Optimizer-in-backward for the LM head vs a separate AdamW step.

    python scripts/bench_adamw.py [--config llama8b] [--steps 10]

(a) lce_forward + lce_backward (dW buffer, fp32) + torch.optim.AdamW(fused=True)
    on the fp32 master copy, then the bf16 working copy refreshed;
(b) lce_forward + lce_backward_adamw: the AdamW step runs in the dW GEMM
    epilogue, no dW buffer exists.
Prints ms/step and peak HBM for both (device time, CUDA events).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import make_config  # noqa: E402


def timed(fn, steps, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps, torch.cuda.max_memory_allocated()


def breakdown(fn):
    """Per-kernel-class device ms of one step (CUDA events around each launch)."""
    F.profile_read()
    F.profile_enable(True)
    fn()
    torch.cuda.synchronize()
    F.profile_enable(False)
    return {k: round(v[0], 3) for k, v in F.profile_read().items() if v[1]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    inp = make_config(args.config, device="cuda")
    H, y = inp.hidden, inp.labels
    res = {}

    # (a) separate optimizer step
    master = torch.nn.Parameter(inp.weight.float())
    W = inp.weight.clone()
    opt = torch.optim.AdamW([master], lr=1e-5, weight_decay=0.01, fused=True)
    dW = torch.empty_like(master)
    ws = F.Workspace()

    def step_a():
        out = F.forward(H, W, y, workspace=ws)
        F.backward(H, W, y, out["lse"], dweight=dW, workspace=ws)
        master.grad = dW
        opt.step()
        W.copy_(master.detach())

    res["separate"] = timed(step_a, args.steps)
    prof = {"separate": breakdown(step_a)}
    del opt, master, dW
    torch.cuda.empty_cache()

    # (b) AdamW fused into the dW epilogue
    theta = inp.weight.float()
    m = torch.zeros_like(theta)
    v = torch.zeros_like(theta)
    W2 = inp.weight.clone()
    count = [0]

    def step_b():
        count[0] += 1
        out = F.forward(H, W2, y, workspace=ws)
        F.backward_adamw(H, W2, y, out["lse"], theta, m, v, lr=1e-5, weight_decay=0.01, step=count[0], workspace=ws)

    res["in_backward"] = timed(step_b, args.steps)
    prof["in_backward"] = breakdown(step_b)
    print(json.dumps({k: {"ms_per_step": round(t, 3), "peak_hbm_gb": round(mem / 1e9, 2), "kernels_ms": prof[k]}
                      for k, (t, mem) in res.items()}))


if __name__ == "__main__":
    main()
