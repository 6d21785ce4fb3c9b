"""Throughput of the SURVEY 8f NEXT rows and of the vocab-parallel exchange path
at a BASELINE shape, on one GPU (device time, CUDA events, inputs resident).

    python scripts/bench_next.py [--config llama8b] [--steps 10]

* none_fused   NEXT-1: reduction "none" (per-token -log p and per-token upstream
               gradients, the GRPO / DPO log-prob objective) through the fused path
* kd_fused     NEXT-4: chunked linear KD (forward KL) with a teacher head of the
               same shape: 4 GEMMs of 2 N V D per step (student and teacher forward,
               dH, dW), no logit recompute
* vp1_fused    the vocab-parallel code path (MAX / SUM exchanges of the row
               statistics, side-stream fp32 dH all-reduce) on a one-rank NCCL
               communicator: the cost of the exchange plumbing itself
* mean_fused   the bench.py default, for reference
Prints one JSON object: ms/step, tokens/s (non-ignored), executed tensor flops
per step and their rate, the dominant kernel's SM clock and peak HBM.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import IGNORE, make_config, make_inputs  # noqa: E402


def timed(fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    F.profile_read()
    F.profile_enable(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    prof = F.profile_read()
    F.profile_enable(False)
    mhz = [v[2] for v in prof.values() if v[2]]
    return a.elapsed_time(b) / steps, torch.cuda.max_memory_allocated(), (sum(mhz) / len(mhz)) if mhz else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    inp = make_config(args.config, device="cuda")
    H, W, y = inp.hidden, inp.weight, inp.labels
    N, D = H.shape
    V = W.shape[0]
    nv = int((y != IGNORE).sum().item())
    dH = torch.empty_like(H)
    dW = torch.empty(V, D, dtype=torch.float32, device=H.device)
    res = {}

    def record(name, fn, gemms):
        ms, mem, mhz = timed(fn, args.steps)
        flops = gemms * 2.0 * nv * V * D
        res[name] = {"ms_per_step": round(ms, 3), "tokens_per_s": round(nv / (ms / 1e3)),
                     "tensor_flops_per_step": flops, "tflops": round(flops / (ms / 1e3) / 1e12, 1),
                     "gemm_sm_mhz": round(mhz) if mhz else None, "peak_hbm_gb": round(mem / 1e9, 2)}

    ws = F.Workspace()
    record("mean_fused", lambda: F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws), 3)

    g = torch.full((N,), 1.0 / max(nv, 1), dtype=torch.float32, device=H.device)
    record("none_fused", lambda: F.forward_backward(H, W, y, reduction="none", grad_loss=g, dhidden=dH, dweight=dW,
                                                    workspace=ws), 3)

    comm = F.Comm.single()
    record("vp1_fused", lambda: F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws, comm=comm,
                                                   vocab_start=0, vocab_total=V), 3)
    comm.close()
    del ws
    torch.cuda.empty_cache()

    # teacher head of the same shape (a distinct random head, seeds of config k + 10)
    t = make_inputs(N, D, V, k=12, device=H.device, label_override=y.cpu().numpy())
    Ht, Wt = t.hidden, t.weight
    wk = F.Workspace()
    record("kd_fused", lambda: F.kd_forward_backward(H, W, Ht, Wt, y, dhidden=dH, dweight=dW, workspace=wk), 4)
    print(json.dumps({"config": args.config, "N": N, "N_valid": nv, "D": D, "V": V, "steps": args.steps,
                      "results": res}))


if __name__ == "__main__":
    main()
