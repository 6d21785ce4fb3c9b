"""cuBLAS (torch.matmul, bf16) on the three GEMM shapes of one fused 8B row
chunk, timed back to back for a few seconds each with the SM clock sampled:
the library reference point for the per-class TF/s `bench.py` reports.

    python scripts/gemm_vs_cublas.py [--rows 8192] [--D 4096] [--V 128256] [--seconds 3]

cuBLAS writes a bf16 output (the fwd shape's 2.1 GB logit matrix included),
which our kernels do not; the comparison is of tensor throughput and clock.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402


def run(fn, flops, seconds):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    reps = max(3, int(seconds * 1e3 / max(a.elapsed_time(b), 1e-3)))
    cs = ClockSampler(torch.cuda.current_device())
    cs.start()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    clk = cs.stop()
    ms = a.elapsed_time(b) / reps
    return {"ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1), "clocks": clk}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--D", type=int, default=4096)
    ap.add_argument("--V", type=int, default=128256)
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    H = torch.randn(a.rows, a.D, device="cuda", generator=g).bfloat16()
    W = (torch.randn(a.V, a.D, device="cuda", generator=g) / a.D ** 0.5).bfloat16()
    G = (torch.randn(a.rows, a.V, device="cuda", generator=g) * 1e-5).bfloat16()
    flops = 2.0 * a.rows * a.V * a.D
    out = {}
    out["fwd  H W^T"] = run(lambda: torch.matmul(H, W.t()), flops, a.seconds)
    out["dH   G W"] = run(lambda: torch.matmul(G, W), flops, a.seconds)
    out["dW   G^T H"] = run(lambda: torch.matmul(G.t(), H), flops, a.seconds)
    print(json.dumps({"shape": vars(a), "cublas_bf16": out}))


if __name__ == "__main__":
    main()
