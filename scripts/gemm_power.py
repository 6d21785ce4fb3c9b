"""Power / clock of one GEMM shape run back to back: cuBLAS vs the library's
pair and wide mainloops (fp32 output through the dW epilogue's TMA-store
drain, LCE_DEBUG_GEMM_TMA) on the same operands (the three GEMMs of one fused
8B row chunk, with the step's value distributions: H ~ N(0,1), W ~ N(0,1/D),
q = e^(z - ref) in bf16).  Prints ms, TF/s, median SM MHz, power and
TF/s per GHz (utilisation at clock) per arm.

    python scripts/gemm_power.py [--rows 8192] [--seconds 3] [--shapes fwd,dh,dw]
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from bench import ClockSampler  # noqa: E402

CLS = {"fwd": "2", "dh": "5", "dw": "6"}  # kernel class whose raster / hints the GEMM uses
PEAK_PER_GHZ = 148 * 8192 / 1e3  # dense bf16 TF/s per GHz of SM clock (2.25 PF at ~1.9 GHz)


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
    clk = cs.stop() or {}
    ms = a.elapsed_time(b) / reps
    tf = flops / ms / 1e9
    mhz = clk.get("sm_mhz") or 0
    return {"ms": round(ms, 3), "tflops": round(tf, 1), "sm_mhz": mhz, "power_w": clk.get("power_w"),
            "util_at_clock": round(tf / (PEAK_PER_GHZ * mhz / 1e3), 3) if mhz else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--D", type=int, default=4096)
    ap.add_argument("--V", type=int, default=128256)
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--shapes", default="fwd,dh,dw")
    ap.add_argument("--arms", default="cublas,cublas32,pair,wide")
    ap.add_argument("--once", action="store_true", help="one launch per arm (under ncu)")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    n, D, V = a.rows, a.D, a.V
    H = torch.randn(n, D, device="cuda", generator=g).bfloat16()
    W = (torch.randn(V, D, device="cuda", generator=g) / D ** 0.5).bfloat16()
    z = torch.empty(n, V, device="cuda")
    G = torch.empty(n, V, device="cuda", dtype=torch.bfloat16)
    for r in range(0, n, 1024):  # q = e^(z - ref), z = h W^T, ref = a random row's logit
        zz = H[r:r + 1024].float() @ W.float().t()
        ref = zz.gather(1, torch.randint(0, V, (zz.shape[0], 1), device="cuda", generator=g))
        G[r:r + 1024] = torch.exp(zz - ref).bfloat16()
    del z
    flops = 2.0 * n * V * D
    shapes = {
        "fwd": ((H, W.t()), lambda: F.debug_gemm(H, W, n, V, D, False, False)),
        "dh": ((G, W), lambda: F.debug_gemm(G, W, n, D, V, False, True)),
        "dw": ((G.t(), H), lambda: F.debug_gemm(G, H, V, D, n, True, True)),
    }
    out = {}
    for s in a.shapes.split(","):
        cub, ours = shapes[s]
        for arm in a.arms.split(","):
            if a.once:
                fn = (lambda: torch.mm(*cub, out_dtype=torch.float32)) if arm == "cublas32" else (
                    (lambda: torch.mm(*cub)) if arm == "cublas" else ours)
                if arm not in ("cublas", "cublas32"):
                    os.environ["LCE_GEMM"] = arm
                    os.environ["LCE_DEBUG_GEMM_TMA"] = "1"
                os.environ["LCE_DEBUG_GEMM_CLS"] = CLS[s]
                torch.cuda.nvtx.range_push("measure")
                fn()
                torch.cuda.synchronize()
                torch.cuda.nvtx.range_pop()
                os.environ.pop("LCE_GEMM", None)
                os.environ.pop("LCE_DEBUG_GEMM_TMA", None)
                continue
            if arm == "cublas":  # bf16 output
                r = run(lambda: torch.mm(*cub), flops, a.seconds)
            elif arm == "cublas32":  # fp32 output, as ours
                r = run(lambda: torch.mm(*cub, out_dtype=torch.float32), flops, a.seconds)
            else:
                os.environ["LCE_GEMM"] = arm
                os.environ["LCE_DEBUG_GEMM_TMA"] = "1"
                os.environ["LCE_DEBUG_GEMM_CLS"] = CLS[s]
                r = run(ours, flops, a.seconds)
                del os.environ["LCE_GEMM"], os.environ["LCE_DEBUG_GEMM_TMA"]
            out[f"{s}/{arm}"] = r
            print(f"{s:4s} {arm:7s} {json.dumps(r)}", flush=True)
    print(json.dumps({"shape": vars(a), "results": out}))


if __name__ == "__main__":
    main()
