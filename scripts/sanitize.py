"""Small workload over every entry point for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): every GEMM variant (256x256 CTA pairs,
512x256 wide pairs, single CTA), ragged shapes, ignored
rows, several vocab / row chunks, reduction NONE, the fused path (with and
without a one-rank communicator), AdamW-in-backward and the KD loss.

    compute-sanitizer --tool memcheck python scripts/sanitize.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import make_inputs  # noqa: E402


def main():
    comm = F.Comm.single()
    for variant in ("pair", "wide", "single"):
        os.environ["LCE_GEMM"] = variant
        for (N, D, V, budget) in [(300, 72, 1000, 0), (130, 64, 513, 300 * 2 * 256)]:
            inp = make_inputs(N, D, V, k=N, device="cuda", ignore_frac=0.2)
            h, w, y = inp.hidden, inp.weight, inp.labels
            out = F.forward(h, w, y, with_token_loss=True, chunk_budget_bytes=budget)
            F.backward(h, w, y, out["lse"], chunk_budget_bytes=budget)
            g = torch.randn(N, device="cuda")
            o2 = F.forward(h, w, y, reduction="none")
            F.backward(h, w, y, o2["lse"], grad_loss=g, reduction="none")
            F.forward_backward(h, w, y, chunk_budget_bytes=256 * 6 * 1024)
            F.forward_backward(h, w, y, comm=comm, chunk_budget_bytes=256 * 6 * 1024)
            os.environ["LCE_NVLS"] = "2"  # the NVLS dH sequence (one-rank unicast emulation)
            F.forward_backward(h, w, y, comm=comm, chunk_budget_bytes=256 * 2 * 1024)
            o3 = F.forward(h, w, y, comm=comm)
            F.backward(h, w, y, o3["lse"], comm=comm, chunk_budget_bytes=budget)
            del os.environ["LCE_NVLS"]
            F.backward(h, w, y, out["lse"], chunk_budget_bytes=budget, dweight_dtype=torch.bfloat16)
            theta = w.float().clone()
            m = torch.zeros_like(theta)
            v = torch.zeros_like(theta)
            F.backward_adamw(h, w, y, out["lse"], theta, m, v, lr=1e-3, step=1, chunk_budget_bytes=budget)
            t = make_inputs(N, 2 * D, V, k=N + 1, device="cuda", label_override=y.cpu().numpy())
            F.kd_forward_backward(h, w, t.hidden, t.weight, y, chunk_budget_bytes=256 * 10 * 1024)
            torch.cuda.synchronize()
            print(variant, N, D, V, "loss", out["loss"].item(), flush=True)
    comm.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
