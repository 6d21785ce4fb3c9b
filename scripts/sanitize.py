"""Small LCE fwd+bwd workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck), both GEMM variants, ragged shapes and ignored rows.

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
    for variant in ("pair", "single"):
        os.environ["LCE_GEMM"] = variant
        for (N, D, V, budget) in [(300, 72, 1000, 0), (130, 64, 513, 300 * 2 * 256)]:
            inp = make_inputs(N, D, V, k=N, device="cuda", ignore_frac=0.2)
            out = F.forward(inp.hidden, inp.weight, inp.labels, with_token_loss=True, chunk_budget_bytes=budget)
            F.backward(inp.hidden, inp.weight, inp.labels, out["lse"], chunk_budget_bytes=budget)
            torch.cuda.synchronize()
            print(variant, N, D, V, "loss", out["loss"].item())
    print("sanitize workload done")


if __name__ == "__main__":
    main()
