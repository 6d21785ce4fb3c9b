"""(GPU) One (or a few) LCE steps of a config -- the target command for ncu captures.

    ncu --metrics dram__bytes_read.sum,... -k regex:EpiDW python scripts/one_step.py --config llama8b --path fused
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--path", default="fused", choices=["fused", "split"])
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    inp = make_config(a.config, device="cuda")
    H, W, y = inp.hidden, inp.weight, inp.labels
    dH = torch.empty_like(H)
    dW = torch.empty(W.shape, dtype=torch.float32, device="cuda")
    ws = F.Workspace()
    for _ in range(a.steps):
        if a.path == "fused":
            F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws)
        else:
            o = F.forward(H, W, y, workspace=ws)
            F.backward(H, W, y, o["lse"], dhidden=dH, dweight=dW, workspace=ws)
    torch.cuda.synchronize()
    print("done", F.launch_count())


if __name__ == "__main__":
    main()
