"""Measured parity margins vs the fp64 oracle (writes a markdown table).

    python scripts/parity_report.py > profiles/round1_parity_margins.md
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from oracle import lce_backward, lce_forward  # noqa: E402
from synth.inputs import CONFIGS, make_config, make_inputs, packed_labels  # noqa: E402


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a))


def run(inp, path):
    if path == "fused":
        o = F.forward_backward(inp.hidden, inp.weight, inp.labels, with_token_loss=True)
        dh, dw = o["dhidden"], o["dweight"]
    else:
        o = F.forward(inp.hidden, inp.weight, inp.labels, with_token_loss=True)
        dh, dw = F.backward(inp.hidden, inp.weight, inp.labels, o["lse"])
    torch.cuda.synchronize()
    return o["loss"].item(), o["lse"].cpu().double().numpy(), dh.float().cpu().double().numpy(), \
        dw.cpu().double().numpy()


def main():
    cases = [("tiny", "random", make_config("tiny", device="cuda")),
             ("tiny", "confident", make_config("tiny", device="cuda", regime="confident"))]
    for name in ("llama8b", "qwen7b", "llama70b"):
        c = CONFIGS[name]
        lab = packed_labels(2048, c["V"], seed=0)[1000:1300] if c["labels"] == "packed" else None
        for regime in ("random", "confident"):
            cases.append((f"{name} (N=300)", regime,
                          make_inputs(300, c["D"], c["V"], k=c["k"], device="cuda", ignore_frac=0.1,
                                      label_override=lab, regime=regime)))
    print("# Parity margins vs the fp64 oracle (round 1, one B200)\n")
    print("Bars: loss 2e-3 relative; dH, dW 1e-2 relative Frobenius; lse 1e-3 relative.\n")
    print("| shape | regime | path | loss rel err | lse max rel err | dH rel Frobenius | dW rel Frobenius |")
    print("|---|---|---|---|---|---|---|")
    for name, regime, inp in cases:
        H, W, y = inp.hidden.float().cpu().numpy(), inp.weight.float().cpu().numpy(), inp.labels.cpu().numpy()
        f = lce_forward(H, W, y)
        b = lce_backward(H, W, y)
        for path in ("split", "fused"):
            loss, lse, dh, dw = run(inp, path)
            lerr = np.abs(lse - f["lse"]) / np.maximum(1, np.abs(f["lse"]))
            lrel = abs(loss - f["loss"]) / abs(f["loss"]) if f["loss"] else abs(loss)
            print(f"| {name} | {regime} | {path} | {lrel:.2e} | {lerr.max():.2e} | "
                  f"{rel(dh, b['dH']):.2e} | {rel(dw, b['dW']):.2e} |", flush=True)


if __name__ == "__main__":
    main()
