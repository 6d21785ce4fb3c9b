"""Measured parity margins vs the fp64 oracle (writes a markdown table).

    python scripts/parity_report.py > profiles/round2_parity_margins.md

Part 1: every config's exact (D, V) at N = 300, full oracle, both regimes,
both paths.  Part 2: every config at FULL size, both paths (bench launch
configuration): the oracle's own lse for every row (lce_lse), loss, every
row's lse, 48 sampled dH rows (lce_rows) and ~570 sampled dW rows
(lce_dweight_rows) -- the quantities tests/test_parity.py bounds.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from oracle import lce_backward, lce_dweight_rows, lce_forward, lce_lse, lce_rows  # noqa: E402
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
    for name in ("llama1b", "llama8b", "qwen7b", "llama70b"):
        c = CONFIGS[name]
        lab = packed_labels(2048, c["V"], seed=0)[1000:1300] if c["labels"] == "packed" else None
        for regime in ("random", "confident"):
            cases.append((f"{name} (N=300)", regime,
                          make_inputs(300, c["D"], c["V"], k=c["k"], device="cuda", ignore_frac=0.1,
                                      label_override=lab, regime=regime)))
    print("# Parity margins vs the fp64 oracle (round 2, one B200)\n")
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
    print("\n## Full size (bench launch configuration; dH / dW on sampled rows, oracle lse of every row)\n")
    print("| config | regime | path | loss rel err | lse max rel err (all rows) | dH rel Frobenius (50 rows) | "
          "dW rel Frobenius (~570 vocab rows) |")
    print("|---|---|---|---|---|---|---|")
    for name, regime in (("llama1b", "random"), ("llama8b", "random"), ("llama8b", "confident"),
                         ("qwen7b", "random"), ("llama70b", "random")):
        inp = make_config(name, device="cuda", regime=regime)
        H, W, y = inp.hidden.float().cpu().numpy(), inp.weight.float().cpu().numpy(), inp.labels.cpu().numpy()
        lse_o = lce_lse(H, W, y)
        valid = y != -100
        rows = np.flatnonzero(valid)
        nv = rows.size
        zt = np.einsum("ij,ij->i", H[rows].astype(np.float64), W[y[rows]].astype(np.float64))
        loss_o = float((lse_o[rows] - zt).sum() / nv)
        rng = np.random.default_rng(7)
        V = W.shape[0]
        J = np.unique(np.concatenate([rng.choice(V, 256, replace=False), np.arange(V - 256, V),
                                      y[rng.choice(rows, 64, replace=False)]]))
        dwo = lce_dweight_rows(H, W, y, J, lse=lse_o)["dW_rows"]
        R = np.sort(np.concatenate([rng.choice(len(y), 48, replace=False), [0, len(y) - 1]]))
        dho = lce_rows(H, W, y, R, n_valid=nv)["dH"]
        for path in ("split", "fused"):
            if path == "fused":
                o = F.forward_backward(inp.hidden, inp.weight, inp.labels)
                dh, dw = o["dhidden"], o["dweight"]
            else:
                o = F.forward(inp.hidden, inp.weight, inp.labels)
                dh, dw = F.backward(inp.hidden, inp.weight, inp.labels, o["lse"])
            torch.cuda.synchronize()
            lerr = np.abs(o["lse"].cpu().double().numpy() - lse_o) / np.maximum(1, np.abs(lse_o))
            g_dw = dw[torch.from_numpy(J).cuda()].cpu().double().numpy()
            g_dh = dh[torch.from_numpy(R).cuda()].float().cpu().double().numpy()
            print(f"| {name} | {regime} | {path} | {abs(o['loss'].item() - loss_o) / abs(loss_o):.2e} | "
                  f"{lerr.max():.2e} | {rel(g_dh, dho):.2e} | {rel(g_dw, dwo):.2e} |", flush=True)
            del o, dh, dw
        del inp


if __name__ == "__main__":
    main()
