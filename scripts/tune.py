"""In-process sweep of GEMM schedule knobs (raster group, L2 hints, variant).

    python scripts/tune.py --path fused --sweep hints

Each configuration is a set of LCE_* environment variables (read by liblce.so
at every launch); per-kernel device times come from the library's event
profiler.  Prints one line per configuration: step ms and per-class ms.
"""

import argparse
import itertools
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import make_config  # noqa: E402

K = {"fwd": 2, "g": 4, "dh": 5, "dw": 6}


def run(step, steps=4):
    step()
    torch.cuda.synchronize()
    F.profile_enable(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    prof = F.profile_read()
    F.profile_enable(False)
    return a.elapsed_time(b) / steps, {k: round(v[0] / steps, 2) for k, v in prof.items() if v[1]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--path", default="fused", choices=["fused", "split"])
    ap.add_argument("--sweep", default="hints", choices=["hints", "group", "both"])
    a = ap.parse_args()
    inp = make_config(a.config, device="cuda")
    H, W, y = inp.hidden, inp.weight, inp.labels
    dH = torch.empty_like(H)
    dW = torch.empty(W.shape, dtype=torch.float32, device="cuda")
    ws = F.Workspace()

    def step():
        if a.path == "fused":
            F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws)
        else:
            o = F.forward(H, W, y, workspace=ws)
            F.backward(H, W, y, o["lse"], dhidden=dH, dweight=dW, workspace=ws)

    classes = ["fwd", "dh", "dw"] + (["g"] if a.path == "split" else [])
    configs = [{}]
    if a.sweep in ("hints", "both"):
        for c in classes:
            for ha, hb in itertools.product([0, 1, 2], [0, 1, 2]):
                configs.append({f"LCE_HINT_A_{K[c]}": str(ha), f"LCE_HINT_B_{K[c]}": str(hb)})
    if a.sweep in ("group", "both"):
        for c in classes:
            for g in (1, 2, 4, 8, 16, 32):
                configs.append({f"LCE_GROUP_M_{K[c]}": str(g)})
    base = None
    for cfg in configs:
        for k, v in cfg.items():
            os.environ[k] = v
        ms, per = run(step)
        for k in cfg:
            del os.environ[k]
        if base is None:
            base = ms
        print(f"{ms:8.2f} ms ({(base / ms - 1) * 100:+5.1f}%) {cfg} {per}", flush=True)
        time.sleep(0.2)


if __name__ == "__main__":
    main()
