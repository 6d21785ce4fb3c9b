"""Interleaved A/B sweep of LCE_* schedule knobs on one box.

    python scripts/sweep_env.py --config llama8b --path fused --reps 3 \
        '' 'LCE_GROUP_M_6=4' 'LCE_HINT_A_6=1 LCE_HINT_B_6=2'

Each argument is a space-separated list of VAR=VALUE (read by liblce.so at
every launch; '' is the default schedule).  Configurations are run round-robin
`--reps` times, `--steps` steps each; prints the median step time and the
median per-kernel-class device ms (library event profiler) per configuration.
"""

import argparse
import os
import statistics
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("configs", nargs="+")
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

    cfgs = [dict(kv.split("=", 1) for kv in c.split()) for c in a.configs]
    res = [[] for _ in cfgs]
    for _ in range(2):
        step()
    for rep in range(a.reps):
        for i, cfg in enumerate(cfgs):
            os.environ.update(cfg)
            step()
            torch.cuda.synchronize()
            F.profile_read()
            F.profile_enable(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            prof = F.profile_read()
            F.profile_enable(False)
            for k in cfg:
                del os.environ[k]
            res[i].append((e0.elapsed_time(e1) / a.steps, {k: v[0] / a.steps for k, v in prof.items() if v[1]},
                           {k: v[2] for k, v in prof.items() if v[1] and v[2]}))
    base = statistics.median(r[0] for r in res[0])
    for c, rs in zip(a.configs, res):
        ms = statistics.median(r[0] for r in rs)
        per = {k: round(statistics.median(r[1][k] for r in rs), 2) for k in rs[0][1]}
        mhz = {k: round(statistics.median(r[2][k] for r in rs)) for k in rs[0][2]}
        print(f"{ms:8.2f} ms ({(base / ms - 1) * 100:+5.1f}%) [{c or 'default'}] {per} MHz {mhz}", flush=True)


if __name__ == "__main__":
    main()
