"""Per-rank workload of the P-GPU vocab-parallel run, timed on one GPU: the
fused path on rank r's W shard through a one-rank communicator (the exchanges
run, over one rank).  Used to pick tile shapes for the P > 1 GEMM extents.

    python scripts/bench_shard.py [--config llama8b] [--world 8] [--rank 2] [--steps 10]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import CONFIGS, IGNORE, make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    inp = make_config(a.config, device="cuda")
    v0, vl = F.shard_range(c["V"], a.world, a.rank)
    W = inp.weight[v0:v0 + vl].contiguous()
    del inp.weight
    H, y = inp.hidden, inp.labels
    nv = int((y != IGNORE).sum().item())
    dH = torch.empty_like(H)
    dW = torch.empty(vl, c["D"], dtype=torch.float32, device="cuda")
    ws = F.Workspace()
    comm = F.Comm.single()

    def step():
        F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws, comm=comm, vocab_start=v0,
                           vocab_total=c["V"])

    for _ in range(3):
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
    comm.close()
    ms = e0.elapsed_time(e1) / a.steps
    flops = 2.0 * nv * vl * c["D"]
    out = {"config": a.config, "world": a.world, "rank": a.rank, "V_l": vl, "ms_per_step": round(ms, 3),
           "tokens_per_s_per_rank_step": round(nv / (ms / 1e3))}
    for k, v in prof.items():
        if v[1]:
            d = {"ms": round(v[0] / a.steps, 3)}
            if v[2] and k in ("fwd_gemm", "bwd_dh", "bwd_dw"):
                d["util_at_clock"] = round(flops / (v[0] / a.steps / 1e3) / (148 * 8192 * v[2] * 1e6), 3)
                d["mhz"] = round(v[2])
            out[k] = d
    print(json.dumps(out))


if __name__ == "__main__":
    main()
