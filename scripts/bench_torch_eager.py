"""(GPU) Context, not the product: the paper-equivalent UNFUSED head in eager
PyTorch -- logits = F.linear(H, W) (bf16, cuBLAS), F.cross_entropy on the fp32
upcast, autograd backward -- on the same synthetic inputs, for time and peak
HBM next to liblce (SURVEY.md 8d "optional context").

    python scripts/bench_torch_eager.py [--configs llama1b llama8b] [--steps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn.functional as Fn  # noqa: E402

from synth.inputs import IGNORE, make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["llama1b", "llama8b"])
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    for name in a.configs:
        inp = make_config(name, device="cuda")
        H = inp.hidden.clone().requires_grad_(True)
        W = inp.weight.clone().requires_grad_(True)
        y = inp.labels.long()
        nv = int((y != IGNORE).sum())

        def step():
            H.grad = None
            W.grad = None
            loss = Fn.cross_entropy(Fn.linear(H, W).float(), y, ignore_index=IGNORE)
            loss.backward()
            return loss

        try:
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            print(json.dumps({"config": name, "impl": "eager torch F.linear + F.cross_entropy (fp32 upcast) + autograd",
                              "tokens_s": nv / (ms / 1e3), "ms_per_step": ms,
                              "peak_hbm_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
        except torch.OutOfMemoryError as e:
            print(json.dumps({"config": name, "oom": str(e)[:200]}), flush=True)
        del H, W, y, inp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
