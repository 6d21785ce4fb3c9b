"""KD step time and peak HBM against the chunk budget (8B student, same-shape teacher).

    python scripts/kd_budget.py
"""
import sys, os, torch, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_21442_b200 as F
from synth.inputs import make_config, make_inputs
inp = make_config("llama8b", device="cuda")
H, W, y = inp.hidden, inp.weight, inp.labels
t = make_inputs(H.shape[0], H.shape[1], W.shape[0], k=12, device="cuda", label_override=y.cpu().numpy())
for b in (0, 6 << 30, 8 << 30, 11 << 30, 0, 11 << 30):
    ws = F.Workspace()
    f = lambda: F.kd_forward_backward(H, W, t.hidden, t.weight, y, workspace=ws, chunk_budget_bytes=b)
    for _ in range(2): f()
    torch.cuda.synchronize(); torch.cuda.reset_peak_memory_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(b >> 30, round(ms, 2), round(16384 / ms * 1e3), round(torch.cuda.max_memory_allocated() / 1e9, 2))
    del ws; torch.cuda.empty_cache()
