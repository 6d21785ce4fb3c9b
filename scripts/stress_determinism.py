"""200 fused 8B steps on one workspace: the loss and the gradient checksums stay
bitwise identical (no state leaks between calls, no nondeterminism).

    python scripts/stress_determinism.py
"""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_21442_b200 as F
from synth.inputs import make_config
inp = make_config("llama8b", device="cuda")
H, W, y = inp.hidden, inp.weight, inp.labels
ws = F.Workspace()
dH = torch.empty_like(H); dW = torch.empty(W.shape, dtype=torch.float32, device="cuda")
ref = None
for i in range(200):
    out = F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws)
    if i == 0:
        ref = (out["loss"].item(), dH.float().sum().item(), dW.sum().item())
    elif i % 50 == 0 or i == 199:
        cur = (out["loss"].item(), dH.float().sum().item(), dW.sum().item())
        assert cur == ref, (i, cur, ref)
torch.cuda.synchronize()
print("stress ok", ref)
