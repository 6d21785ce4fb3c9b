import sys, os, json, torch
sys.path.insert(0, "/root/repo")
import paper_2605_21442_b200 as F
from synth.inputs import make_config, make_inputs
inp = make_config("llama8b", device="cuda")
H, W, y = inp.hidden, inp.weight, inp.labels
t = make_inputs(H.shape[0], H.shape[1], W.shape[0], k=12, device="cuda", label_override=y.cpu().numpy())
ws = F.Workspace()
for _ in range(3): F.kd_forward_backward(H, W, t.hidden, t.weight, y, workspace=ws)
torch.cuda.synchronize(); F.profile_read(); F.profile_enable(True)
for _ in range(5): F.kd_forward_backward(H, W, t.hidden, t.weight, y, workspace=ws)
torch.cuda.synchronize()
p = F.profile_read()
print({k: (round(v[0]/5, 2), v[1]//5, round(v[2]) if v[2] else None) for k, v in p.items() if v[1]})
