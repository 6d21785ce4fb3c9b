"""Per-kernel-class device time of the linear KD loss (NEXT-4) at the 8B head
shape with a same-shape teacher head: which stage of the KD step costs what.

    python scripts/kd_profile.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import make_config, make_inputs  # noqa: E402


def main():
    inp = make_config("llama8b", device="cuda")
    H, W, y = inp.hidden, inp.weight, inp.labels
    t = make_inputs(H.shape[0], H.shape[1], W.shape[0], k=12, device="cuda", label_override=y.cpu().numpy())
    ws = F.Workspace()
    for _ in range(3):
        F.kd_forward_backward(H, W, t.hidden, t.weight, y, workspace=ws)
    torch.cuda.synchronize()
    F.profile_read()
    F.profile_enable(True)
    steps = 5
    for _ in range(steps):
        F.kd_forward_backward(H, W, t.hidden, t.weight, y, workspace=ws)
    torch.cuda.synchronize()
    prof = F.profile_read()
    F.profile_enable(False)
    print({k: (round(v[0] / steps, 2), v[1] // steps, round(v[2]) if v[2] else None)
           for k, v in prof.items() if v[1]})


if __name__ == "__main__":
    main()
