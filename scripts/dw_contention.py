"""(GPU) Is the dW epilogue's cost per-SM or chip-wide?  The fused 8B step through a
one-rank vocab communicator, with the dW GEMM given all SMs or only half of them
(LCE_VP_RESERVE_TEST=1 LCE_VP_RESERVE_SMS=74): if the drain is bound by chip-wide
L2 write contention, the per-SM rate of the half grid rises."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_21442_b200 as F  # noqa: E402
from synth.inputs import make_config  # noqa: E402

inp = make_config("llama8b", device="cuda")
H, W, y = inp.hidden, inp.weight, inp.labels
dH = torch.empty_like(H)
dW = torch.empty(W.shape, dtype=torch.float32, device="cuda")
ws = F.Workspace()
comm = F.Comm.single()
flops = 2.0 * 16384 * 128256 * 4096
for rep in range(3):
    for reserve, dbg in ((0, 0), (74, 0), (0, 1), (74, 1)):
        os.environ["LCE_VP_RESERVE_TEST"] = "1"
        os.environ["LCE_VP_RESERVE_SMS"] = str(reserve)
        os.environ["LCE_DBG_EPI"] = str(dbg)
        for _ in range(2):
            F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws, comm=comm)
        torch.cuda.synchronize()
        F.profile_read()
        F.profile_enable(True)
        for _ in range(6):
            F.forward_backward(H, W, y, dhidden=dH, dweight=dW, workspace=ws, comm=comm)
        torch.cuda.synchronize()
        p = F.profile_read()
        F.profile_enable(False)
        ms, n, mhz = p["bwd_dw"]
        sms = 148 - reserve
        per = ms / 6
        util = flops / (per / 1e3) / (sms * 8192 * mhz * 1e6)
        print(f"rep {rep} reserve {reserve:3d} dbg {dbg}: dW {per:.2f} ms/step on {sms} SMs @ {mhz:.0f} MHz, "
              f"util per active SM at clock {util:.3f}", flush=True)
comm.close()
