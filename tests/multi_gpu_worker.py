"""One rank of the multi-GPU parity run (tests/test_multi_gpu.py launches it
under torch.distributed.run, one process per GPU, NCCL).

Every rank drives liblce.so through its own NCCL communicator (the library's
collectives, not an oracle protocol), gathers the results with
torch.distributed, and rank 0 checks them against the fp64 CPU oracle:
  * vocab-parallel (P:180 loss parallel): split and fused paths, uneven
    shards; loss and lse bitwise identical on every rank, dH identical on
    every rank, dW shards concatenated in rank order;
  * the KD loss vocab-parallel;
  * token-parallel: rows split over ranks (one rank may hold none), the loss
    identical everywhere, dW shares summed over ranks;
  * a bad label on one rank only is reported by every rank (token mode).
Writes a JSON verdict to argv[1] (rank 0).
"""

import json
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LOSS_TOL, GRAD_TOL, LSE_TOL = 2e-3, 1e-2, 1e-3


def fro_rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a))


def gather(t):
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t.contiguous())
    return parts


def gather_var(t):
    """all_gather of tensors whose first dimension differs per rank."""
    n = torch.tensor([t.shape[0]], device=t.device)
    ns = gather(n)
    m = int(max(x.item() for x in ns))
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    return [p[:int(k.item())] for p, k in zip(gather(pad), ns)]


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2605_21442_b200 as F
    from oracle import kd_backward, kd_forward, lce_backward, lce_forward
    from synth.inputs import make_inputs

    checks = {}

    def ok(name, cond, info=None):
        checks[name] = {"ok": bool(cond), "info": info}

    cv = F.Comm.from_process_group(mode="vocab")
    ct = F.Comm.from_process_group(mode="token")
    try:
        for (N, D, V, seed) in [(600, 128, 1000, 1), (333, 72, 1003, 2)]:
            inp = make_inputs(N, D, V, k=seed, device=dev, ignore_frac=0.1)
            H, W, y = inp.hidden, inp.weight, inp.labels
            v0, vl = F.shard_range(V, world, rank)
            Wsh = W[v0:v0 + vl].contiguous()
            Hn, Wn, yn = H.float().cpu().numpy(), W.float().cpu().numpy(), y.cpu().numpy()
            o_f = lce_forward(Hn, Wn, yn)
            o_b = lce_backward(Hn, Wn, yn)
            for path, nvls in (("split", 0), ("fused", 0), ("split", 1), ("fused", 1)):
                tag = f"vocab_{path}{'_nvls' if nvls else ''}_N{N}_V{V}"
                os.environ["LCE_NVLS"] = str(nvls)  # 1: dH summed in the switch by the GEMM epilogue
                try:
                    if path == "split":
                        out = F.forward(H, Wsh, y, comm=cv, vocab_start=v0, vocab_total=V, with_token_loss=True)
                        dh, dw = F.backward(H, Wsh, y, out["lse"], comm=cv, vocab_start=v0, vocab_total=V)
                    else:
                        out = F.forward_backward(H, Wsh, y, comm=cv, vocab_start=v0, vocab_total=V,
                                                 with_token_loss=True, chunk_budget_bytes=256 * 2 * 512)
                        dh, dw = out["dhidden"], out["dweight"]
                except F.LceError as e:
                    if nvls and e.code == 7:  # no multicast support on this box: recorded, not failed
                        if rank == 0:
                            checks[tag + "_skipped"] = {"ok": True, "info": "multicast unsupported"}
                        continue
                    raise
                finally:
                    os.environ["LCE_NVLS"] = "0"
                torch.cuda.synchronize()
                losses = gather(out["loss"])
                lses = gather(out["lse"])
                dhs = gather(dh)
                dws = gather_var(dw)
                if rank == 0:
                    ok(tag + "_loss_bitwise_across_ranks", all(torch.equal(losses[0], x) for x in losses))
                    ok(tag + "_lse_bitwise_across_ranks", all(torch.equal(lses[0], x) for x in lses))
                    if not nvls:  # NVLS: in-switch order may differ per copy; checked against the oracle
                        ok(tag + "_dH_identical_across_ranks", all(torch.equal(dhs[0], x) for x in dhs))
                    L = losses[0].item()
                    ok(tag + "_loss", abs(L - o_f["loss"]) <= LOSS_TOL * abs(o_f["loss"]), (L, o_f["loss"]))
                    lerr = float(np.max(np.abs(lses[0].cpu().double().numpy() - o_f["lse"])
                                        / np.maximum(1, np.abs(o_f["lse"]))))
                    ok(tag + "_lse", lerr <= LSE_TOL, lerr)
                    e = fro_rel(dhs[0].float().cpu().double().numpy(), o_b["dH"])
                    ok(tag + "_dH", e <= GRAD_TOL, e)
                    dW_full = torch.cat(dws).cpu().double().numpy()
                    e = fro_rel(dW_full, o_b["dW"])
                    ok(tag + "_dW_concat", dW_full.shape == o_b["dW"].shape and e <= GRAD_TOL, e)

        # KD, vocab-parallel
        N, Ds, Dt, V = 400, 64, 128, 1000
        s = make_inputs(N, Ds, V, k=7, device=dev, ignore_frac=0.1)
        t = make_inputs(N, Dt, V, k=8, device=dev, ignore_frac=0.0, label_override=s.labels.cpu().numpy())
        v0, vl = F.shard_range(V, world, rank)
        kd = F.kd_forward_backward(s.hidden, s.weight[v0:v0 + vl].contiguous(), t.hidden,
                                   t.weight[v0:v0 + vl].contiguous(), s.labels, comm=cv, vocab_start=v0,
                                   vocab_total=V, chunk_budget_bytes=256 * 10 * 512)
        torch.cuda.synchronize()
        losses = gather(kd["loss"])
        dws = gather_var(kd["dweight"])
        if rank == 0:
            Hs, Ws, y = s.hidden.float().cpu().numpy(), s.weight.float().cpu().numpy(), s.labels.cpu().numpy()
            Ht, Wt = t.hidden.float().cpu().numpy(), t.weight.float().cpu().numpy()
            f = kd_forward(Hs, Ws, Ht, Wt, y)
            b = kd_backward(Hs, Ws, Ht, Wt, y)
            ok("kd_vocab_loss_bitwise_across_ranks", all(torch.equal(losses[0], x) for x in losses))
            ok("kd_vocab_loss", abs(losses[0].item() - f["loss"]) <= LOSS_TOL * abs(f["loss"]))
            ok("kd_vocab_dH", fro_rel(kd["dhidden"].float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL)
            ok("kd_vocab_dW_concat", fro_rel(torch.cat(dws).cpu().double().numpy(), b["dW"]) <= GRAD_TOL)

        # token-parallel: rows split unevenly, the last rank holds none
        N, D, V = 700, 128, 3000
        inp = make_inputs(N, D, V, k=9, device=dev, ignore_frac=0.3)
        bounds = np.linspace(0, N, world).astype(int).tolist() + [N]  # last rank: empty
        r0, r1 = bounds[rank], bounds[rank + 1]
        H, y = inp.hidden[r0:r1].contiguous(), inp.labels[r0:r1].contiguous()
        Hn, Wn, yn = inp.hidden.float().cpu().numpy(), inp.weight.float().cpu().numpy(), inp.labels.cpu().numpy()
        o_f = lce_forward(Hn, Wn, yn)
        o_b = lce_backward(Hn, Wn, yn)
        for path in ("split", "fused"):
            if path == "split":
                out = F.forward(H, inp.weight, y, comm=ct, with_token_loss=True)
                dh, dw = F.backward(H, inp.weight, y, out["lse"], comm=ct)
            else:
                out = F.forward_backward(H, inp.weight, y, comm=ct, with_token_loss=True)
                dh, dw = out["dhidden"], out["dweight"]
            dist.all_reduce(dw)  # the data-parallel gradient reduction the caller owns
            torch.cuda.synchronize()
            losses = gather(out["loss"])
            dhs = gather_var(dh)
            nvs = gather(out["n_valid"])
            if rank == 0:
                tag = f"token_{path}"
                ok(tag + "_loss_identical", all(torch.equal(losses[0], x) for x in losses))
                ok(tag + "_loss", abs(losses[0].item() - o_f["loss"]) <= LOSS_TOL * abs(o_f["loss"]))
                ok(tag + "_global_n_valid", all(int(x.item()) == o_f["n_valid"] for x in nvs))
                ok(tag + "_dH_rows", fro_rel(torch.cat(dhs).float().cpu().double().numpy(), o_b["dH"]) <= GRAD_TOL)
                ok(tag + "_dW_sum", fro_rel(dw.cpu().double().numpy(), o_b["dW"]) <= GRAD_TOL)

        # a bad label on one rank only (one that holds rows): every rank's loss is
        # NaN and every rank reports it, also the rank without rows
        yb = y.clone()
        if rank == (0 if world <= 2 else 1) and yb.numel():
            yb[0] = V + 5
        ws = F.Workspace()
        out = F.forward(H, inp.weight, yb, comm=ct, workspace=ws)
        torch.cuda.synchronize()
        try:
            F.check_device_status(ws)
            code = 0
        except F.LceError as e:
            code = e.code
        codes = gather(torch.tensor([code], device=dev))
        nan = gather(torch.tensor([1 if math.isnan(out["loss"].item()) else 0], device=dev))
        if rank == 0:
            ok("token_bad_label_reported_on_every_rank", all(int(c.item()) == 6 for c in codes),
               [int(c.item()) for c in codes])
            ok("token_bad_label_nan_loss_on_every_rank", all(int(x.item()) == 1 for x in nan))
        cv.check()
        ct.check()
    finally:
        cv.close()
        ct.close()
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump({"world": world, "checks": checks}, f, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
