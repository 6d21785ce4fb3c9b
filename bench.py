"""LCE fwd+bwd benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (vocab-parallel, NCCL)

A step is one pass of the whole hot path: lce_forward +
lce_backward on one synthetic batch already resident in HBM.  value =
non-ignored tokens per second of the whole job (all ranks cooperate on one
batch: vocab-parallel strong scaling).  The inputs (W is 1.05 GB at the 8B
head shape) are larger than the 126 MB L2, so no explicit flush is needed.
`--impl reference` times the fp64 CPU oracle (the only reference this tier
has) on a bounded row sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.inputs import CONFIGS, IGNORE, make_config  # noqa: E402

METRIC = "LCE fwd+bwd tokens/sec and % bf16 tensor peak at 1/2/4/8 B200; peak HBM bytes"
SMS = 148  # B200 SMs (dense bf16 tcgen05: 8192 flop/clk/SM)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops_sustained", 1383.0), d.get("bf16_tflops", 1638.5), d.get("hbm_gbs", 6545.3), "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.05)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        loaded = [x for x in sm if x > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons, "samples": len(rows)}


def oracle_sample(cfg_name: str, n_rows: int, seed: int = 0):
    """Rows of the same workload for the CPU oracle (exact bf16 values)."""
    from synth.inputs import make_inputs, make_labels

    c = CONFIGS[cfg_name]
    y = make_labels(c["N"], c["V"], c["labels"], c["ignore_frac"], 3000 + c["k"])
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(c["N"], size=min(n_rows, c["N"]), replace=False))
    inp = make_inputs(len(rows), c["D"], c["V"], k=c["k"], device="cpu", label_override=y[rows])
    return inp.hidden.float().numpy(), inp.weight.float().numpy(), inp.labels.numpy()


def run_oracle_step(H, W, y):
    from oracle import lce_backward, lce_forward

    f = lce_forward(H, W, y)
    lce_backward(H, W, y)
    return f["n_valid"]


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return len(os.sched_getaffinity(0))


def time_oracle(cfg_name: str, target_s: float = 12.0):
    """Oracle fwd+bwd on a bounded row sample; returns (tokens/s, rows, seconds)."""
    # calibrate on 128 rows (all oracle costs are linear in the row count), then
    # size the sample for ~target_s seconds of fp64 work
    H, W, y = oracle_sample(cfg_name, 128)
    t0 = time.perf_counter()
    run_oracle_step(H, W, y)
    t128 = time.perf_counter() - t0
    n = int(max(16, min(CONFIGS[cfg_name]["N"], 128 * target_s / max(t128, 1e-3))))
    H3, W3, y3 = oracle_sample(cfg_name, n)
    t0 = time.perf_counter()
    nv = run_oracle_step(H3, W3, y3)
    dt = time.perf_counter() - t0
    return nv / dt, n, nv, dt


def reference_arm(args, rank):
    if rank != 0:
        return
    c = CONFIGS[args.config]
    # each step is a bounded row sample sized so the whole run stays ~1-2 minutes
    target = min(8.0, max(1.0, 60.0 / max(1, args.steps + min(args.warmup, 1))))
    H, W, y = oracle_sample(args.config, 128)
    t0 = time.perf_counter()
    run_oracle_step(H, W, y)
    t128 = time.perf_counter() - t0
    n = int(max(16, min(c["N"], 128 * target / max(t128, 1e-3))))
    H, W, y = oracle_sample(args.config, n)
    for _ in range(min(args.warmup, 1)):
        run_oracle_step(H, W, y)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        nv = run_oracle_step(H, W, y)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = nv / t
    cores = cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config), "N": c["N"], "D": c["D"], "V": c["V"]},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n} of {c['N']} rows ({nv} valid), full D={c['D']}, V={c['V']}, fwd+bwd fp64 per step"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_name(cfg):
    c = CONFIGS[cfg]
    tag = {"llama1b": "Llama-3.2-1B head", "llama8b": "Llama-3.1-8B head", "qwen7b": "Qwen2.5-7B head packed",
           "llama70b": "Llama-3.1-70B head", "tiny": "tiny",
           "llama1b_1m": "Llama-3.2-1B head, 1M-token packed context (App. A)"}[cfg]
    return f"{tag}: N={c['N']} D={c['D']} V={c['V']}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama8b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--chunk-budget", type=int, default=0,
                    help="chunk_budget_bytes (fused: bf16 q/G chunk bytes, default 2 GiB; split: G chunk, 512 MiB)")
    ap.add_argument("--parallel", default="vocab", choices=["vocab", "token"],
                    help="N>1: vocab = W sharded by rows, identical batch on every rank (P:180 loss parallel, the "
                         "benchmarked mode); token = W replicated, the batch's rows split over ranks, N_v and the loss "
                         "exchanged by the library and dW all-reduced (the data-parallel gradient reduction)")
    ap.add_argument("--path", default="auto", choices=["auto", "fused", "split"],
                    help="fused = lce_forward_backward (no logit recompute, 6 N_v V D flops); split = "
                         "lce_forward + lce_backward (recompute from lse, 8 N_v V D flops); auto = fused")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, rank)

    import paper_2605_21442_b200 as F
    from paper_2605_21442_b200.dist import max_over_ranks

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        comm = F.Comm.from_process_group(mode=args.parallel)
    c = CONFIGS[args.config]
    inp = make_config(args.config, device=dev)
    N, D, V = c["N"], c["D"], c["V"]
    token = world > 1 and args.parallel == "token"
    vstart, vl = F.shard_range(V, world, rank) if world > 1 and not token else (0, V)
    W = inp.weight[vstart:vstart + vl].contiguous()
    del inp.weight
    H, y = inp.hidden, inp.labels
    nv = int((y != IGNORE).sum().item())  # non-ignored tokens of the whole (global) batch
    if token:  # this rank's rows of the global batch (contiguous, the last rank shorter)
        r0, nr = F.shard_range(N, world, rank)
        H, y = H[r0:r0 + nr].clone(), y[r0:r0 + nr].clone()
        N = nr
    ws = F.Workspace()
    stream = torch.cuda.current_stream()
    out = {
        "loss": torch.empty(1, dtype=torch.float32, device=dev), "lse": torch.empty(N, dtype=torch.float32, device=dev),
        "n_valid": torch.empty(1, dtype=torch.int32, device=dev), "token_loss": None,
    }
    dH = torch.empty_like(H)
    dW = torch.empty(vl, D, dtype=torch.float32, device=dev)

    fused = args.path in ("fused", "auto")

    def run_path(Hx, Wx, yx):
        if fused:  # lce_forward_backward: logits kept per row chunk, 6 N_v V D flops
            F.forward_backward(Hx, Wx, yx, dhidden=dH, dweight=dW, workspace=ws, out=out,
                               chunk_budget_bytes=args.chunk_budget, comm=comm, vocab_start=vstart, vocab_total=V)
        else:      # lce_forward + lce_backward: recompute from lse, 8 N_v V D flops
            F.forward(Hx, Wx, yx, comm=comm, vocab_start=vstart, vocab_total=V, workspace=ws, out=out,
                      chunk_budget_bytes=args.chunk_budget)
            F.backward(Hx, Wx, yx, out["lse"], comm=comm, vocab_start=vstart, vocab_total=V, dhidden=dH,
                       dweight=dW, workspace=ws, chunk_budget_bytes=args.chunk_budget)

    def step():
        run_path(H, W, y)
        if token:  # the data-parallel gradient reduction of the replicated head
            dist.all_reduce(dW)

    torch.cuda.reset_peak_memory_stats(dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    F.profile_enable(True)
    l0 = F.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = F.launch_count() - l0
    prof = F.profile_read()
    F.profile_enable(False)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if dist:  # the job's step time is the slowest rank's (device time, max over ranks)
        ms = max_over_ranks(ms, device=dev)
        dist.barrier()
    peak_hbm = torch.cuda.max_memory_allocated(dev)
    ms_step = ms / args.steps
    value = nv * args.steps / (ms / 1e3)
    sus, burst, hbm, src = peaks()
    flops_step = (6.0 if fused else 8.0) * nv * V * D  # executed tensor-core flops per step
    tensor_frac = flops_step / (ms_step / 1e3) / (sus * 1e12 * world)

    # dominant kernel (by device time inside the timed region, on the launching stream)
    nv_rank = nv if not token else int((y != IGNORE).sum().item())  # rows this rank projects
    gemm_flops = {k: 2.0 * nv_rank * vl * D for k in ("fwd_gemm", "bwd_dh", "bwd_dw")}
    if not fused:
        gemm_flops["bwd_g"] = 2.0 * nv_rank * vl * D  # the recompute GEMM (fused: an HBM-bound fix-up kernel)
    dom = max(prof, key=lambda k: prof[k][0])
    dom_ms, dom_n = prof[dom][:2]
    kernels = {}
    for k, v in prof.items():
        if not v[1]:
            continue
        kernels[k] = {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
        if v[2]:  # GEMM classes: SM clock inside the step (in-kernel clock64 / globaltimer probe)
            kernels[k]["sm_mhz"] = v[2]
            if k in gemm_flops:
                tf = gemm_flops[k] / (v[0] / args.steps / 1e3) / 1e12
                kernels[k]["tflops"] = tf
                # tensor-pipe utilisation at the clock the power cap allowed: achieved / (148 SMs x
                # 8192 dense bf16 flop/clk x that clock)
                kernels[k]["util_at_clock"] = tf * 1e12 / (SMS * 8192 * v[2] * 1e6)
    roof = None
    if dom in gemm_flops and dom_n:
        per_launch_flops = gemm_flops[dom] * args.steps / dom_n
        achieved = per_launch_flops / (dom_ms / dom_n / 1e3) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(args.config + ("_fused" if fused else ""), {}).get(dom)
        mhz = prof[dom][2]
        roof = {"bound": "tensor", "achieved": achieved, "peak": sus, "unit": "TFLOP/s", "frac": achieved / sus,
                "sm_mhz": mhz, "util_at_clock": (achieved * 1e12 / (SMS * 8192 * mhz * 1e6)) if mhz else None,
                "traffic": traffic, "kernel": dom, "peak_source": f"{src} bf16_tflops_sustained (MEASURED_PEAKS.json)",
                "flops_per_launch": per_launch_flops,
                "share_of_step": dom_ms / ms if world == 1 else None}

    # e2e through the public API with host buffers (pinned): every step copies
    # its H, W, y host->device and reads its loss back, inside the timed region.
    # The copies of step i+1 run on a copy stream into the other of two device
    # buffer sets while step i computes (double-buffered input pipeline).
    e2e = None
    if not args.no_e2e:
        Hh = H.cpu().pin_memory()
        Wh = W.cpu().pin_memory()
        yh = y.cpu().pin_memory()
        lossh = torch.empty(args.steps + 2, dtype=torch.float32).pin_memory()
        bufs = [(torch.empty_like(H), torch.empty_like(W), torch.empty_like(y)) for _ in range(2)]
        cstream = torch.cuda.Stream(device=dev)
        loaded = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def issue_copy(i):
            k = i % 2
            cstream.wait_event(consumed[k])  # the compute of step i-2 released this buffer set
            with torch.cuda.stream(cstream):
                for dst, src in zip(bufs[k], (Hh, Wh, yh)):
                    dst.copy_(src, non_blocking=True)
            loaded[k].record(cstream)

        def e2e_steps(n):
            issue_copy(0)
            for i in range(n):
                if i + 1 < n:
                    issue_copy(i + 1)
                k = i % 2
                stream.wait_event(loaded[k])
                run_path(*bufs[k])
                consumed[k].record(stream)
                lossh[i].copy_(out["loss"][0], non_blocking=True)

        e2e_steps(2)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cstream)
        stream.wait_stream(cstream)
        e2e_steps(args.steps)
        b.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b)
        if dist:
            ems = max_over_ranks(ems, device=dev)
        e2e = {"value": nv * args.steps / (ems / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": H.numel() * 2 + W.numel() * 2 + y.numel() * 4, "d2h_bytes_per_step": 4,
               "ms_per_step": ems / args.steps,
               "pipeline": "H2D of step i+1 on a copy stream overlaps step i (two device buffer sets)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v_cpu, n_rows, nv_rows, dt = time_oracle(args.config)
        cpu = {"value": v_cpu, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{n_rows} of {N} rows ({nv_rows} valid), full D={D}, V={V}, one fp64 fwd+bwd in {dt:.1f}s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_name(args.config), "N": c["N"], "N_valid": nv, "D": D, "V": V,
                       "parallelism": f"{args.parallel}-parallel x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (W alone is %.2f GB > 126 MB); no flush" % (V * D * 2 / 1e9)},
            "path": "fused lce_forward_backward" if fused else "lce_forward + lce_backward",
            "flops_per_step": flops_step,
            "tensor_frac": tensor_frac,
            "tensor_frac_note": f"{'6' if fused else '8'}*N_v*V*D executed flops per step / (time x {src} sustained bf16 peak x GPUs)",
            "peak_hbm_bytes": peak_hbm, "naive_logits_bytes_fp32": c["N"] * V * 4,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "clocks": clk, "kernels": kernels,
        }
        print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
