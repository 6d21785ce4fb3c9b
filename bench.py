"""LCE fwd+bwd benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (vocab-parallel, NCCL)
    python bench.py --gpus N ...   (N > 1 without torchrun: re-launches itself
                                    under torch.distributed.run with N ranks)
    python bench.py --sweep llama70b   (1/2/4/8-GPU strong-scaling sweep, t1 / (P tP))

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
import functools
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
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons, "samples": len(rows),
                "power_w": statistics.median(pw) if pw else None}


@functools.lru_cache(maxsize=2)
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


def cpu_info():
    """CPU model and the BLAS behind numpy (the oracle's dgemm)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info

        for i in threadpool_info():
            if i.get("user_api") == "blas":
                blas = f"{i.get('internal_api')} {i.get('version')} ({i.get('threading_layer', '')})".strip()
                break
    except Exception:
        pass
    return model, blas


def oracle_call(cfg_name: str, n: int):
    """One oracle fwd+bwd on n rows of the workload: (non-ignored rows, seconds)."""
    H, W, y = oracle_sample(cfg_name, n)
    t0 = time.perf_counter()
    nv = run_oracle_step(H, W, y)
    return nv, time.perf_counter() - t0


def oracle_rows_for(cfg_name: str, seconds: float) -> int:
    """Rows whose row-proportional oracle work (8 V D fp64 flops per valid row:
    z in the forward, z, G W and G^T H in the backward) takes ~`seconds` at
    this host's measured dgemm rate."""
    c = CONFIGS[cfg_name]
    a = np.random.default_rng(0).standard_normal((256, 4096))
    b = np.random.default_rng(1).standard_normal((4096, 4096))
    a @ b
    t0 = time.perf_counter()
    for _ in range(3):
        a @ b
    rate = 3 * 2 * 256 * 4096 * 4096 / (time.perf_counter() - t0)
    per_row = 8.0 * c["V"] * c["D"] / rate
    return int(max(32, min(c["N"] // 2, seconds / per_row)))


def marginal_rate(samples):
    """samples: [(n_rows, nv, seconds)] at two sizes.  The oracle's cost is
    a + b nv (a: per-call work independent of the row count, e.g. widening W
    to fp64 in both the forward and the backward); the per-token rate is the
    marginal 1 / b, so it does not depend on the sample size."""
    sizes = sorted({n for n, _, _ in samples})
    lo = [x for x in samples if x[0] == sizes[0]]
    hi = [x for x in samples if x[0] == sizes[-1]]
    nv1, t1 = statistics.mean(x[1] for x in lo), statistics.mean(x[2] for x in lo)
    nv2, t2 = statistics.mean(x[1] for x in hi), statistics.mean(x[2] for x in hi)
    return (nv2 - nv1) / max(t2 - t1, 1e-9), nv1, t1, nv2, t2


def time_oracle(cfg_name: str, target_s: float = 24.0):
    """Oracle fwd+bwd per-token rate on two bounded row samples (n, 2n)."""
    n = oracle_rows_for(cfg_name, target_s / 3)
    samples = [(m, *oracle_call(cfg_name, m)) for m in (n, 2 * n)]
    rate, nv1, t1, nv2, t2 = marginal_rate(samples)
    return rate, n, nv1, t1, nv2, t2


def cpu_record(rate, n, nv1, t1, nv2, t2, c, calls=2):
    model, blas = cpu_info()
    return {"value": rate, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": (f"{n} and {2 * n} of {c['N']} rows ({nv1:.0f} / {nv2:.0f} valid), full D={c['D']}, V={c['V']}: "
                       f"{calls} fp64 fwd+bwd calls, mean {t1:.1f} s / {t2:.1f} s per size; value = marginal per-token "
                       f"rate (nv2 - nv1) / (t2 - t1), independent of the oracle's per-call fixed cost"),
            "cpu_model": model, "blas": blas}


def reference_arm(args, rank):
    if rank != 0:
        return
    c = CONFIGS[args.config]
    # steps alternate bounded row samples of n and 2n rows, each ~3-6 s of fp64
    # work, so the whole run stays within a few minutes; value = marginal rate
    steps = max(2, args.steps)
    n = oracle_rows_for(args.config, min(6.0, max(1.0, 90.0 / steps)) / 2)
    for _ in range(min(args.warmup, 1)):
        oracle_call(args.config, n)
    samples = []
    for i in range(steps):
        m = n * (1 + i % 2)
        samples.append((m, *oracle_call(args.config, m)))
    v, nv1, t1, nv2, t2 = marginal_rate(samples)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": statistics.mean(x[2] for x in samples) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config), "N": c["N"], "D": c["D"], "V": c["V"]},
        "cpu_baseline": cpu_record(v, n, nv1, t1, nv2, t2, c, calls=steps),
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_name(cfg):
    c = CONFIGS[cfg]
    tag = {"llama1b": "Llama-3.2-1B head", "llama8b": "Llama-3.1-8B head", "qwen7b": "Qwen2.5-7B head packed",
           "llama70b": "Llama-3.1-70B head", "tiny": "tiny",
           "llama1b_1m": "Llama-3.2-1B head, 1M-token packed context (App. A)"}[cfg]
    return f"{tag}: N={c['N']} D={c['D']} V={c['V']}"


def self_launch(args) -> int:
    """--gpus N > 1 without a torch.distributed launcher: re-run this script
    under torch.distributed.run with N ranks (one process per GPU, rendezvous
    on 127.0.0.1) and NCCL's INIT log, so the run really has N ranks.  Fails
    loudly when the box has fewer than N GPUs."""
    import socket

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}"}), flush=True)
        sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {have} GPU(s) visible\n")
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def sweep(args) -> int:
    """Strong-scaling sweep of one workload over 1/2/4/8 GPUs (vocab-parallel,
    fixed N): one bench line per P, then efficiency t1 / (P tP).  P larger
    than the visible GPU count is reported as skipped, never faked."""
    have = torch.cuda.device_count()
    res = {}
    for P in (1, 2, 4, 8):
        if P > have:
            res[P] = {"skipped": f"{have} GPU(s) visible"}
            continue
        cmd = [sys.executable, os.path.abspath(__file__), "--gpus", str(P), "--config", args.config,
               "--steps", str(args.steps), "--warmup", str(args.warmup), "--no-cpu-baseline", "--no-e2e",
               "--no-split", "--path", args.path]
        outp = subprocess.run(cmd, capture_output=True, text=True).stdout.strip().splitlines()
        line = next((json.loads(x) for x in reversed(outp) if x.startswith("{")), None)
        res[P] = {"ms_per_step": line["ms_per_step"], "value": line["value"]} if line and "value" in line else \
            {"error": "no bench line"}
    t1 = res[1].get("ms_per_step")
    for P, r in res.items():
        if t1 and "ms_per_step" in r:
            r["efficiency"] = t1 / (P * r["ms_per_step"])
    print(json.dumps({"sweep": args.config, "path": args.path, "scaling": "strong", "per_gpus": res}), flush=True)
    return 0


def gemm_flops_of(nv_rank, vl, D, fused):
    f = {k: 2.0 * nv_rank * vl * D for k in ("fwd_gemm", "bwd_dh", "bwd_dw")}
    if not fused:
        f["bwd_g"] = 2.0 * nv_rank * vl * D  # the recompute GEMM (fused: an HBM-bound prep kernel)
    return f


def kernel_table(prof, steps, gemm_flops):
    kernels = {}
    for k, v in prof.items():
        if not v[1]:
            continue
        kernels[k] = {"ms_per_step": v[0] / steps, "launches_per_step": v[1] / steps}
        if v[2]:  # GEMM classes: SM clock inside the step (in-kernel clock64 / globaltimer probe)
            kernels[k]["sm_mhz"] = v[2]
            if k in gemm_flops:
                tf = gemm_flops[k] / (v[0] / steps / 1e3) / 1e12
                kernels[k]["tflops"] = tf
                # tensor-pipe utilisation at the clock the power cap allowed: achieved / (148 SMs x
                # 8192 dense bf16 flop/clk x that clock)
                kernels[k]["util_at_clock"] = tf * 1e12 / (SMS * 8192 * v[2] * 1e6)
    return kernels


def roofline_of(prof, steps, gemm_flops, config, fused, sus, src, step_ms_total):
    dom = max(prof, key=lambda k: prof[k][0])
    dom_ms, dom_n = prof[dom][:2]
    if dom not in gemm_flops or not dom_n:
        return None
    per_launch_flops = gemm_flops[dom] * steps / dom_n
    achieved = per_launch_flops / (dom_ms / dom_n / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(config + ("_fused" if fused else ""), {}).get(dom)
    mhz = prof[dom][2]
    return {"bound": "tensor", "achieved": achieved, "peak": sus, "unit": "TFLOP/s", "frac": achieved / sus,
            "sm_mhz": mhz, "util_at_clock": (achieved * 1e12 / (SMS * 8192 * mhz * 1e6)) if mhz else None,
            "traffic": traffic, "kernel": dom, "peak_source": f"{src} bf16_tflops_sustained (MEASURED_PEAKS.json)",
            "flops_per_launch": per_launch_flops,
            "share_of_step": (dom_ms / step_ms_total) if step_ms_total else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama8b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-split", action="store_true", help="skip the recompute-path sub-record")
    ap.add_argument("--sweep", metavar="CONFIG", default=None,
                    help="strong-scaling sweep of CONFIG over 1/2/4/8 GPUs (efficiency t1 / (P tP))")
    ap.add_argument("--chunk-budget", type=int, default=0,
                    help="chunk_budget_bytes (fused: bf16 q/G chunk bytes, default 2 GiB; split: G chunk)")
    ap.add_argument("--parallel", default="vocab", choices=["vocab", "token"],
                    help="N>1: vocab = W sharded by rows, identical batch on every rank (P:180 loss parallel, the "
                         "benchmarked mode); token = W replicated, the batch's rows split over ranks, N_v and the loss "
                         "exchanged by the library and dW all-reduced (the data-parallel gradient reduction)")
    ap.add_argument("--path", default="auto", choices=["auto", "fused", "split"],
                    help="fused = lce_forward_backward (no logit recompute, 6 N_v V D flops); split = "
                         "lce_forward + lce_backward (recompute from lse, 8 N_v V D flops); auto = fused, with "
                         "the split path as a sub-record")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, rank)
    if args.sweep:
        args.config = args.sweep
        return sweep(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU\n")
        return 2

    import paper_2605_21442_b200 as F
    from paper_2605_21442_b200.dist import max_over_ranks

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    comm = None
    # LCE_BENCH_FORCE_COMM=1 (tests): the multi-rank plumbing -- process group,
    # NCCL id broadcast, the library's communicator, max-over-ranks timing --
    # also at WORLD_SIZE=1, so it is exercised on a one-GPU box
    if world > 1 or os.environ.get("LCE_BENCH_FORCE_COMM") == "1":
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
    nv_rank = nv if not token else int((y != IGNORE).sum().item())  # rows this rank projects
    ws = F.Workspace()
    stream = torch.cuda.current_stream()
    out = {
        "loss": torch.empty(1, dtype=torch.float32, device=dev), "lse": torch.empty(N, dtype=torch.float32, device=dev),
        "n_valid": torch.empty(1, dtype=torch.int32, device=dev), "token_loss": None,
    }
    dH = torch.empty_like(H)
    dW = torch.empty(vl, D, dtype=torch.float32, device=dev)
    fused_head = args.path in ("fused", "auto")

    def run_path(Hx, Wx, yx, fused):
        if fused:  # lce_forward_backward: logits kept per row chunk, 6 N_v V D flops
            F.forward_backward(Hx, Wx, yx, dhidden=dH, dweight=dW, workspace=ws, out=out,
                               chunk_budget_bytes=args.chunk_budget, comm=comm, vocab_start=vstart, vocab_total=V)
        else:      # lce_forward + lce_backward: recompute from lse, 8 N_v V D flops
            F.forward(Hx, Wx, yx, comm=comm, vocab_start=vstart, vocab_total=V, workspace=ws, out=out,
                      chunk_budget_bytes=args.chunk_budget)
            F.backward(Hx, Wx, yx, out["lse"], comm=comm, vocab_start=vstart, vocab_total=V, dhidden=dH,
                       dweight=dW, workspace=ws, chunk_budget_bytes=args.chunk_budget)

    def step(fused):
        run_path(H, W, y, fused)
        if token:  # the data-parallel gradient reduction of the replicated head
            dist.all_reduce(dW)

    def timed(fused, steps, profile=False, clocks=False):
        """W warm-up steps, then `steps` steps bracketed by barrier + synchronize,
        one CUDA event pair per step on the launching stream.  Returns
        (total ms (max over ranks), per-step ms list, launches, profile, clocks)."""
        for _ in range(args.warmup):
            step(fused)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        clk = ClockSampler(local) if clocks else None
        if clk:
            clk.start()
        if profile:
            F.profile_enable(True)
        l0 = F.launch_count()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        torch.cuda.synchronize()
        ev[0].record(stream)
        for i in range(steps):
            step(fused)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
        launches = F.launch_count() - l0
        prof = None
        if profile:
            prof = F.profile_read()
            F.profile_enable(False)
        clk_rec = clk.stop() if clk else None
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
        total = ev[0].elapsed_time(ev[steps])
        if dist:  # the job's step time is the slowest rank's (device time, max over ranks)
            total = max_over_ranks(total, device=dev)
            per = [max_over_ranks(x, device=dev) for x in per]
            dist.barrier()
        return total, per, launches, prof, clk_rec

    torch.cuda.reset_peak_memory_stats(dev)
    # headline: profiler off; clocks sampled during the timed region
    ms, per, launches, _, clk = timed(fused_head, args.steps, clocks=True)
    peak_hbm = torch.cuda.max_memory_allocated(dev)
    ms_step = ms / args.steps
    value = nv * args.steps / (ms / 1e3)
    sus, burst, hbm, src = peaks()
    flops_step = (6.0 if fused_head else 8.0) * nv * V * D  # executed tensor-core flops per step
    tensor_frac = flops_step / (ms_step / 1e3) / (sus * 1e12 * world)
    # per-kernel profile in a separate pass (CUDA events around every launch)
    pms, _, _, prof, _ = timed(fused_head, args.steps, profile=True)
    gflops = gemm_flops_of(nv_rank, vl, D, fused_head)
    kernels = kernel_table(prof, args.steps, gflops)
    roof = roofline_of(prof, args.steps, gflops, args.config, fused_head, sus, src, pms if world == 1 else None)

    # the north star's recompute path (lce_forward + lce_backward) as a sub-record
    split = None
    if fused_head and not args.no_split:
        sms_total, sper, slaunch, _, sclk = timed(False, args.steps, clocks=True)
        spms, _, _, sprof, _ = timed(False, args.steps, profile=True)
        sg = gemm_flops_of(nv_rank, vl, D, False)
        s_step = sms_total / args.steps
        split = {"path": "lce_forward + lce_backward (backward recomputes the logit tiles from the saved lse)",
                 "value": nv * args.steps / (sms_total / 1e3), "unit": "tokens/s", "ms_per_step": s_step,
                 "ms_per_step_median": statistics.median(sper), "ms_per_step_min": min(sper),
                 "ms_per_step_max": max(sper), "flops_per_step": 8.0 * nv * V * D,
                 "tensor_frac": 8.0 * nv * V * D / (s_step / 1e3) / (sus * 1e12 * world),
                 "tensor_frac_note": f"8*N_v*V*D algorithmic flops (SURVEY 8d) / (time x {src} sustained bf16 peak x GPUs)",
                 "roofline": roofline_of(sprof, args.steps, sg, args.config, False, sus, src,
                                         spms if world == 1 else None),
                 "kernels": kernel_table(sprof, args.steps, sg), "gpu_launches_per_step": slaunch / args.steps,
                 "clocks": sclk}

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
                for dst, src_ in zip(bufs[k], (Hh, Wh, yh)):
                    dst.copy_(src_, non_blocking=True)
            loaded[k].record(cstream)

        def e2e_steps(n):
            issue_copy(0)
            for i in range(n):
                if i + 1 < n:
                    issue_copy(i + 1)
                k = i % 2
                stream.wait_event(loaded[k])
                run_path(*bufs[k], fused_head)
                if token:
                    dist.all_reduce(dW)
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
        cpu = cpu_record(*time_oracle(args.config), c)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_median": statistics.median(per),
            "ms_per_step_min": min(per), "ms_per_step_max": max(per), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_name(args.config), "N": c["N"], "N_valid": nv, "D": D, "V": V,
                       "parallelism": f"{args.parallel}-parallel x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (W alone is %.2f GB > 126 MB); no flush" % (V * D * 2 / 1e9)},
            "path": "fused lce_forward_backward" if fused_head else "lce_forward + lce_backward",
            "flops_per_step": flops_step,
            "tensor_frac": tensor_frac,
            "tensor_frac_note": f"{'6' if fused_head else '8'}*N_v*V*D executed flops per step / (time x {src} sustained bf16 peak x GPUs)",
            "peak_hbm_bytes": peak_hbm, "naive_logits_bytes_fp32": c["N"] * V * 4,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "clocks": clk, "kernels": kernels,
            "kernels_note": "per-kernel times from a separate profiled pass (CUDA events around every launch); "
                            "the headline step time is measured with the profiler off",
            "split": split,
        }
        print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
