"""GPU parity: the CUDA path (through the C ABI) vs the fp64 CPU oracle.

Bars (BASELINE.json north_star):
  loss        |L_gpu - L_or| <= 2e-3 |L_or|
  dH, dW      ||X_gpu - X_or||_F <= 1e-2 ||X_or||_F
  lse         |lse_gpu - lse_or| <= 1e-3 max(1, |lse_or|)
  ignored rows: lse = token loss = dH row = 0 exactly.
The oracle always consumes the exact bf16 values the GPU consumed.
"""

import math
import sys
import os

import numpy as np
import pytest
import torch

from oracle import lce_backward, lce_dweight_rows, lce_forward, lce_lse, lce_rows
from synth.inputs import CONFIGS, IGNORE, LceInputs, make_config, make_inputs, packed_labels

pytestmark = pytest.mark.gpu

LOSS_TOL, GRAD_TOL, LSE_TOL = 2e-3, 1e-2, 1e-3


@pytest.fixture(params=["default", "pair", "wide", "single"])
def variant(request, monkeypatch):
    """Every tcgen05 mainloop: the shipped per-class mix (default: 256x256 CTA-pair
    tiles for the forward / recompute GEMMs, 512x256 wide pair tiles for dH / dW),
    CTA pairs everywhere, wide pair tiles everywhere, and the single-CTA kernel."""
    monkeypatch.delenv("LCE_WIDE", raising=False)
    if request.param == "default":
        monkeypatch.delenv("LCE_GEMM", raising=False)
    else:
        monkeypatch.setenv("LCE_GEMM", request.param)
    return request.param


def gpu_run(inp, reduction="mean", grad=None, budget=0, comm=None, accumulate_into=None):
    import paper_2605_21442_b200 as F

    out = F.forward(inp.hidden, inp.weight, inp.labels, ignore_index=inp.ignore_index, reduction=reduction,
                    with_token_loss=True, chunk_budget_bytes=budget, comm=comm)
    g = None if grad is None else torch.tensor([grad], dtype=torch.float32, device=inp.hidden.device)
    dw0 = None if accumulate_into is None else accumulate_into.clone()
    dh, dw = F.backward(inp.hidden, inp.weight, inp.labels, out["lse"], grad_loss=g, ignore_index=inp.ignore_index,
                        reduction=reduction, chunk_budget_bytes=budget, comm=comm, dweight=dw0,
                        accumulate_dweight=accumulate_into is not None)
    torch.cuda.synchronize()
    return {
        "loss": out["loss"].item(),
        "n_valid": int(out["n_valid"].item()),
        "lse": out["lse"].cpu().double().numpy(),
        "tok": out["token_loss"].cpu().double().numpy(),
        "dH": dh.float().cpu().double().numpy(),
        "dW": dw.cpu().double().numpy(),
    }


def np_inputs(inp):
    return (inp.hidden.float().cpu().numpy(), inp.weight.float().cpu().numpy(), inp.labels.cpu().numpy())


def oracle_run(inp, reduction="mean", grad=1.0):
    H, W, y = np_inputs(inp)
    f = lce_forward(H, W, y, ignore_index=inp.ignore_index, reduction=reduction)
    b = lce_backward(H, W, y, ignore_index=inp.ignore_index, reduction=reduction, grad_loss=grad)
    return {"loss": f["loss"], "n_valid": f["n_valid"], "lse": f["lse"], "tok": f["token_loss"], "dH": b["dH"],
            "dW": b["dW"]}


def fro_rel(a, b):
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def assert_parity(g, o, labels, ignore=IGNORE):
    assert g["n_valid"] == o["n_valid"]
    if o["loss"] == 0:
        assert g["loss"] == 0
    else:
        assert abs(g["loss"] - o["loss"]) <= LOSS_TOL * abs(o["loss"]), (g["loss"], o["loss"])
    lerr = np.abs(g["lse"] - o["lse"]) / np.maximum(1.0, np.abs(o["lse"]))
    assert lerr.max() <= LSE_TOL, lerr.max()
    terr = np.abs(g["tok"] - o["tok"]) / np.maximum(1.0, np.abs(o["lse"]))
    assert terr.max() <= LSE_TOL, terr.max()
    assert fro_rel(g["dH"], o["dH"]) <= GRAD_TOL, fro_rel(g["dH"], o["dH"])
    assert fro_rel(g["dW"], o["dW"]) <= GRAD_TOL, fro_rel(g["dW"], o["dW"])
    ign = labels == ignore
    assert np.all(g["lse"][ign] == 0) and np.all(g["tok"][ign] == 0)
    assert np.all(g["dH"][ign] == 0)


# ------------------------------------------------------------ the C ABI from plain C
def test_plain_c_client(cuda_lib, tmp_path):
    """tests/c_abi_check.c drives liblce.so through include/lce.h only (cudaMalloc
    buffers, no Python / torch) on the closed-form W = 0 case (P1)."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2605_21442_b200")
    exe = str(tmp_path / "c_abi_check")
    cuda = "/usr/local/cuda"
    subprocess.run(["gcc", "-O2", "-I", os.path.join(root, "include"), "-I", f"{cuda}/include",
                    os.path.join(root, "tests", "c_abi_check.c"), "-o", exe, "-L", pkg, "-llce",
                    f"-Wl,-rpath,{pkg}", "-L", f"{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{cuda}/lib64", "-lm"],
                   check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 2


# ------------------------------------------------------------ mainloop descriptors
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (296, 520, 200), (64, 40, 16), (136, 264, 72)])
def test_debug_gemm_matches_fp64(cuda_lib, variant, a_mn, b_mn, M, N, K):
    """The tcgen05 mainloop (smem/instruction descriptors, TMA swizzle, both
    operand majors, ragged M/N/K tails) computes A B^T."""
    import paper_2605_21442_b200 as F

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K + 10 * a_mn + b_mn)
    A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
    As = A.t().contiguous() if a_mn else A
    Bs = B.t().contiguous() if b_mn else B
    C = F.debug_gemm(As, Bs, M, N, K, bool(a_mn), bool(b_mn))
    torch.cuda.synchronize()
    ref = A.double().cpu() @ B.double().cpu().T
    err = (C.double().cpu() - ref).abs().max().item()
    assert err <= 1e-4 * math.sqrt(K) * max(1.0, ref.abs().max().item()), err


# ------------------------------------------------------------ tiny config (full oracle)
@pytest.mark.parametrize("reduction", ["mean", "sum"])
@pytest.mark.parametrize("regime", ["random", "confident"])
def test_tiny_config(cuda_lib, variant, reduction, regime):
    inp = make_config("tiny", device="cuda", regime=regime)
    g = gpu_run(inp, reduction)
    o = oracle_run(inp, reduction)
    assert_parity(g, o, inp.labels.cpu().numpy())


# ------------------------------------------------------------ exact (D, V) of every config, reduced N
@pytest.mark.parametrize("name", ["llama1b", "llama8b", "qwen7b", "llama70b"])
def test_config_shapes_reduced_n(cuda_lib, variant, name):
    """Each BASELINE config's exact (D, V) (incl. the vocab tail tile) with a
    ragged N spanning several 128-row tiles; 10% ignored rows (qwen: the packed
    label structure)."""
    c = CONFIGS[name]
    N = 300
    labels = None
    if c["labels"] == "packed":
        labels = packed_labels(2048, c["V"], seed=0)[:N]
    inp = make_inputs(N, c["D"], c["V"], k=c["k"], device="cuda", ignore_frac=0.1, label_override=labels,
                      regime="confident" if name == "llama8b" else "random")
    g = gpu_run(inp, "mean")
    o = oracle_run(inp, "mean")
    assert_parity(g, o, inp.labels.cpu().numpy())


# ------------------------------------------------------------ edge cases
def small(N, D, V, seed=0, ignore_frac=0.1, labels=None, regime="random"):
    return make_inputs(N, D, V, k=seed, device="cuda", ignore_frac=ignore_frac, label_override=labels, regime=regime)


@pytest.mark.parametrize("N,D,V", [(1, 64, 1000), (127, 64, 257), (129, 72, 256), (200, 8, 513), (260, 136, 2)])
def test_ragged_shapes(cuda_lib, variant, N, D, V):
    inp = small(N, D, V, seed=N)
    assert_parity(gpu_run(inp), oracle_run(inp), inp.labels.cpu().numpy())


def test_single_class_vocab(cuda_lib):
    """V = 1: softmax is 1, loss 0, every gradient 0."""
    inp = small(100, 64, 1, labels=np.zeros(100, dtype=np.int32))
    g = gpu_run(inp)
    assert g["n_valid"] == 100 and abs(g["loss"]) <= 1e-6
    assert np.abs(g["dH"]).max() <= 1e-6 and np.abs(g["dW"]).max() <= 1e-6


def test_empty_and_all_ignored(cuda_lib, variant):
    """N = 0 and N_v = 0: loss 0, lse 0, dH 0, dW 0."""
    inp = small(0, 64, 1000)
    g = gpu_run(inp)
    assert g["loss"] == 0 and g["n_valid"] == 0 and not g["dW"].any()
    lab = np.full(300, IGNORE, dtype=np.int32)
    inp = small(300, 64, 1000, labels=lab)
    for red in ("mean", "sum"):
        g = gpu_run(inp, red)
        assert g["loss"] == 0 and g["n_valid"] == 0
        assert not g["lse"].any() and not g["dH"].any() and not g["dW"].any()


def test_label_edges_and_ignore_inside_range(cuda_lib):
    """Labels at 0, V-1 and both sides of the 256-column tile boundaries; an
    ignore_index that is a legal vocab id (R3)."""
    V = 1000
    lab = np.array([0, V - 1, 255, 256, 511, 512, 767, 768, 5, 5] * 20, dtype=np.int32)
    inp = small(len(lab), 64, V, labels=lab)
    assert_parity(gpu_run(inp), oracle_run(inp), lab)
    inp.ignore_index = 5
    g = gpu_run(inp)
    o = oracle_run(inp)
    assert_parity(g, o, lab, ignore=5)


def test_bad_label_poisons_loss_and_sets_status(cuda_lib):
    """R4: a label outside [0, V) excludes its row, makes the loss NaN and is
    reported by lce_check_device_status."""
    import paper_2605_21442_b200 as F

    lab = np.arange(200, dtype=np.int32) % 1000
    lab[17] = 1000
    inp = small(200, 64, 1000, labels=lab)
    out = F.forward(inp.hidden, inp.weight, inp.labels, with_token_loss=True)
    torch.cuda.synchronize()
    assert math.isnan(out["loss"].item())
    assert out["n_valid"].item() == 199
    assert out["lse"][17].item() == 0
    with pytest.raises(F.LceError) as e:
        F.check_device_status(device=inp.hidden.device)
    assert e.value.code == 6
    lab[17] = 3
    ok = small(200, 64, 1000, labels=lab)
    F.forward(ok.hidden, ok.weight, ok.labels)
    F.check_device_status(device=inp.hidden.device)  # status reflects the latest call


def test_grad_scale_sum_and_accumulate(cuda_lib):
    """R11: upstream gradient scales dH/dW; accumulate_dweight adds into dW."""
    inp = small(300, 64, 1000, seed=3)
    o = oracle_run(inp, "sum", grad=-2.5)
    g = gpu_run(inp, "sum", grad=-2.5)
    assert_parity(g, o, inp.labels.cpu().numpy())
    base = torch.randn(1000, 64, device="cuda")
    ga = gpu_run(inp, "sum", grad=-2.5, accumulate_into=base)
    assert fro_rel(ga["dW"] - base.cpu().double().numpy(), o["dW"]) <= GRAD_TOL


def test_chunk_budget_is_not_semantics(cuda_lib, variant):
    """R7: several vocab chunks (tiny budget) give the same result as one."""
    inp = small(384, 128, 3000, seed=4)
    one = gpu_run(inp)
    many = gpu_run(inp, budget=384 * 2 * 256)  # one 256-column tile per chunk
    o = oracle_run(inp)
    assert_parity(many, o, inp.labels.cpu().numpy())
    assert many["loss"] == one["loss"]
    np.testing.assert_array_equal(many["lse"], one["lse"])
    np.testing.assert_array_equal(many["dW"], one["dW"])
    assert fro_rel(many["dH"], one["dH"]) <= 1e-2


def test_garbage_in_ignored_rows_is_bitwise_invisible(cuda_lib):
    """P3 mask-first: NaN/Inf in ignored rows of H never reaches the
    projection: every output is bitwise unchanged and their dH rows are 0."""
    inp = small(300, 128, 1000, seed=5, ignore_frac=0.3)
    g0 = gpu_run(inp)
    ign = inp.labels == IGNORE
    h = inp.hidden.clone()
    h[ign] = float("nan")
    h[torch.nonzero(ign)[0, 0]] = float("inf")
    inp.hidden = h
    g1 = gpu_run(inp)
    for k in ("lse", "tok", "dH", "dW"):
        np.testing.assert_array_equal(g0[k], g1[k])
    assert g0["loss"] == g1["loss"]


def test_deterministic_rerun(cuda_lib):
    """H8: fixed-order reductions and single-writer tiles -> bitwise reruns."""
    inp = small(500, 256, 5000, seed=6)
    a, b = gpu_run(inp), gpu_run(inp)
    for k in ("lse", "tok", "dH", "dW"):
        np.testing.assert_array_equal(a[k], b[k])
    assert a["loss"] == b["loss"]


def test_default_workspaces_are_per_stream(cuda_lib):
    """Calls without an explicit workspace on two streams at once get separate
    default scratch (a shared buffer would race): both results equal the
    serial ones bitwise."""
    import paper_2605_21442_b200 as F

    a = small(3000, 256, 2000, seed=41)
    b = small(2000, 256, 3000, seed=42)
    ref_a = F.forward_backward(a.hidden, a.weight, a.labels)
    ref_b = F.forward_backward(b.hidden, b.weight, b.labels)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        got_a = F.forward_backward(a.hidden, a.weight, a.labels)
    with torch.cuda.stream(s2):
        got_b = F.forward_backward(b.hidden, b.weight, b.labels)
    torch.cuda.synchronize()
    for ref, got in ((ref_a, got_a), (ref_b, got_b)):
        for k in ("loss", "lse", "dhidden", "dweight"):
            assert torch.equal(ref[k], got[k]), k
    F.check_device_status()


@pytest.mark.parametrize("lock", ["0", "1"])
@pytest.mark.parametrize("path", ["fused", "split"])
def test_k_lockstep_is_timing_only(cuda_lib, monkeypatch, lock, path):
    """The K-lockstep of the persistent grids (LCE_LOCK; on by default for wide
    tiles) only delays TMA producers: forcing it on every GEMM (pair tiles too,
    a tight drift bound) or off leaves every output bitwise equal to the
    default schedule (whose parity the other tests check)."""
    inp = small(16384, 256, 5000, seed=34, ignore_frac=0.1)
    run = fused_run if path == "fused" else (lambda i: gpu_run(i))
    monkeypatch.delenv("LCE_LOCK", raising=False)
    ref = run(inp)
    monkeypatch.setenv("LCE_LOCK", lock)
    monkeypatch.setenv("LCE_LOCK_D", "2")
    got = run(inp)
    for k in ("lse", "tok", "dH", "dW"):
        np.testing.assert_array_equal(ref[k], got[k])
    assert ref["loss"] == got["loss"]


@pytest.mark.parametrize("gemm", ["default", "pair"])
def test_fused_deterministic_and_mask_first(cuda_lib, monkeypatch, gemm):
    """H8 and P3 for the fused path at a shape that takes its wide dH / dW tiles
    (8,192-row chunks), split-K dH and the TMA reduce-add of the second chunk's
    dW: two runs are bitwise identical, and NaN / Inf in ignored rows of H leave
    every output bitwise unchanged (their dH rows exactly 0)."""
    if gemm == "default":
        monkeypatch.delenv("LCE_GEMM", raising=False)
    else:
        monkeypatch.setenv("LCE_GEMM", gemm)
    inp = small(16384, 256, 5000, seed=33, ignore_frac=0.2)
    a, b = fused_run(inp), fused_run(inp)
    for k in ("lse", "tok", "dH", "dW"):
        np.testing.assert_array_equal(a[k], b[k])
    assert a["loss"] == b["loss"]
    ign = inp.labels == IGNORE
    h = inp.hidden.clone()
    h[ign] = float("nan")
    h[torch.nonzero(ign)[0, 0]] = float("inf")
    c = fused_run(LceInputs(hidden=h, weight=inp.weight, labels=inp.labels))
    for k in ("lse", "tok", "dH", "dW"):
        np.testing.assert_array_equal(a[k], c[k])
    assert a["loss"] == c["loss"] and np.all(c["dH"][ign.cpu().numpy()] == 0)


def test_single_rank_communicator_path(cuda_lib):
    """The vocab-parallel exchange (MAX / SUM all-reduce + finalize) on a
    one-rank NCCL communicator matches the oracle."""
    import paper_2605_21442_b200 as F

    comm = F.Comm.single()
    try:
        inp = small(300, 64, 1000, seed=7)
        g = gpu_run(inp, comm=comm)
        assert_parity(g, oracle_run(inp), inp.labels.cpu().numpy())
    finally:
        comm.close()


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("path", ["split", "fused"])
def test_nvls_in_switch_dh_reduction_single_rank(cuda_lib, monkeypatch, path, mode):
    """LCE_NVLS (SURVEY 8e upgrade): the dH GEMM's epilogue adds its
    partials (split-K items included) into a shared fp32 buffer, an NVLS
    barrier kernel closes the chunk, the cast / scatter reads the local copy --
    against the oracle over several row / vocab chunks, twice (the buffer
    persists on the communicator).
    mode 1: a real multicast object (cuMulticastCreate / AddDevice / BindMem,
    multimem.red.add.v4.f32); skips where the driver refuses multicast objects
    (LCE_ERR_DEVICE -- the one-GPU gpurun containers do, profiles/
    round2_multicast_probe.log).  mode 2: the same sequence on a unicast
    buffer with plain red.global.add (one rank), which runs everywhere."""
    import paper_2605_21442_b200 as F

    monkeypatch.setenv("LCE_NVLS", mode)
    inp = small(900, 256, 5000, seed=26)
    lab = inp.labels.cpu().numpy()
    comm = F.Comm.single()
    try:
        for _ in range(2):
            try:
                if path == "split":
                    g = gpu_run(inp, comm=comm, budget=900 * 2 * 1024)
                else:
                    g = fused_run(inp, comm=comm, budget=256 * 2 * 5120)
            except F.LceError as e:
                if mode == "1" and e.code == 7:
                    pytest.skip("the driver refuses multicast objects on this box (LCE_ERR_DEVICE)")
                raise
            assert_parity(g, oracle_run(inp), lab)
    finally:
        comm.close()


@pytest.mark.parametrize("sms", ["132", "100", "38"])
def test_fewer_sms_than_the_plan_assumes(cuda_lib, monkeypatch, sms):
    """The workspace plan is host-pure and sized for a full B200 (148 SMs); on a
    part with fewer SMs (LCE_SMS emulates one) every grid shrinks and the fused
    path re-derives its dH split-K factor for the SM count, capped by the slab
    space the plan reserved -- results stay within the bars."""
    monkeypatch.setenv("LCE_SMS", sms)
    inp = small(1100, 256, 6000, seed=28, ignore_frac=0.2)
    o = oracle_run(inp)
    lab = inp.labels.cpu().numpy()
    assert_parity(fused_run(inp, budget=256 * 2 * 6144), o, lab)
    assert_parity(gpu_run(inp, budget=1280 * 2 * 2048), o, lab)


def test_nvls_emulation_kd_and_adamw_single_rank(cuda_lib, monkeypatch):
    """The NVLS dH sequence (LCE_NVLS=2, one-rank unicast emulation) on the
    remaining entry points that reduce dH over ranks: the KD loss (fused chunk
    path) and AdamW-in-backward (recompute path), against the oracle / the
    NCCL path."""
    import paper_2605_21442_b200 as F
    from oracle import adamw_step, kd_backward, kd_forward

    s, t = _kd_inputs(400, 128, 64, 3000, seed=27)
    comm = F.Comm.single()
    try:
        monkeypatch.setenv("LCE_NVLS", "2")
        out = F.kd_forward_backward(s.hidden, s.weight, t.hidden, t.weight, s.labels, comm=comm,
                                    chunk_budget_bytes=256 * 10 * 1024)
        theta, m, v = _adam_state(3000, 128, 7)
        w = theta.to(torch.bfloat16).cuda()
        th_d, m_d, v_d = theta.cuda(), m.cuda(), v.cuda()
        fo = F.forward(s.hidden, w, s.labels, comm=comm)
        dh_a = F.backward_adamw(s.hidden, w, s.labels, fo["lse"], th_d, m_d, v_d, lr=1e-3, step=3, comm=comm,
                                chunk_budget_bytes=400 * 2 * 1024)
        torch.cuda.synchronize()
    finally:
        comm.close()
    Hs, Ws, y = np_inputs(s)
    Ht, Wt = t.hidden.float().cpu().numpy(), t.weight.float().cpu().numpy()
    f = kd_forward(Hs, Ws, Ht, Wt, y)
    b = kd_backward(Hs, Ws, Ht, Wt, y)
    assert abs(out["loss"].item() - f["loss"]) <= LOSS_TOL * abs(f["loss"])
    assert fro_rel(out["dhidden"].float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL
    assert fro_rel(out["dweight"].cpu().double().numpy(), b["dW"]) <= GRAD_TOL
    Wb = theta.to(torch.bfloat16).float().numpy()
    o = lce_backward(Hs, Wb, y)
    assert fro_rel(dh_a.float().cpu().double().numpy(), o["dH"]) <= GRAD_TOL
    th_o, _, _ = adamw_step(theta.double().numpy(), o["dW"], m.double().numpy(), v.double().numpy(), 3, lr=1e-3)
    dth = th_d.cpu().double().numpy() - theta.double().numpy()
    assert fro_rel(dth, th_o - theta.double().numpy()) <= GRAD_TOL


@pytest.mark.parametrize("reserve", [16, 38])
def test_communicator_with_reserved_sms(cuda_lib, monkeypatch, reserve):
    """Under vocab parallelism the dW GEMM that overlaps the dH all-reduce runs
    on a reduced persistent grid (SMs left to the collective): the result is
    unchanged, for the recompute and fused paths, pair and wide tiles."""
    import paper_2605_21442_b200 as F

    monkeypatch.setenv("LCE_VP_RESERVE_TEST", "1")
    monkeypatch.setenv("LCE_VP_RESERVE_SMS", str(reserve))
    comm = F.Comm.single()
    try:
        for gemm in ("pair", "wide"):
            monkeypatch.setenv("LCE_GEMM", gemm)
            inp = small(1100, 136, 3000, seed=9, ignore_frac=0.2)
            o = oracle_run(inp)
            lab = inp.labels.cpu().numpy()
            assert_parity(gpu_run(inp, comm=comm), o, lab)
            assert_parity(fused_run(inp, comm=comm, budget=256 * 2 * 3072), o, lab)
    finally:
        comm.close()


def test_token_parallel_communicator_one_rank(cuda_lib):
    """LCE_PAR_TOKEN on one rank is the single-GPU problem: forward / backward,
    fused and KD match the oracle through the token-parallel code path (the
    N_v and loss exchanges); the in-backward AdamW refuses it (needs the full
    dW); a rank with no tokens still completes its exchanges."""
    import paper_2605_21442_b200 as F
    comm = F.Comm.single("token")
    try:
        assert F.lib.lce_comm_mode(comm.handle) == 1
        inp = small(700, 136, 3000, seed=21, ignore_frac=0.3)
        lab = inp.labels.cpu().numpy()
        for red in ("mean", "sum"):
            o = oracle_run(inp, red)
            assert_parity(gpu_run(inp, red, comm=comm), o, lab)
            assert_parity(fused_run(inp, red, comm=comm, budget=256 * 2 * 3072), o, lab)
        t = make_inputs(700, 72, 3000, k=22, device="cuda", label_override=lab)
        kd = F.kd_forward_backward(inp.hidden, inp.weight, t.hidden, t.weight, inp.labels, comm=comm)
        kd0 = F.kd_forward_backward(inp.hidden, inp.weight, t.hidden, t.weight, inp.labels)
        assert abs(kd["loss"].item() - kd0["loss"].item()) <= 1e-6 * abs(kd0["loss"].item())
        assert torch.equal(kd["dhidden"], kd0["dhidden"])
        theta = inp.weight.float().clone()
        with pytest.raises(F.LceError):
            F.backward_adamw(inp.hidden, inp.weight.clone(), inp.labels, torch.zeros(700, device="cuda"), theta,
                             torch.zeros_like(theta), torch.zeros_like(theta), lr=1e-3, step=1, comm=comm)
        e = small(0, 64, 1000, seed=23)
        out = F.forward_backward(e.hidden, e.weight, e.labels, comm=comm)
        torch.cuda.synchronize()
        assert out["loss"].item() == 0.0 and int(out["n_valid"].item()) == 0
        assert torch.count_nonzero(out["dweight"]).item() == 0
    finally:
        comm.close()


def test_token_parallel_bad_label_status_and_comm_check(cuda_lib):
    """Token parallelism: the bad-label flag is all-reduced and raised into the
    status word of every rank (tp_scale_kernel), so every rank's
    check_device_status reports LCE_ERR_LABEL_RANGE and every loss is NaN
    (one rank here; tests/test_multi_gpu.py covers two).  lce_comm_check polls
    NCCL's asynchronous error state (clean here)."""
    import paper_2605_21442_b200 as F

    comm = F.Comm.single("token")
    try:
        inp = small(300, 64, 1000, seed=25)
        y = inp.labels.clone()
        y[7] = 5000
        for fused in (False, True):
            ws = F.Workspace()
            if fused:
                out = F.forward_backward(inp.hidden, inp.weight, y, comm=comm, workspace=ws)
            else:
                out = F.forward(inp.hidden, inp.weight, y, comm=comm, workspace=ws)
            torch.cuda.synchronize()
            assert math.isnan(out["loss"].item())
            with pytest.raises(F.LceError) as e:
                F.check_device_status(ws)
            assert e.value.code == 6
        comm.check()
    finally:
        comm.close()


@pytest.mark.parametrize("path", ["split", "fused"])
def test_token_parallel_decomposition(cuda_lib, path):
    """What each token-parallel rank computes, checked on one GPU through the
    public API: rows split unevenly into shards, each shard with reduction SUM
    and upstream gradient 1 / N_v(global) (the scale LCE_PAR_TOKEN applies to
    MEAN) -- the shard losses and dW shares sum to, and the dH rows
    concatenate to, the full batch's MEAN result."""
    inp = small(1100, 136, 3000, seed=24, ignore_frac=0.25)
    lab = inp.labels.cpu().numpy()
    o = oracle_run(inp, "mean")
    nv = int((lab != IGNORE).sum())
    cuts = [0, 0, 313, 1100]  # the first shard holds no tokens
    loss, dW, dH, tok = 0.0, 0.0, [], []
    for a, b in zip(cuts, cuts[1:]):
        part = LceInputs(hidden=inp.hidden[a:b].clone(), weight=inp.weight, labels=inp.labels[a:b].clone())
        g = gpu_run(part, "sum", grad=1.0 / nv) if path == "split" else fused_run(part, "sum", grad=1.0 / nv)
        loss += g["loss"] / nv
        dW = dW + g["dW"]
        dH.append(g["dH"])
        tok.append(g["tok"])
    assert abs(loss - o["loss"]) <= LOSS_TOL * abs(o["loss"])
    assert fro_rel(np.concatenate(dH), o["dH"]) <= GRAD_TOL
    assert fro_rel(dW, o["dW"]) <= GRAD_TOL
    assert np.abs(np.concatenate(tok) - o["tok"]).max() <= LSE_TOL * max(1.0, np.abs(o["lse"]).max())


@pytest.mark.parametrize("reduction", ["mean", "none"])
def test_fused_scaled_q_fallback_rows(cuda_lib, reduction):
    """R25: the fused path keeps q relative to each row's target logit; a chunk
    with a row whose logits exceed it by more than e^64 (a target logit ~100
    below the row's lse) redoes its forward in the tile-max form on the GPU.
    Both chunks -- one with such rows, one without -- match the oracle, and so
    do the unscaled fix-up form and a confident (p_target ~ 1) batch."""
    N, D, V = 700, 128, 3000
    inp = small(N, D, V, seed=31, ignore_frac=0.1)
    lab = inp.labels.cpu().numpy()
    # rows 5..20 (first chunk): push the target logit ~100 below the others
    y = inp.labels.long().clamp(min=0)
    Wy = inp.weight[y].float()
    bump = -100.0 * Wy / (Wy * Wy).sum(dim=1, keepdim=True)
    rows = torch.zeros(N, dtype=torch.bool, device="cuda")
    rows[5:21] = True
    rows &= inp.labels != IGNORE
    h = torch.where(rows[:, None], inp.hidden.float() + bump, inp.hidden.float()).to(torch.bfloat16)
    spiky = LceInputs(hidden=h.contiguous(), weight=inp.weight, labels=inp.labels)
    g = None if reduction == "mean" else np.linspace(-1.0, 2.0, N)
    budget = 256 * 2 * 3072  # 512-row chunks: rows 0..511 flagged, the rest not
    for case in (spiky, small(N, D, V, seed=32, regime="confident")):
        o = oracle_run(case, reduction, grad=1.0 if g is None else g)
        assert o["loss"] > 0
        assert_parity(fused_run(case, reduction, grad=g, budget=budget), o, case.labels.cpu().numpy())
    os.environ["LCE_FUSED_SCALED"] = "0"
    try:
        o = oracle_run(spiky, reduction, grad=1.0 if g is None else g)
        assert_parity(fused_run(spiky, reduction, grad=g, budget=budget), o, lab)
    finally:
        del os.environ["LCE_FUSED_SCALED"]
    # the fallback really ran for the spiky batch (and only there): its
    # tile-max re-forward shows up as GEMM work in the G-formation class
    import paper_2605_21442_b200 as F

    import ctypes

    def g_gemm_cycles(case):
        """SM cycles the G-formation class's GEMM launches (the re-forwards) spent."""
        fused_run(case, reduction, grad=g, budget=budget)
        F.profile_read()
        F.profile_enable(True)
        fused_run(case, reduction, grad=g, budget=budget)
        k = 9  # LCE_K_COUNT
        ms, n = (ctypes.c_double * k)(), (ctypes.c_int64 * k)()
        cyc, ns = (ctypes.c_double * k)(), (ctypes.c_double * k)()
        assert F.lib.lce_profile_read_clocks(ms, n, cyc, ns) == 0
        F.profile_enable(False)
        return cyc[4], n[4]  # LCE_K_BWD_G
    calm = small(N, D, V, seed=31, ignore_frac=0.1)
    cyc_spiky, n_spiky = g_gemm_cycles(spiky)
    cyc_calm, n_calm = g_gemm_cycles(calm)
    assert n_spiky == n_calm  # the same launches: the redo is empty unless a row flagged its chunk
    assert cyc_spiky > 3 * cyc_calm, (cyc_spiky, cyc_calm)


def test_fused_scaled_q_vocab_shard_fallback(cuda_lib):
    """R25 under a one-rank vocab-parallel communicator over a shard: the
    per-row references are exchanged (rows whose label lies outside the shard
    get 0), rows with a target ~100 nats below the shard's logits flag their
    chunk, and the result is still the oracle's shard statistics / gradients."""
    import paper_2605_21442_b200 as F
    from oracle import shard_backward, shard_stats

    N, D, V, v0, vl = 700, 128, 3000, 1000, 1500
    inp = small(N, D, V, seed=34, ignore_frac=0.1)
    y = inp.labels.long().clamp(min=0)
    Wy = inp.weight[y].float()
    own = (inp.labels >= v0) & (inp.labels < v0 + vl)
    rows = torch.zeros(N, dtype=torch.bool, device="cuda")
    rows[:40] = True
    rows &= own
    h = torch.where(rows[:, None], inp.hidden.float() - 100.0 * Wy / (Wy * Wy).sum(1, keepdim=True),
                    inp.hidden.float()).to(torch.bfloat16).contiguous()
    Wsh = inp.weight[v0:v0 + vl].contiguous()
    comm = F.Comm.single()
    try:
        out = F.forward_backward(h, Wsh, inp.labels, comm=comm, vocab_start=v0, vocab_total=V, with_token_loss=True,
                                 chunk_budget_bytes=256 * 2 * 1536)
        torch.cuda.synchronize()
    finally:
        comm.close()
    H = h.float().cpu().numpy()
    Wn = Wsh.float().cpu().numpy()
    lab = inp.labels.cpu().numpy()
    st = shard_stats(H, Wn, lab, v0, V)
    valid = st["valid"]
    lse_sh = np.where(valid, st["m"] + np.log(np.where(valid, st["s"], 1.0)), 0.0)
    assert np.abs(out["lse"].cpu().double().numpy() - lse_sh).max() <= LSE_TOL * max(1, np.abs(lse_sh).max())
    sb = shard_backward(H, Wn, lab, v0, lse_sh, 1.0 / int(valid.sum()))
    assert fro_rel(out["dhidden"].float().cpu().double().numpy(), sb["dH_partial"]) <= GRAD_TOL
    assert fro_rel(out["dweight"].cpu().double().numpy(), sb["dW_shard"]) <= GRAD_TOL


def test_autograd_function(cuda_lib):
    import paper_2605_21442_b200 as F

    inp = small(200, 64, 1000, seed=8)
    h = inp.hidden.clone().requires_grad_(True)
    w = inp.weight.clone().requires_grad_(True)
    loss = F.linear_cross_entropy(h, w, inp.labels)
    loss.backward()
    o = oracle_run(inp)
    assert abs(loss.item() - o["loss"]) <= LOSS_TOL * abs(o["loss"])
    assert fro_rel(h.grad.float().cpu().double().numpy(), o["dH"]) <= GRAD_TOL
    assert fro_rel(w.grad.float().cpu().double().numpy(), o["dW"]) <= 2e-2  # dW rounded to bf16 for autograd


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
def test_drop_in_batched_int64_labels(cuda_lib, fused, reduction):
    """P:132 drop-in: hidden [B, S, D], labels [B, S] int64 (torch's class-index
    dtype), gradients through autograd into the [B, S, D] leaf; 'none' returns
    [B, S]; an int64 label outside the int32 range is flagged, not wrapped."""
    import paper_2605_21442_b200 as F

    if fused and reduction == "none":
        pytest.skip("fused autograd needs a scalar loss")
    B, S, D, V = 2, 150, 64, 1000
    inp = small(B * S, D, V, seed=21)
    h = inp.hidden.reshape(B, S, D).clone().requires_grad_(True)
    w = inp.weight.clone().requires_grad_(True)
    y64 = inp.labels.reshape(B, S).long()
    loss = F.linear_cross_entropy(h, w, y64, reduction=reduction, fused=fused)
    g = torch.linspace(-1, 1, B * S, device="cuda").reshape(B, S) if reduction == "none" else None
    (loss * g).sum().backward() if g is not None else loss.backward()
    torch.cuda.synchronize()
    H, W, y = np_inputs(inp)
    f = lce_forward(H, W, y, reduction=reduction)
    gb = g.reshape(-1).double().cpu().numpy() if g is not None else 1.0
    b = lce_backward(H, W, y, reduction=reduction, grad_loss=gb)
    if reduction == "none":
        assert tuple(loss.shape) == (B, S)
        tok = loss.detach().reshape(-1).double().cpu().numpy()
        assert np.abs(tok - f["token_loss"]).max() <= LSE_TOL * np.abs(f["lse"]).max()
    else:
        assert abs(loss.item() - f["loss"]) <= LOSS_TOL * abs(f["loss"])
    assert tuple(h.grad.shape) == (B, S, D)
    assert fro_rel(h.grad.reshape(-1, D).float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL
    assert fro_rel(w.grad.float().cpu().double().numpy(), b["dW"]) <= 2e-2  # bf16 dW for a bf16 leaf
    if reduction == "mean" and not fused:
        bad = y64.clone()
        bad[0, 3] = 2 ** 32 + 5  # would wrap to 5 as a plain int32 cast
        with torch.no_grad():
            out = F.linear_cross_entropy(h.detach(), w.detach(), bad)
        assert math.isnan(out.item())
        with pytest.raises(F.LceError) as e:
            F.check_device_status(device=h.device)
        assert e.value.code == 6


def test_loss_module_with_lm_head(cuda_lib):
    """LinearCrossEntropyLoss (the paper's module name) around a bias-free
    nn.Linear LM head: same loss and gradients as the oracle."""
    import paper_2605_21442_b200 as F

    B, S, D, V = 3, 100, 64, 1000
    inp = small(B * S, D, V, seed=23)
    head = torch.nn.Linear(D, V, bias=False, device="cuda", dtype=torch.bfloat16)
    with torch.no_grad():
        head.weight.copy_(inp.weight)
    h = inp.hidden.reshape(B, S, D).clone().requires_grad_(True)
    loss = F.LinearCrossEntropyLoss(head)(h, inp.labels.reshape(B, S).long())
    loss.backward()
    o = oracle_run(inp)
    assert abs(loss.item() - o["loss"]) <= LOSS_TOL * abs(o["loss"])
    assert fro_rel(h.grad.reshape(-1, D).float().cpu().double().numpy(), o["dH"]) <= GRAD_TOL
    assert fro_rel(head.weight.grad.float().cpu().double().numpy(), o["dW"]) <= 2e-2
    with pytest.raises(ValueError):
        F.LinearCrossEntropyLoss(torch.nn.Linear(D, V, device="cuda", dtype=torch.bfloat16))(h, inp.labels.reshape(B, S))


@pytest.mark.parametrize("N,D,V", [(300, 128, 3000), (257, 4096, 128256)])
def test_none_reduction_per_token_logprobs(cuda_lib, variant, N, D, V):
    """R21 (GRPO / DPO token log-probs): per-token losses and
    the backward of sum_i g_i loss_i for an arbitrary upstream vector g."""
    import paper_2605_21442_b200 as F

    inp = small(N, D, V, seed=9)
    g = torch.randn(N, generator=torch.Generator().manual_seed(1)).float()
    out = F.forward(inp.hidden, inp.weight, inp.labels, reduction="none")
    dh, dw = F.backward(inp.hidden, inp.weight, inp.labels, out["lse"], grad_loss=g.cuda(), reduction="none")
    torch.cuda.synchronize()
    H, W, y = np_inputs(inp)
    f = lce_forward(H, W, y, reduction="none")
    b = lce_backward(H, W, y, reduction="none", grad_loss=g.double().numpy())
    tok = out["token_loss"].cpu().double().numpy()
    assert np.abs(tok - f["token_loss"]).max() <= LSE_TOL * np.abs(f["lse"]).max()
    assert abs(out["loss"].item() - f["loss"]) <= LOSS_TOL * abs(f["loss"])
    assert fro_rel(dh.float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL
    assert fro_rel(dw.cpu().double().numpy(), b["dW"]) <= GRAD_TOL
    assert np.all(dh.float().cpu().numpy()[y == IGNORE] == 0)


@pytest.mark.parametrize("scale", [1.0, -0.5])
def test_autograd_fused(cuda_lib, scale):
    """fused=True: the gradients are produced in the forward call for the
    upstream gradient stated up front (grad_scale), which the library applies
    in its epilogues; backward returns them untouched and the device check of
    the actual upstream gradient stays clean."""
    import paper_2605_21442_b200 as F

    inp = small(300, 64, 1000, seed=19)
    h = inp.hidden.clone().requires_grad_(True)
    w = inp.weight.clone().requires_grad_(True)
    loss = F.linear_cross_entropy(h, w, inp.labels, fused=True, grad_scale=scale)
    (loss * scale).backward()
    F.check_device_status()
    H, W, y = np_inputs(inp)
    o = lce_forward(H, W, y)
    b = lce_backward(H, W, y, grad_loss=scale)
    assert abs(loss.item() - o["loss"]) <= LOSS_TOL * abs(o["loss"])
    assert fro_rel(h.grad.float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL
    assert fro_rel(w.grad.float().cpu().double().numpy(), b["dW"]) <= 2e-2


def test_autograd_fused_upstream_mismatch_is_reported(cuda_lib):
    """An upstream gradient other than the stated grad_scale is never silently
    rescaled: lce_expect_grad flags it on the device and check_device_status
    raises LCE_ERR_UPSTREAM; the next call clears the status."""
    import paper_2605_21442_b200 as F

    inp = small(300, 64, 1000, seed=21)
    h = inp.hidden.clone().requires_grad_(True)
    w = inp.weight.clone().requires_grad_(True)
    loss = F.linear_cross_entropy(h, w, inp.labels, fused=True)
    (loss * 0.5).backward()
    with pytest.raises(F.LceError) as e:
        F.check_device_status()
    assert e.value.code == 12
    loss = F.linear_cross_entropy(h, w, inp.labels, fused=True)
    loss.backward()
    F.check_device_status()


def test_fused_without_grad_runs_forward_only(cuda_lib):
    """No gradient wanted (torch.no_grad or no input requiring grad): the fused
    entry runs lce_forward only -- no dH / dW GEMMs, no fp32 dW buffer."""
    import paper_2605_21442_b200 as F

    inp = small(300, 64, 1000, seed=22)
    ref = F.linear_cross_entropy(inp.hidden, inp.weight, inp.labels).item()
    torch.cuda.synchronize()
    for ctx in (torch.no_grad(), torch.enable_grad()):
        with ctx:
            n0 = F.launch_count()
            loss = F.linear_cross_entropy(inp.hidden, inp.weight, inp.labels, fused=True)
            torch.cuda.synchronize()
            assert F.launch_count() - n0 <= 4  # prep, gather, forward GEMM, combine
            assert loss.item() == ref


def test_native_bf16_dweight(cuda_lib):
    """LCE_DW_BF16: the library rounds the fp32 dW accumulator to bf16 itself
    (RNE); equal to the bf16 rounding of its own fp32 dW up to one ulp of
    summation-order difference, and within the gradient bar of the oracle."""
    import paper_2605_21442_b200 as F

    inp = small(700, 256, 5000, seed=23)
    out = F.forward(inp.hidden, inp.weight, inp.labels)
    _, dw32 = F.backward(inp.hidden, inp.weight, inp.labels, out["lse"])
    _, dw16 = F.backward(inp.hidden, inp.weight, inp.labels, out["lse"], dweight_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert dw16.dtype == torch.bfloat16
    assert torch.equal(dw16, dw32.to(torch.bfloat16))  # same GEMM, same order: exactly RNE(fp32)
    b = lce_backward(*np_inputs(inp))
    assert fro_rel(dw16.float().cpu().double().numpy(), b["dW"]) <= GRAD_TOL
    with pytest.raises(F.LceError):
        F.backward(inp.hidden, inp.weight, inp.labels, out["lse"], dweight_dtype=torch.bfloat16,
                   accumulate_dweight=True)


def test_binding_rejects_mismatched_shapes(cuda_lib):
    """Shapes the C ABI would trust are validated in the binding (ValueError /
    TypeError before any launch)."""
    import paper_2605_21442_b200 as F

    inp = small(64, 64, 300, seed=24)
    h, w, y = inp.hidden, inp.weight, inp.labels
    with pytest.raises(ValueError):
        F.forward(h, w[:, :56].contiguous(), y)          # D mismatch
    with pytest.raises(ValueError):
        F.forward(h, w, y[:63].contiguous())             # labels length
    out = F.forward(h, w, y)
    with pytest.raises(TypeError):
        F.backward(h, w, y, out["lse"].double())         # lse dtype
    with pytest.raises(ValueError):
        F.backward(h, w, y, out["lse"][:10].contiguous())  # lse length
    with pytest.raises(ValueError):
        F.backward(h, w, y, out["lse"], dweight=torch.empty(299, 64, device="cuda"))
    with pytest.raises(ValueError):
        F.backward(h, w, y, out["lse"], grad_loss=torch.ones(2, device="cuda"))
    with pytest.raises(ValueError):
        F.forward_backward(h, w, y, dhidden=torch.empty(64, 56, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError):
        F.kd_forward_backward(h, w, h, w[:200].contiguous(), y)


def test_autograd_none_reduction(cuda_lib):
    import paper_2605_21442_b200 as F

    inp = small(200, 64, 1000, seed=10)
    h = inp.hidden.clone().requires_grad_(True)
    w = inp.weight.clone().requires_grad_(True)
    tok = F.linear_cross_entropy(h, w, inp.labels, reduction="none")
    assert tok.shape == (200,)
    g = torch.linspace(-1, 1, 200, device="cuda")
    (tok * g).sum().backward()
    H, W, y = np_inputs(inp)
    b = lce_backward(H, W, y, reduction="none", grad_loss=g.double().cpu().numpy())
    assert fro_rel(h.grad.float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL


# ------------------------------------------------------------ fused fwd+bwd (no recompute)
def fused_run(inp, reduction="mean", grad=None, budget=0, accumulate_into=None, comm=None):
    import paper_2605_21442_b200 as F

    g = None
    if grad is not None:
        g = torch.as_tensor(grad, dtype=torch.float32, device=inp.hidden.device).reshape(-1)
    dw0 = None if accumulate_into is None else accumulate_into.clone()
    out = F.forward_backward(inp.hidden, inp.weight, inp.labels, grad_loss=g, ignore_index=inp.ignore_index,
                             reduction=reduction, with_token_loss=True, chunk_budget_bytes=budget, dweight=dw0,
                             accumulate_dweight=accumulate_into is not None, comm=comm)
    torch.cuda.synchronize()
    return {
        "loss": out["loss"].item(), "n_valid": int(out["n_valid"].item()),
        "lse": out["lse"].cpu().double().numpy(), "tok": out["token_loss"].cpu().double().numpy(),
        "dH": out["dhidden"].float().cpu().double().numpy(), "dW": out["dweight"].cpu().double().numpy(),
    }


@pytest.mark.parametrize("reduction", ["mean", "sum"])
@pytest.mark.parametrize("regime", ["random", "confident"])
def test_fused_tiny_config(cuda_lib, variant, reduction, regime):
    inp = make_config("tiny", device="cuda", regime=regime)
    assert_parity(fused_run(inp, reduction), oracle_run(inp, reduction), inp.labels.cpu().numpy())


@pytest.mark.parametrize("name", ["llama8b", "qwen7b"])
def test_fused_config_shapes_reduced_n(cuda_lib, name):
    c = CONFIGS[name]
    N = 300
    labels = packed_labels(2048, c["V"], seed=0)[:N] if c["labels"] == "packed" else None
    inp = make_inputs(N, c["D"], c["V"], k=c["k"], device="cuda", ignore_frac=0.1, label_override=labels,
                      regime="confident")
    assert_parity(fused_run(inp), oracle_run(inp), inp.labels.cpu().numpy())


@pytest.mark.parametrize("N,D,V", [(1, 64, 1000), (129, 72, 256), (200, 8, 513), (260, 136, 2)])
def test_fused_ragged_shapes(cuda_lib, N, D, V):
    inp = small(N, D, V, seed=N + 1)
    assert_parity(fused_run(inp), oracle_run(inp), inp.labels.cpu().numpy())


def test_fused_many_row_chunks_with_packed_labels(cuda_lib, variant):
    """Row chunks of 256 (tiny budget): several chunks, trailing chunks with no
    valid row (packed labels compact to the front), dW accumulated across chunks."""
    V, D = 3000, 128
    lab = packed_labels(2048, V, seed=1)[:1100]
    inp = small(1100, D, V, labels=lab)
    budget = 256 * 2 * 3072  # Nc = 256 rows per chunk (2 bytes per chunk element)
    g = fused_run(inp, budget=budget)
    assert_parity(g, oracle_run(inp), lab)
    one = fused_run(inp)
    np.testing.assert_array_equal(g["lse"], one["lse"])
    assert fro_rel(g["dW"], one["dW"]) <= 1e-5


def test_fused_small_vocab_row_bound(cuda_lib):
    """V_l < 4 D: the budget bounds the chunk by its N_c x D row buffers
    (8 bytes per element), not by the q chunk: 512-row chunks here (the q
    chunk alone would allow 1024), six chunks, dW accumulated over them."""
    N, D, V = 3000, 256, 300
    inp = small(N, D, V, seed=5)
    g = fused_run(inp, budget=8 * D * 512)
    assert_parity(g, oracle_run(inp), inp.labels.cpu().numpy())


@pytest.mark.parametrize("n_valid", [511, 512, 513, 1024])
def test_fused_default_plan_chunk_boundary(cuda_lib, n_valid):
    """Default (two-chunk) plan, N = 1024 -> 512-row chunks: the compacted
    valid rows end just before, at and just after the chunk boundary (the
    second chunk empty, or holding one row) and fill both chunks."""
    N, D, V = 1024, 128, 3000
    rng = np.random.default_rng(n_valid)
    lab = rng.integers(0, V, N).astype(np.int32)
    lab[rng.permutation(N)[:N - n_valid]] = IGNORE
    inp = small(N, D, V, seed=n_valid, labels=lab)
    g = fused_run(inp)
    assert g["n_valid"] == n_valid
    assert_parity(g, oracle_run(inp), lab)


def test_fused_none_accumulate_and_empty(cuda_lib):
    inp = small(300, 64, 1000, seed=11)
    gvec = np.linspace(-2, 1, 300)
    H, W, y = np_inputs(inp)
    b = lce_backward(H, W, y, reduction="none", grad_loss=gvec)
    f = lce_forward(H, W, y, reduction="none")
    base = torch.randn(1000, 64, device="cuda")
    g = fused_run(inp, "none", grad=gvec, accumulate_into=base)
    assert np.abs(g["tok"] - f["token_loss"]).max() <= LSE_TOL * np.abs(f["lse"]).max()
    assert fro_rel(g["dH"], b["dH"]) <= GRAD_TOL
    assert fro_rel(g["dW"] - base.cpu().double().numpy(), b["dW"]) <= GRAD_TOL
    e = fused_run(small(0, 64, 1000))
    assert e["loss"] == 0 and e["n_valid"] == 0 and not e["dW"].any()
    allign = fused_run(small(300, 64, 1000, labels=np.full(300, IGNORE, dtype=np.int32)))
    assert allign["loss"] == 0 and not allign["dH"].any() and not allign["dW"].any()


def test_fused_single_rank_communicator_path(cuda_lib):
    """Vocab-parallel fused path (per-chunk MAX/SUM all-reduces, fp32 dH chunk
    all-reduced on the side stream) on a one-rank NCCL communicator."""
    import paper_2605_21442_b200 as F

    comm = F.Comm.single()
    try:
        lab = packed_labels(2048, 3000, seed=2)[:900]
        inp = small(900, 128, 3000, labels=lab)
        out = F.forward_backward(inp.hidden, inp.weight, inp.labels, with_token_loss=True, comm=comm,
                                 chunk_budget_bytes=256 * 2 * 3072)
        torch.cuda.synchronize()
        g = {"loss": out["loss"].item(), "n_valid": int(out["n_valid"].item()),
             "lse": out["lse"].cpu().double().numpy(), "tok": out["token_loss"].cpu().double().numpy(),
             "dH": out["dhidden"].float().cpu().double().numpy(), "dW": out["dweight"].cpu().double().numpy()}
        assert_parity(g, oracle_run(inp), lab)
    finally:
        comm.close()


@pytest.mark.parametrize("v0,vl", [(384, 500), (999, 1), (0, 256)])
@pytest.mark.parametrize("path", ["split", "fused"])
def test_vocab_shard_offsets_single_rank(cuda_lib, path, v0, vl):
    """A one-rank communicator over a vocab SHARD (vocab_start > 0, labels
    global, some outside the shard): the GPU computes exactly the shard
    statistics of P:180's loss parallel -- oracle shard_stats / shard_backward
    (lse of the shard, target logit only from the owning shard, G without the
    onehot for foreign labels)."""
    import paper_2605_21442_b200 as F
    from oracle import shard_backward, shard_stats

    V, D = 1000, 128
    inp = small(300, D, V, seed=17)
    Wsh = inp.weight[v0:v0 + vl].contiguous()
    comm = F.Comm.single()
    try:
        if path == "split":
            out = F.forward(inp.hidden, Wsh, inp.labels, comm=comm, vocab_start=v0, vocab_total=V,
                            with_token_loss=True)
            dh, dw = F.backward(inp.hidden, Wsh, inp.labels, out["lse"], comm=comm, vocab_start=v0, vocab_total=V)
        else:
            out = F.forward_backward(inp.hidden, Wsh, inp.labels, comm=comm, vocab_start=v0, vocab_total=V,
                                     with_token_loss=True, chunk_budget_bytes=256 * 2 * 512)
            dh, dw = out["dhidden"], out["dweight"]
        torch.cuda.synchronize()
    finally:
        comm.close()
    H, W, y = np_inputs(inp)
    st = shard_stats(H, W[v0:v0 + vl], y, v0, V)
    valid = st["valid"]
    lse_sh = np.where(valid, st["m"] + np.log(np.where(valid, st["s"], 1.0)), 0.0)
    tok_sh = np.where(valid, lse_sh - st["z_target"], 0.0)
    assert np.abs(out["lse"].cpu().double().numpy() - lse_sh).max() <= LSE_TOL * max(1, np.abs(lse_sh).max())
    assert np.abs(out["token_loss"].cpu().double().numpy() - tok_sh).max() <= LSE_TOL * max(1, np.abs(lse_sh).max())
    sb = shard_backward(H, W[v0:v0 + vl], y, v0, lse_sh, 1.0 / int(valid.sum()))
    assert fro_rel(dh.float().cpu().double().numpy(), sb["dH_partial"]) <= GRAD_TOL
    assert fro_rel(dw.cpu().double().numpy(), sb["dW_shard"]) <= GRAD_TOL


def test_vocab_shard_full_size_p8_rank(cuda_lib):
    """The per-rank workload of the 8-GPU vocab-parallel 8B run on one GPU:
    rank 2's shard of W (V_l = 16,032 rows, not a tile multiple) at N = 16,384,
    D = 4,096 through the fused path on a one-rank communicator, so the 8,192-row
    chunks take the wide dH / dW tiles over a ragged vocab extent.  Every row's
    lse / token loss and the full dW shard against the oracle's shard
    statistics, with the shard lse the ORACLE computes for every row
    (shard_stats in row blocks): no GPU output enters the oracle."""
    import paper_2605_21442_b200 as F
    from oracle import shard_backward, shard_stats

    c = CONFIGS["llama8b"]
    N, D, V = c["N"], c["D"], c["V"]
    v0, vl = F.shard_range(V, 8, 2)
    inp = make_config("llama8b", device="cuda")
    Wsh = inp.weight[v0:v0 + vl].contiguous()
    comm = F.Comm.single()
    try:
        out = F.forward_backward(inp.hidden, Wsh, inp.labels, comm=comm, vocab_start=v0, vocab_total=V,
                                 with_token_loss=True)
        torch.cuda.synchronize()
    finally:
        comm.close()
    H = inp.hidden.float().cpu().numpy()
    Wn = Wsh.float().cpu().numpy()
    y = inp.labels.cpu().numpy()
    lse_sh = np.zeros(N)
    tok_sh = np.zeros(N)
    for a in range(0, N, 2048):
        st = shard_stats(H[a:a + 2048], Wn, y[a:a + 2048], v0, V)
        v = st["valid"]
        lse_sh[a:a + 2048][v] = st["m"][v] + np.log(st["s"][v])
        tok_sh[a:a + 2048][v] = lse_sh[a:a + 2048][v] - st["z_target"][v]
    bound = LSE_TOL * max(1, np.abs(lse_sh).max())
    assert np.abs(out["lse"].cpu().double().numpy() - lse_sh).max() <= bound
    assert np.abs(out["token_loss"].cpu().double().numpy() - tok_sh).max() <= bound
    nv = int((y != IGNORE).sum())
    dW = np.zeros((vl, D))
    for a in range(0, N, 2048):
        dW += shard_backward(H[a:a + 2048], Wn, y[a:a + 2048], v0, lse_sh[a:a + 2048], 1.0 / nv)["dW_shard"]
    assert fro_rel(out["dweight"].cpu().double().numpy(), dW) <= GRAD_TOL


@pytest.mark.parametrize("path", ["split", "fused"])
def test_cuda_graph_capture_replays_bitwise(cuda_lib, path):
    """Every launch is stream-ordered with no host sync or allocation, so a
    whole fwd+bwd step can be captured in a CUDA graph and replayed."""
    import paper_2605_21442_b200 as F

    inp = small(700, 256, 5000, seed=18)
    h, w, y = inp.hidden, inp.weight, inp.labels
    ws = F.Workspace()
    out = {"loss": torch.empty(1, device="cuda"), "lse": torch.empty(700, device="cuda"),
           "n_valid": torch.empty(1, dtype=torch.int32, device="cuda"), "token_loss": None}
    dH = torch.empty_like(h)
    dW = torch.empty(w.shape, dtype=torch.float32, device="cuda")

    def step():
        if path == "fused":
            F.forward_backward(h, w, y, dhidden=dH, dweight=dW, workspace=ws, out=out,
                               chunk_budget_bytes=256 * 2 * 5120)
        else:
            F.forward(h, w, y, workspace=ws, out=out)
            F.backward(h, w, y, out["lse"], dhidden=dH, dweight=dW, workspace=ws, chunk_budget_bytes=700 * 2 * 1024)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ref = [out["loss"].clone(), out["lse"].clone(), dH.clone(), dW.clone()]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for t in (out["loss"], out["lse"], dH, dW):
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, [out["loss"], out["lse"], dH, dW]):
        assert torch.equal(a, b)


def test_fused_matches_recompute_path(cuda_lib):
    """Same inputs through lce_forward + lce_backward and lce_forward_backward:
    identical lse/loss (same forward GEMM), gradients within bf16 rounding."""
    inp = small(700, 256, 5000, seed=12, regime="confident")
    a, b = gpu_run(inp), fused_run(inp)
    np.testing.assert_array_equal(a["lse"], b["lse"])
    assert abs(a["loss"] - b["loss"]) <= 1e-6 * abs(a["loss"])
    assert fro_rel(b["dH"], a["dH"]) <= 5e-3 and fro_rel(b["dW"], a["dW"]) <= 5e-3


# ------------------------------------------------------------ randomized shapes (property test)
def test_random_shapes_all_paths(cuda_lib):
    """40 seeded random problems (N in [1, 700], D in 8..264 step 8, V in [1, 3000],
    random ignore fraction, both reductions, every GEMM variant, random chunk
    budgets) through the split and fused paths, each against the oracle."""
    rng = np.random.default_rng(2024)
    for case in range(40):
        N = int(rng.integers(1, 700))
        D = int(8 * rng.integers(1, 34))
        V = int(rng.integers(1, 3000))
        frac = float(rng.choice([0.0, 0.1, 0.5, 0.95]))
        red = str(rng.choice(["mean", "sum"]))
        os.environ["LCE_GEMM"] = str(rng.choice(["default", "pair", "wide", "single"]))
        try:
            inp = small(N, D, V, seed=100 + case, ignore_frac=frac)
            o = oracle_run(inp, red)
            lab = inp.labels.cpu().numpy()
            budget = int(rng.choice([0, 256 * 2 * 512, 256 * 6 * 1024]))
            assert_parity(gpu_run(inp, red, budget=budget), o, lab)
            assert_parity(fused_run(inp, red, budget=budget), o, lab)
        finally:
            del os.environ["LCE_GEMM"]


# ------------------------------------------------------------ NEXT-2: AdamW in the dW epilogue
def _adam_state(V, D, seed):
    g = torch.Generator().manual_seed(seed)
    theta = torch.randn(V, D, generator=g) * 0.05
    m = torch.randn(V, D, generator=g) * 1e-3
    v = torch.rand(V, D, generator=g) * 1e-6 + 1e-7
    return theta, m, v


@pytest.mark.parametrize("N,D,V,budget", [(300, 64, 1000, 0), (300, 128, 3000, 300 * 2 * 512), (0, 64, 1000, 0)])
def test_backward_adamw_matches_oracle_step(cuda_lib, variant, N, D, V, budget):
    """P:137-160 optimizer-in-backward: the fused AdamW step on the LM head
    equals the oracle's dW followed by the oracle's AdamW step."""
    import paper_2605_21442_b200 as F
    from oracle import adamw_step

    inp = small(N, D, V, seed=13)
    theta, m, v = _adam_state(V, D, 5)
    hp = dict(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1, step=7)
    w = theta.to(torch.bfloat16).cuda()
    th_d, m_d, v_d = theta.cuda(), m.cuda(), v.cuda()
    out = F.forward(inp.hidden, w, inp.labels)
    F.backward_adamw(inp.hidden, w, inp.labels, out["lse"], th_d, m_d, v_d, chunk_budget_bytes=budget, **hp)
    torch.cuda.synchronize()
    H, _, y = np_inputs(inp)
    Wb = w.float().cpu().numpy() if N == 0 else theta.to(torch.bfloat16).float().numpy()
    gW = lce_backward(H, Wb, y)["dW"] if N > 0 else np.zeros((V, D))
    th_o, m_o, v_o = adamw_step(theta.double().numpy(), gW, m.double().numpy(), v.double().numpy(), hp["step"],
                                lr=hp["lr"], beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    m0, v0 = m.double().numpy(), v.double().numpy()
    # gradient contributions carry the GEMM's bf16-G error; the moments' old parts are exact
    assert fro_rel(m_d.cpu().double().numpy() - 0.9 * m0, m_o - 0.9 * m0) <= GRAD_TOL
    assert fro_rel(v_d.cpu().double().numpy() - 0.95 * v0, v_o - 0.95 * v0) <= 2 * GRAD_TOL
    dth = th_d.cpu().double().numpy() - theta.double().numpy()
    assert fro_rel(dth, th_o - theta.double().numpy()) <= GRAD_TOL
    assert torch.equal(w.cpu(), th_d.cpu().to(torch.bfloat16))  # W = bf16(theta) (RNE)


def test_backward_adamw_equals_dw_then_torch_adamw(cuda_lib):
    """in-backward AdamW == standard AdamW applied to the same dW (K=1)."""
    import paper_2605_21442_b200 as F

    inp = small(500, 256, 5000, seed=14)
    theta, m, v = _adam_state(5000, 256, 6)
    w = theta.to(torch.bfloat16).cuda()
    out = F.forward(inp.hidden, w, inp.labels)
    _, dW = F.backward(inp.hidden, w, inp.labels, out["lse"])
    p = torch.nn.Parameter(theta.clone().cuda())
    opt = torch.optim.AdamW([p], lr=2e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, foreach=False)
    p.grad = torch.zeros_like(p)
    opt.step()  # step 1 on a zero grad to reach step 2 with nonzero state
    opt.state[p]["exp_avg"].copy_(m.cuda())
    opt.state[p]["exp_avg_sq"].copy_(v.cuda())
    p.data.copy_(theta.cuda())
    p.grad = dW.clone()
    opt.step()
    th_d, m_d, v_d = theta.cuda(), m.cuda(), v.cuda()
    F.backward_adamw(inp.hidden, w, inp.labels, out["lse"], th_d, m_d, v_d, lr=2e-4, betas=(0.9, 0.999), eps=1e-8,
                     weight_decay=0.01, step=2)
    torch.cuda.synchronize()
    assert torch.allclose(m_d, opt.state[p]["exp_avg"], rtol=1e-5, atol=1e-9)
    assert torch.allclose(v_d, opt.state[p]["exp_avg_sq"], rtol=1e-5, atol=1e-14)
    dref = p.detach() - theta.cuda()
    dgot = th_d - theta.cuda()
    # DESIGN.md R29: both sides update fp32 theta in fp32 with different operation
    # orders (torch: decay, addcdiv; here: decay, fused divide), so they agree up to
    # a few ulp of |theta| (4e-7 |theta| = 3.4 ulp) plus 1e-4 of the step itself
    assert ((dgot - dref).abs() <= 1e-4 * dref.abs() + 4e-7 * theta.cuda().abs() + 1e-12).all()


# ------------------------------------------------------------ NEXT-4: linear KD loss
def _kd_inputs(N, Ds, Dt, V, seed, ignore_frac=0.1, labels=None):
    s = make_inputs(N, Ds, V, k=seed, device="cuda", ignore_frac=ignore_frac, label_override=labels)
    t = make_inputs(N, Dt, V, k=seed + 100, device="cuda", ignore_frac=0.0,
                    label_override=s.labels.cpu().numpy())
    return s, t


def _kd_check(s, t, reduction="mean", grad=None, budget=0):
    import paper_2605_21442_b200 as F
    from oracle import kd_backward, kd_forward

    g = None if grad is None else torch.as_tensor(grad, dtype=torch.float32, device="cuda").reshape(-1)
    out = F.kd_forward_backward(s.hidden, s.weight, t.hidden, t.weight, s.labels, grad_loss=g, reduction=reduction,
                                chunk_budget_bytes=budget)
    torch.cuda.synchronize()
    Hs, Ws, y = np_inputs(s)
    Ht, Wt = t.hidden.float().cpu().numpy(), t.weight.float().cpu().numpy()
    f = kd_forward(Hs, Ws, Ht, Wt, y, reduction=reduction)
    b = kd_backward(Hs, Ws, Ht, Wt, y, reduction=reduction, grad_loss=1.0 if grad is None else grad)
    assert int(out["n_valid"].item()) == f["n_valid"]
    assert abs(out["loss"].item() - f["loss"]) <= LOSS_TOL * abs(f["loss"])
    tok = out["token_loss"].cpu().double().numpy()
    assert np.abs(tok - f["token_loss"]).max() <= LSE_TOL * max(1.0, np.abs(f["lse_s"]).max())
    assert fro_rel(out["dhidden"].float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL
    assert fro_rel(out["dweight"].cpu().double().numpy(), b["dW"]) <= GRAD_TOL
    assert np.all(out["dhidden"].float().cpu().numpy()[y == IGNORE] == 0)
    return out


@pytest.mark.parametrize("N,Ds,Dt,V", [(300, 64, 128, 1000), (257, 4096, 8192, 128256)])
def test_kd_matches_oracle(cuda_lib, variant, N, Ds, Dt, V):
    """Chunked linear KD (forward KL) vs the fp64 oracle: student 8B head,
    teacher 70B head at the exact (D, V) of the configs."""
    s, t = _kd_inputs(N, Ds, Dt, V, seed=15)
    _kd_check(s, t)


def test_kd_many_chunks_none_and_self_distillation(cuda_lib):
    import paper_2605_21442_b200 as F

    s, t = _kd_inputs(700, 128, 64, 3000, seed=16)
    _kd_check(s, t, "none", grad=np.linspace(-1, 2, 700), budget=256 * 10 * 3072)
    _kd_check(s, t, "sum", budget=256 * 10 * 3072)
    # teacher == student: p_S - p_T is exactly zero, so are the gradients
    out = F.kd_forward_backward(s.hidden, s.weight, s.hidden, s.weight, s.labels)
    torch.cuda.synchronize()
    assert out["dhidden"].abs().max().item() == 0 and out["dweight"].abs().max().item() == 0


def test_kd_vocab_shard_single_rank(cuda_lib):
    """KD under a one-rank communicator over a vocab shard: the softmaxes run
    over the shard's vocabulary only, so the result is kd_forward/kd_backward
    of the shard's heads (exercises the MAX/SUM exchanges and the fp32 dH
    all-reduce path)."""
    import paper_2605_21442_b200 as F
    from oracle import kd_backward, kd_forward

    V, v0, vl = 3000, 1000, 1500
    s, t = _kd_inputs(500, 128, 64, V, seed=20)
    Ws = s.weight[v0:v0 + vl].contiguous()
    Wt = t.weight[v0:v0 + vl].contiguous()
    comm = F.Comm.single()
    try:
        out = F.kd_forward_backward(s.hidden, Ws, t.hidden, Wt, s.labels, comm=comm, vocab_start=v0, vocab_total=V,
                                    chunk_budget_bytes=256 * 10 * 1536)
        torch.cuda.synchronize()
    finally:
        comm.close()
    Hs, _, y = np_inputs(s)
    Ht = t.hidden.float().cpu().numpy()
    Wsn, Wtn = Ws.float().cpu().numpy(), Wt.float().cpu().numpy()
    f = kd_forward(Hs, Wsn, Ht, Wtn, y)
    b = kd_backward(Hs, Wsn, Ht, Wtn, y)
    assert abs(out["loss"].item() - f["loss"]) <= LOSS_TOL * abs(f["loss"])
    assert fro_rel(out["dhidden"].float().cpu().double().numpy(), b["dH"]) <= GRAD_TOL
    assert fro_rel(out["dweight"].cpu().double().numpy(), b["dW"]) <= GRAD_TOL


# ------------------------------------------------------------ full size, bench launch configuration
@pytest.mark.parametrize("name,path", [("llama8b", "fused"), ("llama8b", "split"), ("qwen7b", "fused"),
                                       ("qwen7b", "split"), ("llama1b", "fused"), ("llama70b", "fused"),
                                       ("llama70b", "split"), ("llama1b_1m", "fused")])
def test_full_size_sampled_rows_and_invariants(cuda_lib, name, path):
    """At full size in the bench's launch configuration (fused = bench default):
    sampled rows (lse, token loss, dH) vs the oracle row by row; loss == mean
    of token losses; sum_j dW_j ~ 0 (P2); <H, dH> == <W, dW> (P11).  Full-size
    outputs stay on the GPU; only sampled rows go to the host."""
    import paper_2605_21442_b200 as F

    inp = make_config(name, device="cuda")
    if path == "fused":
        out = F.forward_backward(inp.hidden, inp.weight, inp.labels, with_token_loss=True)
        dH, dW = out["dhidden"], out["dweight"]
    else:
        out = F.forward(inp.hidden, inp.weight, inp.labels, with_token_loss=True)
        dH, dW = F.backward(inp.hidden, inp.weight, inp.labels, out["lse"])
    torch.cuda.synchronize()
    # P11: z is bilinear in (H, W), so sum_i h_i.dH_i = sum_ij G_ij z_ij = sum_j w_j.dW_j
    hdh = float((inp.hidden.double() * dH.double()).sum())
    wdw = float((inp.weight.double() * dW.double()).sum())
    assert abs(hdh - wdw) <= 2e-2 * max(abs(hdh), abs(wdw)), (hdh, wdw)
    col = float(dW.double().sum(dim=0).norm())  # P2
    assert col <= 1e-2 * float(dW.double().norm())
    y = inp.labels.cpu().numpy()
    nv = int((y != IGNORE).sum())
    assert int(out["n_valid"].item()) == nv
    tok = out["token_loss"].double()
    assert abs(out["loss"].item() - tok.sum().item() / nv) <= 1e-4 * abs(out["loss"].item())
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(len(y), size=48, replace=False))
    rows = np.concatenate([rows, [0, len(y) - 1]])
    W = inp.weight.float().cpu().numpy()
    H = inp.hidden[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    o = lce_rows(H, W, y[rows], np.arange(len(rows)), n_valid=nv)
    lse = out["lse"].cpu().double().numpy()[rows]
    lerr = np.abs(lse - o["lse"]) / np.maximum(1, np.abs(o["lse"]))
    assert lerr.max() <= LSE_TOL
    assert np.abs(tok.cpu().numpy()[rows] - o["token_loss"]).max() <= LSE_TOL * max(1, np.abs(o["lse"]).max())
    dh_rows = dH[torch.from_numpy(rows).cuda()].float().cpu().double().numpy()
    assert fro_rel(dh_rows, o["dH"]) <= GRAD_TOL


# oracle lse of every row of a full-size config (fp64, the oracle's own; shared by both paths)
_ORACLE_FULL = {}


def _oracle_full(name, inp):
    if name not in _ORACLE_FULL:
        H = inp.hidden.float().cpu().numpy()
        W = inp.weight.float().cpu().numpy()
        y = inp.labels.cpu().numpy()
        _ORACLE_FULL.clear()  # one config's host copies at a time
        _ORACLE_FULL[name] = (H, W, y, lce_lse(H, W, y))
    return _ORACLE_FULL[name]


@pytest.mark.parametrize("name,path", [(n, p) for n in ("llama1b", "llama8b", "qwen7b", "llama70b")
                                       for p in ("fused", "split")])
def test_full_size_dweight_rows_and_every_lse(cuda_lib, name, path):
    """Full size, in the bench's launch configuration, independent of the GPU:
    the oracle computes its own lse for EVERY valid row (lce_lse, fp64, 2 N_v V D
    flops on the host) and from it the loss, every row's lse / token loss, and
    sampled rows of dW (lce_dweight_rows: dW_j = sum_i c (p_ij - [y_i = j]) h_i):
    256 random vocab rows, the whole last 256-row vocab tile (the ragged end of
    a 512-row wide dW tile at V = 128,256) and the labels of 64 sampled tokens.
    No oracle input comes from a GPU output."""
    import paper_2605_21442_b200 as F

    inp = make_config(name, device="cuda")
    if path == "fused":
        out = F.forward_backward(inp.hidden, inp.weight, inp.labels, with_token_loss=True)
        dW = out["dweight"]
    else:
        out = F.forward(inp.hidden, inp.weight, inp.labels, with_token_loss=True)
        _, dW = F.backward(inp.hidden, inp.weight, inp.labels, out["lse"])
    torch.cuda.synchronize()
    H, W, y, lse_o = _oracle_full(name, inp)
    V = W.shape[0]
    valid = y != IGNORE
    nv = int(valid.sum())
    rows = np.flatnonzero(valid)
    zt = np.einsum("ij,ij->i", H[rows].astype(np.float64), W[y[rows]].astype(np.float64))
    tok_o = np.zeros(len(y))
    tok_o[rows] = lse_o[rows] - zt
    loss_o = tok_o.sum() / nv
    assert abs(out["loss"].item() - loss_o) <= LOSS_TOL * abs(loss_o), (out["loss"].item(), loss_o)
    bound = LSE_TOL * max(1.0, np.abs(lse_o).max())
    assert np.abs(out["lse"].cpu().double().numpy() - lse_o).max() <= bound
    assert np.abs(out["token_loss"].cpu().double().numpy() - tok_o).max() <= bound
    rng = np.random.default_rng(7)
    J = np.unique(np.concatenate([rng.choice(V, 256, replace=False), np.arange(V - 256, V),
                                  y[rng.choice(rows, 64, replace=False)]]))
    o = lce_dweight_rows(H, W, y, J, lse=lse_o)
    got = dW[torch.from_numpy(J).cuda()].cpu().double().numpy()
    assert fro_rel(got, o["dW_rows"]) <= GRAD_TOL, fro_rel(got, o["dW_rows"])
    # the rows that are labels carry the -h_i onehot term: check them on their own too
    lab = np.isin(J, y[rows])
    assert fro_rel(got[lab], o["dW_rows"][lab]) <= GRAD_TOL


def test_debug_sync_build_runs_clean(cuda_lib):
    """liblce_debug.so (-DLCE_DEBUG_SYNC: every device spin wait traps after
    2 s instead of hanging, sm100.cuh SpinGuard) on the sanitizer workload
    (every entry point and GEMM variant at small ragged shapes), the smoke
    parity check and one full-size 1B fused + split step (K-lockstep on):
    no wait may come near the deadline on a correct schedule."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dbg = os.path.join(root, "paper_2605_21442_b200", "liblce_debug.so")
    if not os.path.exists(dbg):
        pytest.fail("liblce_debug.so missing: run __graft_entry__.build()")
    env = dict(os.environ, LCE_LIB_PATH=dbg)
    r = subprocess.run([sys.executable, "-c", "import paper_2605_21442_b200._lib as L; print(L.LIB_PATH)"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.stdout.strip().endswith("liblce_debug.so"), r.stdout + r.stderr
    for cmd in (["scripts/sanitize.py"], ["-c", "import __graft_entry__ as g; g.smoke()"],
                ["scripts/one_step.py", "--config", "llama1b", "--path", "fused", "--steps", "1"],
                ["scripts/one_step.py", "--config", "llama1b", "--path", "split", "--steps", "1"]):
        r = subprocess.run([sys.executable, *cmd], cwd=root, env=env, capture_output=True, text=True, timeout=600)
        out = r.stdout + r.stderr
        assert r.returncode == 0 and "timed out" not in out, (cmd, out[-2000:])
