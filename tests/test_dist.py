"""Multi-process (gloo, CPU) tests of the vocab-parallel path's host logic and
of the exchange protocol the CUDA path implements (P:169, P:180 loss parallel):
all-reduce MAX of the per-row shard max, rescale, all-reduce SUM of
(sum-exp, target logit), then all-reduce SUM of the partial dH.  And the
token-parallel protocol (W replicated, rows sharded): all-reduce SUM of N_v,
each rank's MEAN share with the global N_v, loss and dW summed over ranks."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import IGNORE_INDEX, lce_backward, lce_forward, shard_backward, shard_stats
from paper_2605_21442_b200.dist import broadcast_bytes, max_over_ranks, shard_range


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _problem():
    rng = np.random.default_rng(0)
    N, D, V = 40, 8, 101
    H = rng.standard_normal((N, D))
    W = rng.standard_normal((V, D)) / math.sqrt(D)
    y = rng.integers(0, V, size=N)
    y[rng.permutation(N)[:6]] = IGNORE_INDEX
    return H, W, y


def _worker_plumbing(rank, world, port, out):
    _init(rank, world, port)
    uid = broadcast_bytes(bytes(range(128)) if rank == 0 else None)
    assert uid == bytes(range(128))
    m = max_over_ranks(float(rank) + 0.5)
    assert m == world - 0.5
    dist.barrier()
    dist.destroy_process_group()


def _worker_protocol(rank, world, port, reduction):
    _init(rank, world, port)
    H, W, y = _problem()
    V = W.shape[0]
    v0, vl = shard_range(V, world, rank)
    st = shard_stats(H, W[v0:v0 + vl], y, v0, V)
    valid = st["valid"]
    # C1 step 1: MAX all-reduce of the local max (ignored rows: -inf)
    m_loc = torch.tensor(st["m"])
    M = m_loc.clone()
    dist.all_reduce(M, op=dist.ReduceOp.MAX)
    # rescale, then C1 step 2: SUM all-reduce of (s * e^{m - M}, z_target)
    s = torch.tensor(st["s"]) * torch.exp(torch.where(torch.tensor(valid), m_loc - M, torch.zeros_like(M)))
    sz = torch.cat([s, torch.tensor(st["z_target"])])
    dist.all_reduce(sz, op=dist.ReduceOp.SUM)
    N = len(y)
    S, zt = sz[:N].numpy(), sz[N:].numpy()
    lse = np.where(valid, M.numpy() + np.log(np.where(valid, S, 1.0)), 0.0)
    tok = np.where(valid, lse - zt, 0.0)
    nv = int(valid.sum())
    loss = tok.sum() / nv if reduction == "mean" else tok.sum()
    ref = lce_forward(H, W, y, reduction=reduction)
    np.testing.assert_allclose(lse, ref["lse"], rtol=1e-13, atol=1e-13)
    assert loss == pytest.approx(ref["loss"], rel=1e-12)
    # C2: partial dH summed over ranks; dW shards concatenated in rank order
    c = 1.0 / nv if reduction == "mean" else 1.0
    sb = shard_backward(H, W[v0:v0 + vl], y, v0, lse, c)
    dh = torch.tensor(sb["dH_partial"])
    dist.all_reduce(dh, op=dist.ReduceOp.SUM)
    cap = -(-V // world)
    mine = torch.zeros(cap, W.shape[1], dtype=torch.float64)
    mine[:vl] = torch.tensor(sb["dW_shard"])
    dws = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(dws, mine)
    full = torch.cat([d[:shard_range(V, world, r)[1]] for r, d in enumerate(dws)])
    gref = lce_backward(H, W, y, reduction=reduction)
    np.testing.assert_allclose(dh.numpy(), gref["dH"], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(full.numpy(), gref["dW"], rtol=1e-11, atol=1e-14)
    dist.barrier()
    dist.destroy_process_group()


def _worker_token_protocol(rank, world, port, reduction):
    """Rows sharded unevenly over ranks (rank 0 may hold none): the library's
    LCE_PAR_TOKEN exchange -- N_v all-reduced, MEAN divides by the global N_v
    in the loss and in the gradient scale, loss all-reduced, dW the rank's
    share -- reproduces the full batch."""
    _init(rank, world, port)
    H, W, y = _problem()
    N = len(y)
    bounds = [0] + sorted(np.random.default_rng(world).integers(0, N + 1, size=world - 1).tolist()) + [N]
    bounds[1] = 0 if world > 2 else bounds[1]  # rank 0 without tokens when there are >= 3 ranks
    r0, r1 = bounds[rank], bounds[rank + 1]
    Hr, yr = H[r0:r1], y[r0:r1]
    nv = torch.tensor([int(((yr != IGNORE_INDEX) & (yr >= 0)).sum())], dtype=torch.int64)
    dist.all_reduce(nv, op=dist.ReduceOp.SUM)
    nv = int(nv.item())
    f = lce_forward(Hr, W, yr, reduction="sum") if r1 > r0 else {"loss": 0.0}
    loss = torch.tensor([f["loss"] / nv if reduction == "mean" else f["loss"]], dtype=torch.float64)
    dist.all_reduce(loss, op=dist.ReduceOp.SUM)
    ref = lce_forward(H, W, y, reduction=reduction)
    assert loss.item() == pytest.approx(ref["loss"], rel=1e-12)
    g = 1.0 / nv if reduction == "mean" else 1.0
    if r1 > r0:
        b = lce_backward(Hr, W, yr, reduction="sum", grad_loss=g)
        dw, dh = torch.tensor(b["dW"]), b["dH"]
    else:
        dw, dh = torch.zeros(W.shape, dtype=torch.float64), np.zeros((0, W.shape[1]))
    dist.all_reduce(dw, op=dist.ReduceOp.SUM)
    gref = lce_backward(H, W, y, reduction=reduction)
    np.testing.assert_allclose(dw.numpy(), gref["dW"], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(dh, gref["dH"][r0:r1], rtol=1e-11, atol=1e-14)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,reduction", [(2, "mean"), (3, "mean"), (3, "sum")])
def test_gloo_token_parallel_protocol(world, reduction):
    mp.spawn(_worker_token_protocol, args=(world, free_port(), reduction), nprocs=world, join=True)


@pytest.mark.parametrize("V,P", [(128256, 8), (152064, 8), (1000, 3), (101, 2), (7, 8), (5, 1)])
def test_shard_range_partitions_the_vocab(V, P):
    spans = [shard_range(V, P, r) for r in range(P)]
    assert spans[0][0] == 0
    for (a, n), (b, _) in zip(spans, spans[1:]):
        assert a + n == b
    assert spans[-1][0] + spans[-1][1] == V
    assert all(n <= -(-V // P) for _, n in spans)
    with pytest.raises(ValueError):
        shard_range(V, P, P)


def test_gloo_plumbing_world2():
    mp.spawn(_worker_plumbing, args=(2, free_port(), None), nprocs=2, join=True)


@pytest.mark.parametrize("world,reduction", [(2, "mean"), (3, "sum")])
def test_gloo_loss_parallel_protocol(world, reduction):
    mp.spawn(_worker_protocol, args=(world, free_port(), reduction), nprocs=world, join=True)
