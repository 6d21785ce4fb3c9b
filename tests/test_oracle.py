"""Pins of the fp64 oracle against things other than itself.

Each test names the pin and the passage it follows.  A plausible mistake in
the oracle (dropped term, wrong sign or index, transposed operand, wrong
normaliser, ignored rows leaking) fails at least one of them.
"""

import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import (
    IGNORE_INDEX,
    combine_shard_stats,
    lce_backward,
    lce_dweight_rows,
    lce_forward,
    lce_lse,
    lce_rows,
    shard_stats,
)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "lce_closed_forms.json")


def rand_problem(N, D, V, seed, ignore_frac=0.2, scale=1.0):
    rng = np.random.default_rng(seed)
    H = rng.standard_normal((N, D)) * scale
    W = rng.standard_normal((V, D)) / math.sqrt(D)
    y = rng.integers(0, V, size=N)
    n_ign = int(round(ignore_frac * N))
    y[rng.permutation(N)[:n_ign]] = IGNORE_INDEX
    return H, W, y


# ---------------------------------------------------------------- golden cases
def test_golden_closed_forms():
    """SPEC S:272, S:273, S:282 examples and the hand-derived V=2 case (P5)."""
    with open(GOLDEN) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        H = np.array(c["hidden"], dtype=np.float64)
        W = np.array(c["weight"], dtype=np.float64)
        y = np.array(c["labels"])
        f = lce_forward(H, W, y, reduction=c["reduction"])
        b = lce_backward(H, W, y, reduction=c["reduction"])
        assert f["loss"] == pytest.approx(c["loss"], abs=1e-14), c["name"]
        if "lse" in c:
            np.testing.assert_allclose(f["lse"], c["lse"], rtol=0, atol=1e-14)
        if "dH" in c:
            np.testing.assert_allclose(b["dH"], c["dH"], rtol=0, atol=1e-14)
        if "dW" in c:
            np.testing.assert_allclose(b["dW"], c["dW"], rtol=0, atol=1e-14)


# ---------------------------------------------------------------- P1 uniform logits
@pytest.mark.parametrize("reduction", ["mean", "sum"])
def test_uniform_logits_closed_form(reduction):
    """P1: W = 0 -> z = 0 -> lse = ln V, L = ln V (mean) or N_v ln V (sum),
    dH = 0 and dW_j = c((1/V) sum_valid h_i - sum_{i: y_i = j} h_i)."""
    N, D, V = 40, 6, 17
    H, _, y = rand_problem(N, D, V, 1)
    W = np.zeros((V, D))
    valid = y != IGNORE_INDEX
    nv = int(valid.sum())
    f = lce_forward(H, W, y, reduction=reduction)
    b = lce_backward(H, W, y, reduction=reduction)
    assert np.allclose(f["lse"][valid], math.log(V), rtol=0, atol=1e-14)
    assert np.all(f["lse"][~valid] == 0)
    expect = math.log(V) if reduction == "mean" else nv * math.log(V)
    assert f["loss"] == pytest.approx(expect, rel=1e-14)
    assert np.all(b["dH"] == 0)
    c = 1.0 / nv if reduction == "mean" else 1.0
    dW = np.zeros((V, D))
    hsum = H[valid].sum(axis=0)
    for j in range(V):
        dW[j] = c * (hsum / V - H[valid & (y == j)].sum(axis=0))
    np.testing.assert_allclose(b["dW"], dW, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- P2 row sums
def test_softmax_minus_onehot_rows_sum_to_zero():
    """P2: sum_j G_ij = 0, so the vocab-column sum of dW vanishes and
    dH = G W is unchanged by adding a common vector to every W row (P6)."""
    H, W, y = rand_problem(64, 8, 50, 2)
    b = lce_backward(H, W, y)
    col = b["dW"].sum(axis=0)
    assert np.abs(col).max() < 1e-14 * max(1.0, np.abs(b["dW"]).max() * 50)


def test_bilinear_identity_between_dH_and_dW():
    """P11: z = H W^T is bilinear, so <H, dH> = sum_ij G_ij z_ij = <W, dW>."""
    H, W, y = rand_problem(70, 9, 40, 25)
    b = lce_backward(H, W, y, reduction="sum")
    assert (H * b["dH"]).sum() == pytest.approx((W * b["dW"]).sum(), rel=1e-12)


# ---------------------------------------------------------------- P3 ignore rows
def test_ignored_rows_never_touch_the_projection():
    """P3 / P:166 mask-first: NaN/Inf garbage in ignored rows of H changes
    nothing, ignored rows get lse = loss = 0 and dH rows exactly 0."""
    H, W, y = rand_problem(50, 8, 30, 3, ignore_frac=0.3)
    ign = y == IGNORE_INDEX
    assert ign.any()
    f0 = lce_forward(H, W, y)
    b0 = lce_backward(H, W, y)
    Hg = H.copy()
    Hg[ign] = np.nan
    Hg[np.flatnonzero(ign)[0]] = np.inf
    f1 = lce_forward(Hg, W, y)
    b1 = lce_backward(Hg, W, y)
    assert f1["loss"] == f0["loss"]
    np.testing.assert_array_equal(f1["lse"], f0["lse"])
    np.testing.assert_array_equal(b1["dW"], b0["dW"])
    assert np.all(b1["dH"][ign] == 0)
    assert np.all(f1["lse"][ign] == 0) and np.all(f1["token_loss"][ign] == 0)
    assert f0["n_valid"] == int((~ign).sum())


# ---------------------------------------------------------------- P4 finite differences
def _fd_check(H, W, y, reduction, entries_H, entries_W, tol=1e-6):
    b = lce_backward(H, W, y, reduction=reduction)

    def L(Hx, Wx):
        return lce_forward(Hx, Wx, y, reduction=reduction)["loss"]

    for (i, k) in entries_H:
        eps = 1e-6 * max(1.0, abs(H[i, k]))
        Hp, Hm = H.copy(), H.copy()
        Hp[i, k] += eps
        Hm[i, k] -= eps
        fd = (L(Hp, W) - L(Hm, W)) / (2 * eps)
        assert abs(fd - b["dH"][i, k]) <= tol * max(1.0, abs(fd)), ("dH", i, k, fd, b["dH"][i, k])
    for (j, k) in entries_W:
        eps = 1e-6 * max(1.0, abs(W[j, k]))
        Wp, Wm = W.copy(), W.copy()
        Wp[j, k] += eps
        Wm[j, k] -= eps
        fd = (L(H, Wp) - L(H, Wm)) / (2 * eps)
        assert abs(fd - b["dW"][j, k]) <= tol * max(1.0, abs(fd)), ("dW", j, k, fd, b["dW"][j, k])


@pytest.mark.parametrize("reduction", ["mean", "sum"])
def test_finite_differences_all_entries_small(reduction):
    """P4: every entry of dH and dW at N=8, D=4, V=7 vs central differences."""
    H, W, y = rand_problem(8, 4, 7, 4, ignore_frac=0.25)
    eH = [(i, k) for i in range(8) for k in range(4)]
    eW = [(j, k) for j in range(7) for k in range(4)]
    _fd_check(H, W, y, reduction, eH, eW)


def test_finite_differences_sampled_tiny_config():
    """P4 at the BASELINE tiny shape (N=256, D=64, V=1000, 10% ignored):
    200+ random entries including ignored rows (whose gradient must be 0)."""
    H, W, y = rand_problem(256, 64, 1000, 5, ignore_frac=0.1)
    rng = np.random.default_rng(0)
    eH = [(int(rng.integers(256)), int(rng.integers(64))) for _ in range(120)]
    ign = np.flatnonzero(y == IGNORE_INDEX)
    eH += [(int(i), 3) for i in ign[:10]]
    eW = [(int(rng.integers(1000)), int(rng.integers(64))) for _ in range(80)]
    eW += [(int(y[0]) if y[0] >= 0 else 0, 1)]
    _fd_check(H, W, y, "mean", eH, eW, tol=1e-5)


# ---------------------------------------------------------------- P5 closed forms
def test_two_class_softplus_and_sigmoid():
    """P5: V = 2 -> l = softplus(z_other - z_target), dz_other = c sigma(.)."""
    H, W, y = rand_problem(30, 5, 2, 6, ignore_frac=0.0)
    z = H @ W.T
    t = z[np.arange(30), y]
    o = z[np.arange(30), 1 - y]
    d = o - t
    sp = np.log1p(np.exp(d))
    f = lce_forward(H, W, y, reduction="sum")
    assert f["loss"] == pytest.approx(sp.sum(), rel=1e-13)
    b = lce_backward(H, W, y, reduction="sum")
    sig = 1 / (1 + np.exp(-d))
    # dH_i = sig_i (w_other - w_target)
    dH = sig[:, None] * (W[1 - y] - W[y])
    np.testing.assert_allclose(b["dH"], dH, rtol=1e-12, atol=1e-14)


def test_single_class_is_zero():
    """P5 / S:272: V = 1 -> loss 0, gradients 0."""
    H, _, _ = rand_problem(10, 3, 1, 7, ignore_frac=0.0)
    W = np.array([[0.3, -2.0, 1.0]])
    y = np.zeros(10, dtype=np.int64)
    assert lce_forward(H, W, y)["loss"] == 0.0
    b = lce_backward(H, W, y)
    assert np.abs(b["dH"]).max() == 0 and np.abs(b["dW"]).max() == 0


# ---------------------------------------------------------------- P6 shift invariance
def test_shift_invariance():
    """P6: W_j <- W_j + u for all j adds h_i.u to every logit of row i;
    loss and dH are unchanged."""
    H, W, y = rand_problem(40, 6, 25, 8)
    u = np.random.default_rng(1).standard_normal(6)
    f0, f1 = lce_forward(H, W, y), lce_forward(H, W + u, y)
    b0, b1 = lce_backward(H, W, y), lce_backward(H, W + u, y)
    assert f1["loss"] == pytest.approx(f0["loss"], rel=1e-12)
    np.testing.assert_allclose(b1["dH"], b0["dH"], rtol=0, atol=1e-12)


# ---------------------------------------------------------------- P7 permutations
def test_vocab_and_token_permutation():
    """P7: relabelling the vocab permutes dW rows; permuting tokens permutes
    lse and dH rows; the loss is invariant under both."""
    H, W, y = rand_problem(40, 6, 25, 9)
    rng = np.random.default_rng(2)
    pi = rng.permutation(25)           # new row pi[j] holds old row j
    Wp = np.empty_like(W)
    Wp[pi] = W
    yp = np.where(y == IGNORE_INDEX, y, pi[np.where(y == IGNORE_INDEX, 0, y)])
    f0, f1 = lce_forward(H, W, y), lce_forward(H, Wp, yp)
    b0, b1 = lce_backward(H, W, y), lce_backward(H, Wp, yp)
    assert f1["loss"] == pytest.approx(f0["loss"], rel=1e-13)
    np.testing.assert_allclose(b1["dW"][pi], b0["dW"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(b1["dH"], b0["dH"], rtol=0, atol=1e-13)
    sig = rng.permutation(40)
    f2 = lce_forward(H[sig], W, y[sig])
    b2 = lce_backward(H[sig], W, y[sig])
    assert f2["loss"] == pytest.approx(f0["loss"], rel=1e-13)
    np.testing.assert_allclose(f2["lse"], f0["lse"][sig], rtol=0, atol=1e-13)
    np.testing.assert_allclose(b2["dH"], b0["dH"][sig], rtol=0, atol=1e-13)


# ---------------------------------------------------------------- P8 additivity
def test_sum_is_additive_over_row_splits_and_mean_is_sum_over_nvalid():
    """P8: SUM loss and dW add over any row split; MEAN = SUM / N_v."""
    H, W, y = rand_problem(60, 5, 20, 10)
    fa = lce_forward(H[:23], W, y[:23], reduction="sum")
    fb = lce_forward(H[23:], W, y[23:], reduction="sum")
    f = lce_forward(H, W, y, reduction="sum")
    assert f["loss"] == pytest.approx(fa["loss"] + fb["loss"], rel=1e-13)
    ba = lce_backward(H[:23], W, y[:23], reduction="sum")
    bb = lce_backward(H[23:], W, y[23:], reduction="sum")
    b = lce_backward(H, W, y, reduction="sum")
    np.testing.assert_allclose(b["dW"], ba["dW"] + bb["dW"], rtol=0, atol=1e-13)
    fm = lce_forward(H, W, y, reduction="mean")
    assert fm["loss"] == pytest.approx(f["loss"] / f["n_valid"], rel=1e-14)
    bm = lce_backward(H, W, y, reduction="mean")
    np.testing.assert_allclose(bm["dH"], b["dH"] / f["n_valid"], rtol=1e-13, atol=1e-16)


def test_grad_loss_scales_gradients():
    """R11: the upstream scalar g multiplies both gradients."""
    H, W, y = rand_problem(20, 4, 9, 11)
    b1 = lce_backward(H, W, y)
    b3 = lce_backward(H, W, y, grad_loss=-2.5)
    np.testing.assert_allclose(b3["dH"], -2.5 * b1["dH"], rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(b3["dW"], -2.5 * b1["dW"], rtol=1e-13, atol=1e-16)


# ---------------------------------------------------------------- P9 large logits
def test_spike_construction_exact():
    """P9: every non-target logit at z_t - delta gives
    l = ln(1 + (V - 1) e^{-delta}) exactly, even with logits ~ 1e3."""
    V, D, delta = 13, 2, 3.0
    # h = (1, 0); W_j = (base, 0) for non-targets and (base + delta, 0) for target
    base = 1000.0
    W = np.zeros((V, D))
    W[:, 0] = base
    y = np.array([4, 4])
    W[4, 0] = base + delta
    H = np.array([[1.0, 0.0], [1.0, 0.0]])
    f = lce_forward(H, W, y, reduction="mean")
    assert f["loss"] == pytest.approx(math.log1p((V - 1) * math.exp(-delta)), rel=1e-13)
    assert np.isfinite(lce_backward(H * 100, W, y)["dW"]).all()


def test_one_large_competitor():
    """P9: one non-target at z_t + delta, the rest far below: l ~ ln(1 + e^delta)."""
    V, delta = 9, 40.0
    W = np.zeros((V, 2))
    W[:, 0] = -500.0
    W[2, 0] = 10.0
    W[5, 0] = 10.0 + delta
    H = np.array([[1.0, 0.0]])
    f = lce_forward(H, W, np.array([2]), reduction="sum")
    assert f["loss"] == pytest.approx(math.log1p(math.exp(delta)), rel=1e-13)


# ---------------------------------------------------------------- P10 library routine
@pytest.mark.parametrize("reduction", ["mean", "sum"])
def test_matches_torch_cross_entropy_fp64(reduction):
    """P10: CE(H W^T, y) via torch.nn.functional.cross_entropy on CPU fp64
    plus torch.autograd (P:132 drop-in for the standard CE)."""
    H, W, y = rand_problem(96, 16, 300, 12, ignore_frac=0.15)
    Ht = torch.tensor(H, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    loss = torch.nn.functional.cross_entropy(Ht @ Wt.T, torch.tensor(y), ignore_index=IGNORE_INDEX,
                                             reduction=reduction)
    loss.backward()
    f = lce_forward(H, W, y, reduction=reduction)
    b = lce_backward(H, W, y, reduction=reduction)
    assert f["loss"] == pytest.approx(loss.item(), rel=1e-12)
    np.testing.assert_allclose(b["dH"], Ht.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(b["dW"], Wt.grad.numpy(), rtol=1e-10, atol=1e-14)
    tl = torch.nn.functional.cross_entropy(torch.tensor(H) @ torch.tensor(W).T, torch.tensor(y),
                                           ignore_index=IGNORE_INDEX, reduction="none")
    np.testing.assert_allclose(f["token_loss"], tl.numpy(), rtol=1e-12, atol=1e-14)
    lse = torch.logsumexp(torch.tensor(H) @ torch.tensor(W).T, dim=1).numpy()
    valid = y != IGNORE_INDEX
    np.testing.assert_allclose(f["lse"][valid], lse[valid], rtol=1e-13)


# ---------------------------------------------------------------- edge cases / errors
def test_zero_valid_rows_and_empty_input():
    """R2 / S:303: N_v = 0 (and N = 0) -> loss 0, zero gradients (torch gives NaN)."""
    H, W, _ = rand_problem(5, 3, 4, 13)
    y = np.full(5, IGNORE_INDEX)
    for red in ("mean", "sum"):
        assert lce_forward(H, W, y, reduction=red)["loss"] == 0.0
        b = lce_backward(H, W, y, reduction=red)
        assert not b["dH"].any() and not b["dW"].any()
    e = lce_forward(np.zeros((0, 3)), W, np.zeros(0, dtype=np.int64))
    assert e["loss"] == 0.0 and e["n_valid"] == 0


def test_label_errors():
    """R4 / S:268-270: labels outside [0, V) other than ignore_index raise;
    an ignore_index inside [0, V) is honoured as ignore (R3)."""
    H, W, y = rand_problem(6, 3, 5, 14, ignore_frac=0.0)
    for bad in (5, -1, 10 ** 6):
        yb = y.copy()
        yb[2] = bad
        with pytest.raises(ValueError):
            lce_forward(H, W, yb)
        with pytest.raises(ValueError):
            lce_backward(H, W, yb)
    y2 = y.copy()
    y2[:3] = 1
    f = lce_forward(H, W, y2, ignore_index=1)
    assert f["n_valid"] == int((y2 != 1).sum())
    assert np.all(f["lse"][y2 == 1] == 0)
    with pytest.raises(ValueError):
        lce_forward(H, W, y, reduction="avg")


# ---------------------------------------------------------------- row-local helper
def test_rows_helper_matches_full_oracle():
    """lce_rows (used for sampled checks at full size) equals the full oracle rows."""
    H, W, y = rand_problem(70, 9, 40, 15)
    f = lce_forward(H, W, y)
    b = lce_backward(H, W, y)
    rows = np.array([0, 5, 69, 33, 5])
    r = lce_rows(H, W, y, rows, n_valid=f["n_valid"])
    np.testing.assert_array_equal(r["lse"], f["lse"][rows])
    np.testing.assert_allclose(r["token_loss"], f["token_loss"][rows], rtol=1e-15, atol=0)
    np.testing.assert_allclose(r["dH"], b["dH"][rows], rtol=1e-13, atol=1e-17)


# ---------------------------------------------------------------- loss-parallel decomposition
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_vocab_shard_statistics_combine_to_global(P):
    """P:180 loss parallel: per-shard (max, sum-exp, target logit) merged by
    M = max m_r, S = sum s_r e^{m_r - M} reproduce the unsharded lse/loss,
    including uneven shards (ceil(V/P) rows, last rank shorter)."""
    N, D, V = 48, 7, 1000
    H, W, y = rand_problem(N, D, V, 16)
    Vl = -(-V // P)
    stats = []
    for r in range(P):
        a, b = r * Vl, min(V, (r + 1) * Vl)
        stats.append(shard_stats(H, W[a:b], y, a, V))
    comb = combine_shard_stats(stats)
    f = lce_forward(H, W, y)
    np.testing.assert_allclose(comb["lse"], f["lse"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(comb["token_loss"], f["token_loss"], rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------------- reduction "none" (R21)
def test_none_reduction_matches_torch_per_token_and_vector_grad():
    """R21 / P10: per-token losses equal torch CE(reduction='none'); the
    gradient of sum_i g_i loss_i equals torch autograd with grad vector g."""
    H, W, y = rand_problem(80, 12, 200, 17, ignore_frac=0.2)
    g = np.random.default_rng(3).standard_normal(80)
    Ht = torch.tensor(H, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    lv = torch.nn.functional.cross_entropy(Ht @ Wt.T, torch.tensor(y), ignore_index=IGNORE_INDEX,
                                           reduction="none")
    lv.backward(torch.tensor(g))
    f = lce_forward(H, W, y, reduction="none")
    b = lce_backward(H, W, y, reduction="none", grad_loss=g)
    np.testing.assert_allclose(f["token_loss"], lv.detach().numpy(), rtol=1e-12, atol=1e-14)
    assert f["loss"] == pytest.approx(lv.sum().item(), rel=1e-12)
    np.testing.assert_allclose(b["dH"], Ht.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(b["dW"], Wt.grad.numpy(), rtol=1e-10, atol=1e-14)
    rows = np.array([1, 7, 40])
    r = lce_rows(H, W, y, rows, n_valid=f["n_valid"], reduction="none", grad_loss=g)
    np.testing.assert_allclose(r["dH"], b["dH"][rows], rtol=1e-13, atol=1e-16)


def test_none_with_uniform_weights_is_mean():
    """P8 for R21: g_i = 1/N_v on every token reproduces the MEAN gradients."""
    H, W, y = rand_problem(50, 6, 30, 18)
    nv = int((y != IGNORE_INDEX).sum())
    bn = lce_backward(H, W, y, reduction="none", grad_loss=np.full(50, 1.0 / nv))
    bm = lce_backward(H, W, y, reduction="mean")
    np.testing.assert_allclose(bn["dH"], bm["dH"], rtol=1e-13, atol=1e-17)
    np.testing.assert_allclose(bn["dW"], bm["dW"], rtol=1e-13, atol=1e-17)


# ---------------------------------------------------------------- AdamW (Sec. 4.1)
def test_adamw_spec_examples():
    """S:357 decay-only step (g = 0, wd = 0.01, lr = 2e-5 from App. D) and the
    scalar first step theta = g = 1, betas (0.9, 0.999), wd = 0, hand-derived:
    m = 0.1, v = 0.001, m_hat = v_hat = 1 -> theta' = 1 - lr / (1 + eps)."""
    from oracle import adamw_step

    th, m, v = adamw_step(np.array([3.0, -1.5]), np.zeros(2), np.zeros(2), np.zeros(2), step=1, lr=2e-5,
                          weight_decay=0.01)
    np.testing.assert_allclose(th, np.array([3.0, -1.5]) * (1 - 2e-7), rtol=1e-15)
    assert not m.any() and not v.any()
    th, m, v = adamw_step(np.array([1.0]), np.array([1.0]), np.zeros(1), np.zeros(1), step=1, lr=1e-3)
    assert m[0] == pytest.approx(0.1, rel=1e-15) and v[0] == pytest.approx(0.001, rel=1e-12)
    assert th[0] == pytest.approx(1 - 1e-3 / (1 + 1e-8), rel=1e-14)


def test_adamw_matches_torch_fp64_multi_step():
    """P10-style library pin: torch.optim.AdamW (CPU, fp64) over 5 steps."""
    from oracle import adamw_step

    rng = np.random.default_rng(4)
    th0 = rng.standard_normal((7, 5))
    p = torch.nn.Parameter(torch.tensor(th0))
    opt = torch.optim.AdamW([p], lr=3e-3, betas=(0.9, 0.95), eps=1e-6, weight_decay=0.1)
    th, m, v = th0.copy(), np.zeros_like(th0), np.zeros_like(th0)
    for t in range(1, 6):
        g = rng.standard_normal((7, 5))
        p.grad = torch.tensor(g)
        opt.step()
        th, m, v = adamw_step(th, g, m, v, t, lr=3e-3, beta1=0.9, beta2=0.95, eps=1e-6, weight_decay=0.1)
    np.testing.assert_allclose(th, p.detach().numpy(), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(m, opt.state[p]["exp_avg"].numpy(), rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(v, opt.state[p]["exp_avg_sq"].numpy(), rtol=1e-13, atol=1e-18)


# ---------------------------------------------------------------- KD loss (NEXT-4, R23)
def _kd_problem(seed, N=40, Ds=6, Dt=9, V=23):
    rng = np.random.default_rng(seed)
    Hs, Ws = rng.standard_normal((N, Ds)), rng.standard_normal((V, Ds)) / math.sqrt(Ds)
    Ht, Wt = rng.standard_normal((N, Dt)), rng.standard_normal((V, Dt)) / math.sqrt(Dt)
    y = rng.integers(0, V, size=N)
    y[rng.permutation(N)[:7]] = IGNORE_INDEX
    return Hs, Ws, Ht, Wt, y


def test_kd_teacher_equals_student():
    """Same head for teacher and student: l_i = entropy of p_S and dz = p_S - p_T = 0."""
    from oracle import kd_backward, kd_forward

    Hs, Ws, _, _, y = _kd_problem(20)
    f = kd_forward(Hs, Ws, Hs, Ws, y)
    z = Hs @ Ws.T
    p = np.exp(z - z.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    ent = -(p * np.log(p)).sum(1)
    valid = y != IGNORE_INDEX
    np.testing.assert_allclose(f["token_loss"][valid], ent[valid], rtol=1e-12)
    b = kd_backward(Hs, Ws, Hs, Ws, y)
    assert np.abs(b["dH"]).max() < 1e-15 and np.abs(b["dW"]).max() < 1e-15


def test_kd_uniform_teacher_closed_form():
    """W_T = 0: p_T uniform, l_i = lse_S(i) - mean_j z_S(i, j)."""
    from oracle import kd_forward

    Hs, Ws, Ht, Wt, y = _kd_problem(21)
    f = kd_forward(Hs, Ws, Ht, np.zeros_like(Wt), y, reduction="sum")
    z = Hs @ Ws.T
    lse = np.log(np.exp(z).sum(1))
    valid = y != IGNORE_INDEX
    assert f["loss"] == pytest.approx((lse - z.mean(1))[valid].sum(), rel=1e-13)


def test_kd_one_hot_teacher_is_cross_entropy():
    """A teacher sharply peaked on y_i (spike Delta = 60) reduces KD to the CE
    of the student (up to e^-60)."""
    from oracle import kd_forward

    Hs, Ws, _, _, y = _kd_problem(22)
    N, V = len(y), Ws.shape[0]
    Ht = np.eye(N)                       # one teacher feature per token
    Wt = np.zeros((V, N))
    for i, lab in enumerate(y):
        if lab != IGNORE_INDEX:
            Wt[lab, i] = 60.0
    f = kd_forward(Hs, Ws, Ht, Wt, y)
    ce = lce_forward(Hs, Ws, y)
    assert f["loss"] == pytest.approx(ce["loss"], rel=1e-12)


@pytest.mark.parametrize("reduction", ["mean", "sum"])
def test_kd_matches_torch_fp64(reduction):
    """P10-style: -(softmax(z_T) * log_softmax(z_S)).sum(-1) over non-ignored
    rows with torch autograd (CPU fp64) for the student gradients."""
    from oracle import kd_backward, kd_forward

    Hs, Ws, Ht, Wt, y = _kd_problem(23)
    hs = torch.tensor(Hs, requires_grad=True)
    ws = torch.tensor(Ws, requires_grad=True)
    zt = torch.tensor(Ht) @ torch.tensor(Wt).T
    per = -(torch.softmax(zt, -1) * torch.log_softmax(hs @ ws.T, -1)).sum(-1)
    mask = torch.tensor(y != IGNORE_INDEX)
    L = per[mask].sum() / (mask.sum() if reduction == "mean" else 1)
    L.backward()
    f = kd_forward(Hs, Ws, Ht, Wt, y, reduction=reduction)
    b = kd_backward(Hs, Ws, Ht, Wt, y, reduction=reduction)
    assert f["loss"] == pytest.approx(L.item(), rel=1e-12)
    np.testing.assert_allclose(b["dH"], hs.grad.numpy(), rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(b["dW"], ws.grad.numpy(), rtol=1e-10, atol=1e-15)


def test_kd_finite_differences():
    """P4 for KD: every student gradient entry at a tiny shape."""
    from oracle import kd_backward, kd_forward

    Hs, Ws, Ht, Wt, y = _kd_problem(24, N=6, Ds=3, Dt=4, V=5)
    b = kd_backward(Hs, Ws, Ht, Wt, y)
    for arr, grad, name in ((Hs, b["dH"], "H"), (Ws, b["dW"], "W")):
        for idx in np.ndindex(arr.shape):
            eps = 1e-6 * max(1.0, abs(arr[idx]))
            ap, am = arr.copy(), arr.copy()
            ap[idx] += eps
            am[idx] -= eps
            if name == "H":
                fp, fm = kd_forward(ap, Ws, Ht, Wt, y)["loss"], kd_forward(am, Ws, Ht, Wt, y)["loss"]
            else:
                fp, fm = kd_forward(Hs, ap, Ht, Wt, y)["loss"], kd_forward(Hs, am, Ht, Wt, y)["loss"]
            fd = (fp - fm) / (2 * eps)
            assert abs(fd - grad[idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx)


# ---------------------------------------------------------------- full-size dW helper (sampled vocab rows)
@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
def test_dweight_rows_matches_torch_autograd_fp64(reduction):
    """P10 for lce_dweight_rows / lce_lse (the full-size dW check of the GPU
    tests): selected rows of dW and every row's lse equal torch's CPU fp64
    cross_entropy + autograd, including vocab rows nobody is labelled with,
    rows that are labels, the last row, and a repeated row."""
    H, W, y = rand_problem(90, 7, 41, 31, ignore_frac=0.2)
    g = np.linspace(-1.0, 2.0, 90) if reduction == "none" else 0.75
    J = np.array([0, 40, 40, int(y[y != IGNORE_INDEX][0]), 17, 3])
    o = lce_dweight_rows(H, W, y, J, reduction=reduction, grad_loss=g)
    Ht = torch.tensor(H)
    Wt = torch.tensor(W, requires_grad=True)
    yt = torch.tensor(y)
    loss = torch.nn.functional.cross_entropy(Ht @ Wt.T, yt, ignore_index=IGNORE_INDEX, reduction=reduction)
    if reduction == "none":
        loss.backward(torch.tensor(g))
    else:
        (loss * g).backward()
    np.testing.assert_allclose(o["dW_rows"], Wt.grad.numpy()[J], rtol=1e-12, atol=1e-14)
    lse_t = torch.logsumexp(Ht @ torch.tensor(W).T, dim=1).numpy()
    valid = y != IGNORE_INDEX
    np.testing.assert_allclose(o["lse"][valid], lse_t[valid], rtol=1e-13, atol=0)
    assert np.all(o["lse"][~valid] == 0)


def test_dweight_rows_finite_differences_and_closed_form():
    """P4 + P1 for lce_dweight_rows: central differences of the oracle loss
    in W_jk for the selected rows; with W = 0 (uniform logits) the closed
    form dW_j = c((1/V) sum_valid h_i - sum_{y_i = j} h_i); block size of the
    lse pass (host RAM only) changes nothing."""
    H, W, y = rand_problem(30, 5, 13, 32, ignore_frac=0.2)
    J = np.array([2, 12, int(y[y != IGNORE_INDEX][1])])
    o = lce_dweight_rows(H, W, y, J)
    for a, j in enumerate(J):
        for k in range(5):
            eps = 1e-6
            Wp, Wm = W.copy(), W.copy()
            Wp[j, k] += eps
            Wm[j, k] -= eps
            fd = (lce_forward(H, Wp, y)["loss"] - lce_forward(H, Wm, y)["loss"]) / (2 * eps)
            assert abs(fd - o["dW_rows"][a, k]) <= 1e-7 * max(1.0, abs(fd))
    np.testing.assert_array_equal(lce_lse(H, W, y, block=7), lce_lse(H, W, y))
    Z = np.zeros_like(W)
    valid = y != IGNORE_INDEX
    nv = int(valid.sum())
    oz = lce_dweight_rows(H, Z, y, np.arange(13))
    for j in range(13):
        expect = (H[valid].sum(axis=0) / 13 - H[valid & (y == j)].sum(axis=0)) / nv
        np.testing.assert_allclose(oz["dW_rows"][j], expect, rtol=0, atol=1e-14)
    assert np.allclose(oz["lse"][valid], math.log(13), rtol=0, atol=1e-14)
