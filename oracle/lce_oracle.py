"""Plain, slow, obviously-correct fp64 CPU oracle of the linear cross-entropy loss.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path.

What it computes (PAPER.md = P, SPEC.md = S, line numbers of /root/reference):

* P:166 (Sec. 4.2, "Linear Cross-Entropy loss"): LinearCrossEntropyLoss "fuses
  the final output projection with the cross-entropy computation, masks ignored
  tokens before projection, and processes hidden states in chunks so that the
  dense [B, S, V] tensor is never materialized".
* P:132 (Sec. 3.3): LCE is a one-line drop-in for the standard CE, so its
  result is by definition CE(H W^T, y).  S:279 states the same contract
  ("match cross_entropy(hidden.W^T, targets)").

LCE therefore reaches exactly (up to rounding order) a result with a plain
definition, and this oracle IS that definition written out in fp64 (numpy,
BLAS dgemm for the two products).  Chunking is a memory technique, not
semantics (reading R7), so the oracle does not chunk.  It projects
only the non-ignored rows (mask-first), which is also what makes
garbage in ignored rows harmless.

Readings of points the paper leaves open (full list in DESIGN.md):
  R1 mean divides by N_v = #non-ignored rows
  R2 N_v = 0 -> loss 0, grads 0
  R3 ignore_index default -100; a label equal to it is ignored
  R4 any other label outside [0, V) is an error
  R5 lse / per-token loss of ignored rows are 0
  R6 natural log
  R11 upstream gradient g (dL/dloss) scales the gradients; default 1
  R21 reduction "none" (per-token log-probs, the interface GRPO / DPO need,
      P:322, Table 4): loss_i is the result, `loss` is their sum, and
      the upstream gradient is a per-token vector g_i

Every function is pinned in tests/test_oracle.py against closed forms, brute
force, finite differences and torch's CPU fp64 cross-entropy + autograd.
"""

from __future__ import annotations

import numpy as np

IGNORE_INDEX = -100  # S:498 "ignore_index = -100 -- conventional sentinel"

__all__ = [
    "IGNORE_INDEX",
    "lce_forward",
    "lce_backward",
    "lce_rows",
    "lce_lse",
    "lce_dweight_rows",
    "shard_stats",
    "shard_backward",
    "combine_shard_stats",
    "adamw_step",
    "kd_forward",
    "kd_backward",
]


def _as_f64(a) -> np.ndarray:
    """Exact widening of the inputs (bf16/fp32 values are exactly representable)."""
    return np.asarray(a, dtype=np.float64)


def _valid_rows(y: np.ndarray, vocab: int, ignore_index: int) -> np.ndarray:
    """Step 1 ("masks ignored tokens"): V = {i : y_i != ignore_index}.

    Labels outside [0, V) that are not ignore_index are an error.
    """
    y = np.asarray(y, dtype=np.int64)
    valid = y != ignore_index
    bad = valid & ((y < 0) | (y >= vocab))
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        raise ValueError(f"label {int(y[i])} at row {i} outside [0, {vocab})")
    return valid


def _scale(reduction: str, n_valid: int, grad_loss, rows=None):
    """c = g (sum) or g / N_v (mean); 0 if N_v = 0.
    For "none" (R21) the per-row scale g_i of the selected valid rows."""
    if reduction not in ("mean", "sum", "none"):
        raise ValueError(f"reduction must be 'mean', 'sum' or 'none', got {reduction!r}")
    if reduction == "none":
        if grad_loss is None or np.ndim(grad_loss) == 0:
            g = 1.0 if grad_loss is None else float(grad_loss)
            return np.full(0 if rows is None else len(rows), g)
        return np.asarray(grad_loss, dtype=np.float64)[rows]
    g = 1.0 if grad_loss is None else float(grad_loss)
    if n_valid == 0:
        return 0.0
    return g / n_valid if reduction == "mean" else g


def _log_softmax_stats(z: np.ndarray):
    """Per-row m = max_j z_ij and lse_i = m_i + ln sum_j exp(z_ij - m_i)."""
    m = z.max(axis=1)
    lse = m + np.log(np.exp(z - m[:, None]).sum(axis=1))
    return m, lse


def lce_forward(hidden, weight, labels, ignore_index: int = IGNORE_INDEX,
                reduction: str = "mean") -> dict:
    """Loss, per-token lse and per-token loss of CE(H W^T, y), mask-first.

    hidden [N, D], weight [V, D], labels [N] ints.  Returns a dict with
    ``loss`` (float), ``lse`` [N] (0 on ignored rows), ``token_loss`` [N]
    (0 on ignored rows) and ``n_valid`` (int).
    """
    H = _as_f64(hidden)
    W = _as_f64(weight)
    y = np.asarray(labels, dtype=np.int64)
    N, V = H.shape[0], W.shape[0]
    valid = _valid_rows(y, V, ignore_index)           # step 1
    rows = np.flatnonzero(valid)
    n_valid = int(rows.size)
    lse = np.zeros(N)
    tok = np.zeros(N)
    if n_valid:
        z = H[rows] @ W.T                             # step 2: logits of valid rows only
        _, lse_v = _log_softmax_stats(z)              # step 3
        z_t = z[np.arange(n_valid), y[rows]]
        lse[rows] = lse_v
        tok[rows] = lse_v - z_t                       # step 4: NLL of log-softmax
    total = float(tok.sum())                          # step 5
    if reduction == "mean":
        loss = total / n_valid if n_valid else 0.0    # R1, R2
    elif reduction in ("sum", "none"):                # "none": token_loss is the result (R21)
        loss = total
    else:
        raise ValueError(f"reduction must be 'mean', 'sum' or 'none', got {reduction!r}")
    return {"loss": loss, "lse": lse, "token_loss": tok, "n_valid": n_valid}


def lce_backward(hidden, weight, labels, ignore_index: int = IGNORE_INDEX,
                 reduction: str = "mean", grad_loss=1.0) -> dict:
    """Analytic gradients of the loss: dH = G W, dW = G^T H.

    G_ij = c (softmax(z_i)_j - [j = y_i]) for valid rows, 0 for ignored rows,
    with c from ``_scale`` (for "none": c_i = grad_loss[i], a length-N vector).
    Returns ``dH`` [N, D], ``dW`` [V, D] (fp64), ``n_valid`` and ``c``.
    """
    H = _as_f64(hidden)
    W = _as_f64(weight)
    y = np.asarray(labels, dtype=np.int64)
    N, V = H.shape[0], W.shape[0]
    valid = _valid_rows(y, V, ignore_index)
    rows = np.flatnonzero(valid)
    n_valid = int(rows.size)
    c = _scale(reduction, n_valid, grad_loss, rows)    # step 7
    dH = np.zeros_like(H)
    dW = np.zeros_like(W)
    if n_valid:
        Hv = H[rows]
        z = Hv @ W.T
        _, lse = _log_softmax_stats(z)
        G = np.exp(z - lse[:, None])                   # step 8: p_ij
        G[np.arange(n_valid), y[rows]] -= 1.0          #         p - onehot
        G *= c if np.ndim(c) == 0 else c[:, None]
        dH[rows] = G @ W                               # step 9
        dW = G.T @ Hv
    return {"dH": dH, "dW": dW, "n_valid": n_valid, "c": c}


def lce_rows(hidden, weight, labels, rows, n_valid: int,
             ignore_index: int = IGNORE_INDEX, reduction: str = "mean",
             grad_loss=1.0) -> dict:
    """Row-local quantities for selected rows only (lse, token loss, dH rows).

    Used to check the GPU at sizes where the full oracle is too slow: lse_i,
    l_i and dH_i depend only on row i, W, and (for dH) the scalar c, which
    needs the global ``n_valid``.  Ignored rows give 0.
    """
    W = _as_f64(weight)
    rows = np.asarray(rows, dtype=np.int64)
    H = _as_f64(np.asarray(hidden)[rows])
    y = np.asarray(labels, dtype=np.int64)[rows]
    V = W.shape[0]
    valid = _valid_rows(y, V, ignore_index)
    k = rows.size
    sel = np.flatnonzero(valid)
    c = _scale(reduction, n_valid, grad_loss, rows[sel])
    lse = np.zeros(k)
    tok = np.zeros(k)
    dH = np.zeros((k, W.shape[1]))
    if sel.size:
        z = H[sel] @ W.T
        _, l = _log_softmax_stats(z)
        lse[sel] = l
        tok[sel] = l - z[np.arange(sel.size), y[sel]]
        G = np.exp(z - l[:, None])
        G[np.arange(sel.size), y[sel]] -= 1.0
        dH[sel] = (c if np.ndim(c) == 0 else c[:, None]) * (G @ W)
    return {"lse": lse, "token_loss": tok, "dH": dH}


def lce_lse(hidden, weight, labels, ignore_index: int = IGNORE_INDEX, block: int = 1024) -> np.ndarray:
    """Steps 1-3 for every row: lse_i = m_i + ln sum_j exp(z_ij - m_i) with
    z_i = W h_i over the full vocabulary, 0 on ignored rows (R5).

    Rows are taken ``block`` at a time only to bound host RAM (a [block, V]
    fp64 logit slab); every row is still the textbook formula on its own.
    """
    W = _as_f64(weight)
    hidden = np.asarray(hidden)
    y = np.asarray(labels, dtype=np.int64)
    valid = _valid_rows(y, W.shape[0], ignore_index)
    rows = np.flatnonzero(valid)
    lse = np.zeros(y.shape[0])
    for a in range(0, rows.size, block):
        r = rows[a:a + block]
        _, lse[r] = _log_softmax_stats(_as_f64(hidden[r]) @ W.T)
    return lse


def lce_dweight_rows(hidden, weight, labels, vocab_rows, ignore_index: int = IGNORE_INDEX,
                     reduction: str = "mean", grad_loss=1.0, lse=None) -> dict:
    """Selected rows j of dW = G^T H (step 9) without forming all of G:

        dW_j = sum_{i valid} c_i (exp(z_ij - lse_i) - [y_i = j]) h_i,   z_ij = h_i . w_j

    which needs only the logit columns z[:, J] and each valid row's lse
    (``lce_lse``, the oracle's own, unless the caller passes an oracle-made
    one).  Used to check the GPU's dW at full size, where the whole oracle
    backward would not fit in host memory; the cost is dominated by lse
    (2 N_v V D flops).  Returns ``dW_rows`` [len(J), D] and ``lse`` [N].
    """
    H = np.asarray(hidden)
    W = _as_f64(weight)
    y = np.asarray(labels, dtype=np.int64)
    J = np.asarray(vocab_rows, dtype=np.int64)
    valid = _valid_rows(y, W.shape[0], ignore_index)
    rows = np.flatnonzero(valid)
    n_valid = int(rows.size)
    c = _scale(reduction, n_valid, grad_loss, rows)
    if lse is None:
        lse = lce_lse(H, W, y, ignore_index)
    dW = np.zeros((J.size, W.shape[1]))
    if n_valid:
        Hv = _as_f64(H[rows])
        P = np.exp(Hv @ W[J].T - np.asarray(lse, dtype=np.float64)[rows][:, None])  # p_ij, j in J
        P -= (y[rows][:, None] == J[None, :])                                           # - onehot
        P *= c if np.ndim(c) == 0 else c[:, None]
        dW = P.T @ Hv
    return {"dW_rows": dW, "lse": np.asarray(lse, dtype=np.float64)}


def shard_stats(hidden, weight_shard, labels, vocab_start: int, vocab_total: int,
                ignore_index: int = IGNORE_INDEX) -> dict:
    """Per-row statistics of one vocab shard (loss-parallel).

    P:180: the output projection is sharded "over the vocab dimension across
    the tensor parallelism mesh".  Shard r holds rows [vocab_start,
    vocab_start + V_r) of W and computes, for each valid row i, the partial
    max m_ir, sum-exp s_ir = sum_{j in shard} exp(z_ij - m_ir) and the target
    logit z_{i,y_i} if y_i is in the shard (else 0).  Ignored rows give
    (m, s, z) = (-inf, 0, 0).
    """
    H = _as_f64(hidden)
    Wr = _as_f64(weight_shard)
    y = np.asarray(labels, dtype=np.int64)
    N = H.shape[0]
    valid = _valid_rows(y, vocab_total, ignore_index)
    rows = np.flatnonzero(valid)
    m = np.full(N, -np.inf)
    s = np.zeros(N)
    zt = np.zeros(N)
    if rows.size:
        z = H[rows] @ Wr.T
        mr = z.max(axis=1)
        m[rows] = mr
        s[rows] = np.exp(z - mr[:, None]).sum(axis=1)
        local = y[rows] - vocab_start
        own = (local >= 0) & (local < Wr.shape[0])
        zt[rows[own]] = z[np.flatnonzero(own), local[own]]
    return {"m": m, "s": s, "z_target": zt, "valid": valid}


def shard_backward(hidden, weight_shard, labels, vocab_start: int, lse, c: float,
                   ignore_index: int = IGNORE_INDEX) -> dict:
    """Gradient contributions of one vocab shard given the global lse.

    With G_r the shard's columns of G = c (softmax - onehot):
    dH = sum_r G_r W_r (summed across shards) and dW rows of the shard = G_r^T H.
    """
    H = _as_f64(hidden)
    Wr = _as_f64(weight_shard)
    y = np.asarray(labels, dtype=np.int64)
    lse = np.asarray(lse, dtype=np.float64)
    rows = np.flatnonzero(y != ignore_index)
    dH = np.zeros_like(H)
    dW = np.zeros_like(Wr)
    if rows.size:
        z = H[rows] @ Wr.T
        G = np.exp(z - lse[rows][:, None])
        local = y[rows] - vocab_start
        own = np.flatnonzero((local >= 0) & (local < Wr.shape[0]))
        G[own, local[own]] -= 1.0
        G *= c
        dH[rows] = G @ Wr
        dW = G.T @ H[rows]
    return {"dH_partial": dH, "dW_shard": dW}


def kd_forward(hidden_s, weight_s, hidden_t, weight_t, labels, ignore_index: int = IGNORE_INDEX,
               reduction: str = "mean") -> dict:
    """Linear knowledge-distillation loss (forward KL), fp64 -- NEXT-4.

    P:35 (Fig. 1 objective box: "SFT CE / LCE / DPO / KD") and P:125-126
    ("knowledge distillation with dedicated KD losses") name the objective but
    give no formula.  Reading R23 (torchtune's forward-KL convention): for rows
    with labels != ignore_index,
        l_i = - sum_j p_T(i, j) log p_S(i, j) = lse_S(i) - sum_j p_T(i, j) z_S(i, j),
    z_S = H_S W_S^T (student), z_T = H_T W_T^T (teacher), p = softmax; mean
    over N_v or sum.  Label values are not used, only the ignore mask.
    """
    Hs, Ws, Ht, Wt = (_as_f64(a) for a in (hidden_s, weight_s, hidden_t, weight_t))
    y = np.asarray(labels, dtype=np.int64)
    N = Hs.shape[0]
    rows = np.flatnonzero(y != ignore_index)
    nv = int(rows.size)
    tok = np.zeros(N)
    lse_s = np.zeros(N)
    lse_t = np.zeros(N)
    if nv:
        zs = Hs[rows] @ Ws.T
        zt = Ht[rows] @ Wt.T
        _, ls = _log_softmax_stats(zs)
        _, lt = _log_softmax_stats(zt)
        pt = np.exp(zt - lt[:, None])
        tok[rows] = ls - (pt * zs).sum(axis=1)
        lse_s[rows] = ls
        lse_t[rows] = lt
    total = float(tok.sum())
    if reduction == "mean":
        loss = total / nv if nv else 0.0
    elif reduction in ("sum", "none"):
        loss = total
    else:
        raise ValueError(reduction)
    return {"loss": loss, "token_loss": tok, "lse_s": lse_s, "lse_t": lse_t, "n_valid": nv}


def kd_backward(hidden_s, weight_s, hidden_t, weight_t, labels, ignore_index: int = IGNORE_INDEX,
                reduction: str = "mean", grad_loss=1.0) -> dict:
    """Student gradients of ``kd_forward``: dz_S = c (p_S - p_T); dH_S = dz_S W_S,
    dW_S = dz_S^T H_S (the teacher gets none)."""
    Hs, Ws, Ht, Wt = (_as_f64(a) for a in (hidden_s, weight_s, hidden_t, weight_t))
    y = np.asarray(labels, dtype=np.int64)
    rows = np.flatnonzero(y != ignore_index)
    nv = int(rows.size)
    c = _scale(reduction, nv, grad_loss, rows)
    dH = np.zeros_like(Hs)
    dW = np.zeros_like(Ws)
    if nv:
        zs = Hs[rows] @ Ws.T
        zt = Ht[rows] @ Wt.T
        _, ls = _log_softmax_stats(zs)
        _, lt = _log_softmax_stats(zt)
        G = np.exp(zs - ls[:, None]) - np.exp(zt - lt[:, None])
        G *= c if np.ndim(c) == 0 else c[:, None]
        dH[rows] = G @ Ws
        dW = G.T @ Hs[rows]
    return {"dH": dH, "dW": dW, "n_valid": nv}


def adamw_step(theta, grad, exp_avg, exp_avg_sq, step: int, lr: float, beta1: float = 0.9,
               beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0):
    """One AdamW update in fp64 (the torch.optim.AdamW convention).

    Sec. 4.1: the in-backward optimizer applies exactly this per
    parameter as soon as its gradient is final.  Decoupled decay first:
    theta <- theta (1 - lr wd); m <- b1 m + (1 - b1) g; v <- b2 v + (1 - b2) g^2;
    theta <- theta - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps).
    Returns (theta, m, v) as new arrays.
    """
    th = _as_f64(theta) * (1.0 - lr * weight_decay)
    g = _as_f64(grad)
    m = beta1 * _as_f64(exp_avg) + (1.0 - beta1) * g
    v = beta2 * _as_f64(exp_avg_sq) + (1.0 - beta2) * g * g
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    th = th - lr * (m / bc1) / (np.sqrt(v / bc2) + eps)
    return th, m, v


def combine_shard_stats(stats: list) -> dict:
    """Merge shard statistics into the global lse and per-token loss.

    M_i = max_r m_ir;  lse_i = M_i + ln sum_r s_ir exp(m_ir - M_i);
    z_{i,y_i} = sum_r z_ir (exactly one shard owns the label);
    l_i = lse_i - z_{i,y_i}.  Ignored rows (all m = -inf) give 0.
    """
    m = np.stack([st["m"] for st in stats])
    s = np.stack([st["s"] for st in stats])
    zt = np.stack([st["z_target"] for st in stats]).sum(axis=0)
    valid = stats[0]["valid"]
    M = m.max(axis=0)
    lse = np.zeros(m.shape[1])
    tok = np.zeros(m.shape[1])
    v = np.flatnonzero(valid)
    if v.size:
        w = s[:, v] * np.exp(m[:, v] - M[v])
        lse[v] = M[v] + np.log(w.sum(axis=0))
        tok[v] = lse[v] - zt[v]
    return {"lse": lse, "token_loss": tok}
