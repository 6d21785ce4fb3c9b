/*
 * lce.h -- C ABI of the B200 (sm_100a) linear cross-entropy library (liblce.so).
 *
 * What it computes (PAPER.md = P, /root/reference line numbers):
 *   P:166 (Sec. 4.2 "Linear Cross-Entropy loss"): the loss "fuses the final
 *   output projection with the cross-entropy computation, masks ignored tokens
 *   before projection, and processes hidden states in chunks so that the dense
 *   [B, S, V] tensor is never materialized".  P:132 (Sec. 3.3): it is a drop-in
 *   for the standard CE, i.e. loss = CE(H W^T, y) with ignore_index.
 *   P:169 / P:180 (Sec. 5): under tensor parallelism the output projection is
 *   sharded over the vocabulary ("loss parallel"); see lce_comm_* below.
 *
 * Notation: H = hidden [N, D] bf16, W = weight [V_l, D] bf16 (this rank's
 * vocab rows), y = labels [N] int32, N_v = #{i : y_i != ignore_index},
 * lse_i = ln sum_j exp(z_ij) with z = H W^T (natural log, fp32),
 * loss_i = lse_i - z_{i, y_i}, L = sum_i loss_i (SUM) or sum_i loss_i / N_v
 * (MEAN; 0 when N_v = 0).  Gradients: G_ij = c (softmax(z_i)_j - [j = y_i]),
 * c = g (SUM) or g / N_v (MEAN), dH = G W, dW = G^T H.
 *
 * Conventions for every entry point:
 *  - All tensor pointers are DEVICE pointers unless stated otherwise; all
 *    tensors are dense row-major.  bf16 values are passed as uint16_t bit
 *    patterns.  Every pointer must be 16-byte aligned.
 *  - The caller owns every buffer.  The library never allocates or frees
 *    device memory (the only exception is NCCL state inside an lce_comm_t),
 *    keeps no pointer after return, and never synchronises the stream except
 *    in lce_check_device_status.  All work is enqueued on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Host-detectable errors return before anything is enqueued and leave all
 *    outputs untouched.  CUDA launch errors return LCE_ERR_CUDA.
 *  - Results do not depend on the chunk budget beyond fp32 rounding order.
 *  - Calls on different streams with different workspaces are independent.
 *    (The library image holds one small device-global array, the per-cluster
 *    k-block progress of its persistent wide-tile GEMMs -- the K-lockstep,
 *    DESIGN.md section 5.  It only ever delays a TMA producer, tagged per
 *    launch; GEMMs running concurrently on other streams can make a gate
 *    time out, which costs time, never results.)
 */
#ifndef LCE_H_
#define LCE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: lce_comm_init_mode / lce_comm_mode (token-parallel communicators) and
 *    lce_profile_read_clocks; n_valid reports the global N_v in token mode.
 * 3: dweight_flags (LCE_DW_ACCUMULATE | LCE_DW_BF16) replace accumulate_dweight
 *    (0 / 1 keep their meaning) and dweight is void*; lce_expect_grad,
 *    lce_comm_check; LCE_ERR_ARG, LCE_ERR_UPSTREAM. */
#define LCE_ABI_VERSION 3

typedef enum {
  LCE_OK = 0,
  LCE_ERR_NULL = 1,        /* required pointer is NULL                         */
  LCE_ERR_SHAPE = 2,       /* N<0, D<=0, D%8!=0, V_l<=0, bad vocab range, >2^31 */
  LCE_ERR_ALIGN = 3,       /* a pointer is not 16-byte aligned                 */
  LCE_ERR_REDUCTION = 4,   /* reduction is not LCE_MEAN / LCE_SUM / LCE_NONE   */
  LCE_ERR_WORKSPACE = 5,   /* workspace_bytes < lce_workspace_bytes(problem)   */
  LCE_ERR_LABEL_RANGE = 6, /* a label outside [0, V_total) that is not ignored */
  LCE_ERR_DEVICE = 7,      /* current device is not sm_100 (B200)              */
  LCE_ERR_CUDA = 8,        /* a CUDA runtime / driver call failed              */
  LCE_ERR_NCCL = 9,        /* NCCL missing or an NCCL call failed              */
  LCE_ERR_COMM = 10,       /* communicator does not match the problem          */
  LCE_ERR_ARG = 11,        /* unsupported flag combination                     */
  LCE_ERR_UPSTREAM = 12    /* upstream gradient differs from the one the fused
                              call assumed (see lce_expect_grad)               */
} lce_status_t;

/* dweight_flags of the backward entry points (a bit set).
 *  LCE_DW_ACCUMULATE: dweight += dW instead of dweight = dW (fp32 only;
 *    gradient accumulation).
 *  LCE_DW_BF16: dweight is bf16 [V_l, D] (RNE from the fp32 GEMM accumulator,
 *    written once) instead of fp32.  lce_backward only -- its dW row blocks
 *    are final when they leave the tensor memory; the fused / KD paths sum dW
 *    over row chunks in fp32 and return LCE_ERR_ARG for it, as does
 *    LCE_DW_BF16 | LCE_DW_ACCUMULATE. */
enum { LCE_DW_ACCUMULATE = 1, LCE_DW_BF16 = 2 };

/* MEAN: L = sum_i loss_i / N_v.  SUM: L = sum_i loss_i.
 * NONE (per-token, the log-prob interface GRPO/DPO need -- P:322, P:463,
 * Table 4): the forward's token_loss = -log p(y_i | h_i) is the result and
 * `loss` receives sum_i loss_i; the backward's grad_loss is a [N] vector of
 * per-token upstream gradients g_i = dL/dloss_i (NULL = all ones), so
 * G_ij = g_i (softmax(z_i)_j - [j = y_i]). */
typedef enum { LCE_MEAN = 0, LCE_SUM = 1, LCE_NONE = 2 } lce_reduction_t;

/* Opaque communicator (NCCL over NVLink).  NULL = one GPU. */
typedef struct lce_comm_s* lce_comm_t;

/* How a communicator partitions the problem (north star):
 *  LCE_PAR_VOCAB (lce_comm_init): W sharded by contiguous row blocks
 *    (vocab_start, vocab_local); every rank passes the same hidden / labels;
 *    the row statistics and dH are all-reduced, dW stays local (the rank's
 *    shard).  loss, lse, dH are the global ones on every rank.
 *  LCE_PAR_TOKEN (lce_comm_init_mode): W replicated (vocab_local ==
 *    vocab_total), each rank passes its own rows (N may differ per rank).
 *    Only two scalars are exchanged: the non-ignored count (MEAN divides by
 *    the global N_v in the loss and in the gradient scale) and the loss, which
 *    is the full batch's on every rank.  lse / token_loss / dhidden are the
 *    rank's own rows; dweight is the rank's contribution, i.e. the sum over
 *    ranks of dweight is the full batch's dW -- reduce it with the
 *    data-parallel gradient reduction (e.g. FSDP's reduce-scatter).
 *    n_valid reports the global N_v.  lce_backward_adamw needs the full dW
 *    and returns LCE_ERR_COMM with a token-parallel communicator.  Every rank
 *    must make the same calls (the scalar exchanges are collectives), also a
 *    rank whose N is 0. */
typedef enum { LCE_PAR_VOCAB = 0, LCE_PAR_TOKEN = 1 } lce_parallel_t;

typedef struct {
  int64_t n_tokens;      /* N >= 0                                                  */
  int64_t hidden_dim;    /* D > 0, D % 8 == 0 (16-byte TMA row pitch)               */
  int64_t vocab_local;   /* V_l > 0: rows of `weight` on this rank (= V if 1 GPU)   */
  int64_t vocab_start;   /* global id of local weight row 0 (0 on one GPU)          */
  int64_t vocab_total;   /* V: labels must lie in [0, V) unless ignored             */
  int32_t ignore_index;  /* rows with this label are dropped before projection      */
  int32_t reduction;     /* lce_reduction_t                                         */
  int64_t chunk_budget_bytes; /* bytes of the bounded chunk buffer; 0 = default:
                                 lce_backward: 32768 vocab columns of bf16 G
                                 (2 * ceil256(N) * 32768 bytes) clamped to
                                 [512 MiB, 4 GiB] and never below 4096 columns;
                                 lce_forward_backward: 2 GiB of bf16 q/G rows,
                                 or ceil(N/2) rows (two chunks) when those
                                 take at most 4 GiB; the chunk's N_c x D row
                                 buffers (8 bytes per element) are bounded by
                                 the same budget; KD: 4 GiB.  A performance
                                 knob only.                                      */
} lce_problem_t;

/* Bytes of caller-provided device workspace both lce_forward and lce_backward
 * need for `p` (same value for both).  Pure host function.  Returns 0 if `p`
 * is invalid.  Upper bound is O(N*D + N*V_l/128 + budget) -- never N*V_l. */
size_t lce_workspace_bytes(const lce_problem_t* p);

/* Forward: mask-first compaction, z = H W^T tile by tile on the tensor cores
 * (tcgen05, fp32 accumulation in TMEM), online logsumexp + target pick in the
 * epilogue, fixed-order combine.  The N x V_l logits never exist in memory.
 *   hidden     [N, D]   bf16, row i = token i
 *   weight     [V_l, D] bf16, row j = vocab id vocab_start + j
 *   labels     [N]      int32 global vocab ids or ignore_index
 *   loss       [1] fp32 out: L (NaN if a label was out of range, see below)
 *   lse        [N] fp32 out: lse_i; 0 for ignored rows
 *   token_loss [N] fp32 out or NULL: loss_i; 0 for ignored rows
 *   n_valid    [1] int32 out or NULL: N_v
 *   workspace  device scratch of >= lce_workspace_bytes(p) bytes
 * A label outside [0, V) that is not ignore_index excludes its row from all
 * compute, sets a bit in the workspace status word and makes `loss`
 * NaN (no host sync needed); lce_check_device_status then returns
 * LCE_ERR_LABEL_RANGE.  With comm != NULL every rank passes identical
 * hidden/labels and its own weight shard; loss/lse are then global and
 * bitwise identical on all ranks. */
lce_status_t lce_forward(const lce_problem_t* p, lce_comm_t comm,
                         const uint16_t* hidden, const uint16_t* weight,
                         const int32_t* labels, float* loss, float* lse,
                         float* token_loss, int32_t* n_valid,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Backward: recomputes z tile by tile (same tiling as the forward), forms
 * G = softmax - onehot from the saved lse in the epilogue (bf16 RNE, one
 * bounded vocab chunk at a time), then dH += G_c W_c and dW_c = G_c^T H on
 * the tensor cores with fp32 accumulation.
 *   lse        [N] fp32 in: the forward's lse output (same H, W, labels)
 *   grad_loss  fp32 in (device) or NULL for 1.0: MEAN / SUM: [1], g = dL_total/dL;
 *              NONE: [N], g_i = dL_total/dloss_i (ignored rows' entries unused)
 *   dhidden    [N, D] bf16 out: dH (RNE from fp32); rows of ignored tokens 0
 *   dweight    [V_l, D] fp32 (or bf16 with LCE_DW_BF16) out: dW for this
 *              rank's rows
 *   dweight_flags  0: dweight = dW (fp32); LCE_DW_ACCUMULATE: dweight += dW;
 *              LCE_DW_BF16: bf16 dweight = RNE(dW) (LCE_ERR_ARG with ACCUMULATE)
 * With comm != NULL, dH is summed over ranks (NCCL all-reduce) and is the
 * same on all ranks; dweight is the local shard (concatenate in rank order). */
lce_status_t lce_backward(const lce_problem_t* p, lce_comm_t comm,
                          const uint16_t* hidden, const uint16_t* weight,
                          const int32_t* labels, const float* lse,
                          const float* grad_loss, uint16_t* dhidden,
                          void* dweight, int dweight_flags,
                          void* workspace, size_t workspace_bytes, void* stream);

/* ---- optimizer-in-backward for the LM head (Sec. 4.1) -----------
 * AdamW hyper-parameters (torch.optim.AdamW convention); `step` is
 * the 1-based count of this update (bias corrections 1 - beta^step). */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  int64_t step;
} lce_adamw_t;

/* lce_backward whose dW is consumed by an AdamW step inside the dW GEMM
 * epilogue, the moment each dW row block is final ("the gradient can then be
 * released without being retained"): no dW buffer exists.
 *   weight        [V_l, D] bf16 in/out: read by the GEMMs, then rewritten as
 *                 bf16(master_weight) row block by row block (each block is
 *                 rewritten only after every GEMM that reads it)
 *   master_weight [V_l, D] fp32 in/out (theta); exp_avg / exp_avg_sq [V_l, D]
 *                 fp32 in/out (m, v)
 * Other arguments as lce_backward.  The result equals lce_backward (dW) then
 * one AdamW step on (master_weight, dW) -- P:147's K = 1 equivalence.
 * LCE_ERR_SHAPE for hyper-parameters outside their domain. */
lce_status_t lce_backward_adamw(const lce_problem_t* p, lce_comm_t comm,
                                const uint16_t* hidden, uint16_t* weight,
                                const int32_t* labels, const float* lse,
                                const float* grad_loss, uint16_t* dhidden,
                                float* master_weight, float* exp_avg,
                                float* exp_avg_sq, const lce_adamw_t* hp,
                                void* workspace, size_t workspace_bytes,
                                void* stream);

/* ---- fused forward + backward ----------------------------------------------
 * The same results as lce_forward followed by lce_backward (loss, lse,
 * token_loss, n_valid, dhidden, dweight; same argument meanings), computed
 * without recomputing the logits: P:166's "processes hidden states in
 * chunks" taken literally -- for each chunk of Nc compacted rows the
 * forward epilogue keeps q = exp(z - m_tile) in bf16 (z = H_c W^T in fp32,
 * m_tile the row max over its 256-column tile; in the workspace, Nc x V_l x 2
 * bytes, never N x V_l), the rows are reduced to lse, q is turned into G in
 * place and consumed by the dH and dW GEMMs: 6 N_v V D flops instead of 8.
 * The upstream gradient must be known up front (grad_loss as in lce_backward;
 * NULL = 1; lce_expect_grad checks an autograd caller's actual one later).
 * dW is accumulated across row chunks in fp32 (dweight_flags: 0 or
 * LCE_DW_ACCUMULATE; LCE_DW_BF16 -> LCE_ERR_ARG).  Nc is set by
 * chunk_budget_bytes (bytes of the bf16 chunk buffer; 0 = 2 GiB, raised to
 * ceil(N/2) rows when those take at most 4 GiB) and is at
 * most half the rows, so the buffer never holds all N x V_l probabilities.
 * With a vocab-parallel comm each row chunk's (max, sum-exp, target
 * logit) are combined with the same MAX / SUM all-reduces as lce_forward, and
 * the chunk's fp32 dH partial is all-reduced on the communicator's side stream
 * while the dW GEMM runs (on SMs left free for it).  With a token-parallel
 * comm see lce_parallel_t. */
size_t lce_fused_workspace_bytes(const lce_problem_t* p);
lce_status_t lce_forward_backward(const lce_problem_t* p, lce_comm_t comm,
                                  const uint16_t* hidden, const uint16_t* weight,
                                  const int32_t* labels, const float* grad_loss,
                                  float* loss, float* lse, float* token_loss,
                                  int32_t* n_valid, uint16_t* dhidden, float* dweight,
                                  int dweight_flags, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ---- linear knowledge distillation (NEXT-4) ----------------
 * Forward KL of a teacher head against a student head, both projected and
 * reduced chunk by chunk like lce_forward_backward (neither N x V logit matrix
 * exists):  l_i = -sum_j p_T(i,j) log p_S(i,j) = lse_S(i) - sum_j p_T(i,j) z_S(i,j)
 * for rows with labels[i] != ignore_index (label values are only a mask),
 * z_S = H_S W_S^T, z_T = H_T W_T^T, reductions as lce_problem_t.reduction.
 * Student gradients dz_S = s_i (p_S - p_T):  dhidden_s = dz_S W_S (bf16),
 * dweight_s = dz_S^T H_S (fp32; dweight_flags 0 or LCE_DW_ACCUMULATE); the
 * teacher gets none.
 *   p->hidden_dim = D_S, teacher_dim = D_T (% 8 == 0); hidden_s [N, D_S],
 *   weight_s [V, D_S], hidden_t [N, D_T], weight_t [V, D_T] (bf16);
 *   grad_loss / loss / token_loss / n_valid as lce_forward_backward.
 * With comm != NULL both heads are vocab-sharded alike (weight_s / weight_t
 * hold rows [vocab_start, vocab_start + V_l)): lse_S and lse_T are combined
 * with MAX / SUM all-reduces, sum_j p_T z_S with a SUM all-reduce, and the
 * chunk's dH_S partial is all-reduced as in lce_forward_backward. */
size_t lce_kd_workspace_bytes(const lce_problem_t* p, int64_t teacher_dim);
lce_status_t lce_kd_forward_backward(const lce_problem_t* p, lce_comm_t comm, int64_t teacher_dim,
                                     const uint16_t* hidden_s, const uint16_t* weight_s,
                                     const uint16_t* hidden_t, const uint16_t* weight_t,
                                     const int32_t* labels, const float* grad_loss,
                                     float* loss, float* token_loss, int32_t* n_valid,
                                     uint16_t* dhidden_s, float* dweight_s,
                                     int dweight_flags, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* Synchronises `stream`, reads the status word of `workspace` and returns
 * LCE_ERR_LABEL_RANGE if the most recent lce_forward / lce_backward /
 * lce_forward_backward / KD call that used this workspace saw a bad label
 * (under token parallelism: a bad label on ANY rank, so every rank reports
 * it), else LCE_ERR_UPSTREAM if lce_expect_grad saw a mismatch since that
 * call, else LCE_OK.  Every compute call rewrites the status word, so a fresh
 * (uninitialised) workspace needs no clearing. */
lce_status_t lce_check_device_status(void* workspace, void* stream);

/* For callers (e.g. an autograd function) that ran lce_forward_backward with
 * an assumed upstream gradient `expected` (the grad_loss it passed, 1 if NULL)
 * and later receive the actual one as a device scalar `grad` [1] fp32: one
 * tiny kernel compares them on the device (no host synchronisation) and, if
 * they differ, sets a bit in the status word of `workspace` (the one the
 * fused call used) so that lce_check_device_status returns LCE_ERR_UPSTREAM:
 * the gradients already produced are then for the wrong scale.  Nothing is
 * rescaled. */
lce_status_t lce_expect_grad(const float* grad, float expected, void* workspace, void* stream);

/* ---- communicator (vocab-parallel P:180 loss parallel, or token-parallel) --
 * Rank 0 creates a 128-byte id (host memory) and distributes it out of band
 * (the Python binding uses torch.distributed.broadcast_object_list); every
 * rank then calls lce_comm_init with its own CUDA device current.  NCCL is
 * loaded at run time (libnccl.so.2); LCE_ERR_NCCL if unavailable. */
lce_status_t lce_comm_get_unique_id(uint8_t id[128]);
lce_status_t lce_comm_init(lce_comm_t* comm, const uint8_t id[128], int nranks, int rank);
/* lce_comm_init with an explicit lce_parallel_t mode (lce_comm_init = VOCAB). */
lce_status_t lce_comm_init_mode(lce_comm_t* comm, const uint8_t id[128], int nranks, int rank, int mode);
lce_status_t lce_comm_destroy(lce_comm_t comm);
int lce_comm_size(lce_comm_t comm);
int lce_comm_rank(lce_comm_t comm);
int lce_comm_mode(lce_comm_t comm); /* lce_parallel_t; LCE_PAR_VOCAB for NULL */
/* NVLS (environment LCE_NVLS=1, vocab-parallel communicators): the dH
 * partials are added by the dH GEMM's epilogue into an NVSwitch multicast
 * buffer owned by the communicator (multimem.red.add; the switch sums the
 * ranks), replacing the NCCL dH all-reduce, its side stream and the SMs held
 * back for it.  The first call per problem size sets the buffer up
 * (cuMulticastCreate / AddDevice / BindMem, host-synchronous, collective over
 * the communicator); LCE_ERR_DEVICE if any rank's device or driver offers no
 * multicast objects.  dH is then not bitwise reproducible (in-switch order).
 * LCE_NVLS=2 runs the same sequence on a unicast buffer (one rank; tests). */

/* Polls ncclCommGetAsyncError: LCE_ERR_NCCL if the communicator hit an
 * asynchronous error (a peer died, a network failure) -- the collectives of
 * the calls above would otherwise block forever -- LCE_OK otherwise (also for
 * NULL).  Host-only, no synchronisation; call it from a watchdog loop. */
lce_status_t lce_comm_check(lce_comm_t comm);

/* ---- introspection ------------------------------------------------------- */
const char* lce_status_string(lce_status_t s);
int lce_abi_version(void);
/* Total number of CUDA kernels this library has launched since load. */
uint64_t lce_launch_count(void);

/* NVTX: every lce_forward / lce_backward / lce_backward_adamw /
 * lce_forward_backward / lce_kd_forward_backward call is an NVTX range of
 * that name, and every kernel launch inside it a nested range named by its
 * step (the class names below: "S1+S2 forward GEMM + LSE", "S5 dW GEMM", ...).
 * Header-only NVTX3: free unless a tool is attached (e.g. ncu --nvtx
 * --nvtx-include "lce_forward_backward/").                                  */

/* Kernel classes for the profiler below. */
typedef enum {
  LCE_K_PREP = 0,     /* S0 label scan + stable compaction          */
  LCE_K_GATHER = 1,   /* S0 gather of valid rows of H (+ lse rows)  */
  LCE_K_FWD = 2,      /* S1+S2 forward GEMM + online-LSE epilogue   */
  LCE_K_COMBINE = 3,  /* S3 merge of per-tile partials, loss        */
  LCE_K_BWD_G = 4,    /* S4 recompute GEMM + G epilogue             */
  LCE_K_BWD_DH = 5,   /* S6 dH GEMM                                 */
  LCE_K_BWD_DW = 6,   /* S5 dW GEMM                                 */
  LCE_K_FINAL = 7,    /* S7 dH cast/scatter (multi-GPU)             */
  LCE_K_COMM = 8,     /* NCCL collectives                           */
  LCE_K_COUNT = 9
} lce_kernel_class_t;

/* Opt-in per-kernel timing: while enabled, every launch is bracketed by CUDA
 * events on the launching stream (no extra synchronisation).  lce_profile_read
 * synchronises the recorded events and returns, per lce_kernel_class_t, the
 * summed device milliseconds and launch counts since lce_profile_enable(1);
 * it then clears the record.  Host-thread-global; not for concurrent use. */
lce_status_t lce_profile_enable(int on);
lce_status_t lce_profile_read(double ms[LCE_K_COUNT], int64_t launches[LCE_K_COUNT]);
/* As lce_profile_read, plus for the GEMM classes the SM clock each launch ran
 * at: CTA 0 of every profiled GEMM launch records (%globaltimer, clock64) when
 * its mainloop starts and ends; sm_cycles / sm_ns are the summed differences
 * per class (their ratio is the mean SM clock inside the step, which the
 * power cap sets).  Any output pointer may be NULL.  Clears the record. */
lce_status_t lce_profile_read_clocks(double ms[LCE_K_COUNT], int64_t launches[LCE_K_COUNT],
                                     double sm_cycles[LCE_K_COUNT], double sm_ns[LCE_K_COUNT]);

/* ---- diagnostics (tests only) ---------------------------------------------
 * C[M, N] (fp32, row-major, ldc = N) = A * B^T through the same tcgen05 GEMM
 * mainloop the loss kernels use.  a_mn = 0: A stored [M, K] (K-major);
 * a_mn = 1: A stored [K, M] (M-major).  b_mn = 0: B stored [N, K];
 * b_mn = 1: B stored [K, N].  M, N, K > 0; leading dims are the stored row
 * lengths and must be multiples of 8. */
lce_status_t lce_debug_gemm(const uint16_t* A, const uint16_t* B, float* C,
                            int64_t M, int64_t N, int64_t K, int a_mn, int b_mn,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LCE_H_ */
