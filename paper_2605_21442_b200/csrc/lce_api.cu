// lce_api.cu -- C ABI of liblce.so (include/lce.h): argument validation,
// workspace planning, TMA descriptor encoding, launch sequencing, the
// vocab-parallel NCCL layer and the opt-in kernel profiler.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/lce.h"
#include "kernels.cuh"
#include "nccl.h"

using namespace lce;

namespace {

// ------------------------------------------------------------------ helpers
constexpr int64_t kDefaultChunkBudget = 512ll << 20;
std::atomic<uint64_t> g_launches{0};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

#define LCE_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      if (getenv("LCE_DEBUG")) fprintf(stderr, "lce: %s -> %s\n", #expr, cudaGetErrorString(e_)); \
      return LCE_ERR_CUDA;                                                               \
    }                                                                                    \
  } while (0)

#define LCE_TRY(expr)                  \
  do {                                 \
    lce_status_t st_ = (expr);         \
    if (st_ != LCE_OK) return st_;     \
  } while (0)

// ------------------------------------------------------------------ workspace plan
struct Plan {
  int64_t N, D, Vl, cap, n_tiles, Vc, n_chunks, nblocks;
  size_t hdr, idx, yc, zt, lsec, gsc, bsum, mloc, mglob, sbuf, hc, region, pm, ps, g, dh, total;
};

bool make_plan(const lce_problem_t* p, Plan* pl) {
  if (!p) return false;
  const int64_t N = p->n_tokens, D = p->hidden_dim, Vl = p->vocab_local;
  if (N < 0 || D <= 0 || (D % 8) != 0 || Vl <= 0) return false;
  if (p->vocab_start < 0 || p->vocab_total <= 0 || p->vocab_start + Vl > p->vocab_total) return false;
  if (N >= (1ll << 31) - 256 || D >= (1ll << 31) || p->vocab_total >= (1ll << 31)) return false;
  Plan q{};
  q.N = N;
  q.D = D;
  q.Vl = Vl;
  q.cap = round_up(N > 0 ? N : 1, kPairBM);  // whole 256-row pair tiles (G rows are written per tile)
  q.n_tiles = ceil_div(Vl, BN);
  // Default G chunk: 32768 vocab columns, as bytes clamped to [512 MiB, 4 GiB],
  // and never fewer than 4096 columns.  Every chunk adds into the fp32 dH
  // accumulator (8 N D bytes through the L2) against 6 N V_c D flops of GEMMs,
  // and has its own GEMM tails, so wide chunks pay (8B: 32768 columns = 1 GiB
  // ran 2% faster than 16384 for +0.54 GB of peak HBM); for ~1M-token
  // contexts (App. A) the 4 GiB cap and the 4096-column floor bound the chunk.
  int64_t budget = p->chunk_budget_bytes;
  if (budget <= 0) {
    budget = q.cap * 2 * 32768;
    budget = budget < kDefaultChunkBudget ? kDefaultChunkBudget : (budget > (4ll << 30) ? (4ll << 30) : budget);
    if (budget < q.cap * 2 * 4096) budget = q.cap * 2 * 4096;
  }
  int64_t vc = (budget / (q.cap * 2)) / BN * BN;
  if (vc < BN) vc = BN;
  if (vc > round_up(Vl, BN)) vc = round_up(Vl, BN);
  q.Vc = vc;
  q.n_chunks = ceil_div(Vl, vc);
  q.nblocks = ceil_div(q.cap, kRowsPerCta);  // combine: one warp per row
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = static_cast<size_t>(round_up(static_cast<int64_t>(off + bytes), 1024));
    return o;
  };
  q.hdr = take(sizeof(Header));
  q.idx = take(q.cap * 4);
  q.yc = take(q.cap * 4);
  q.zt = take(q.cap * 4);
  q.lsec = take(q.cap * 4);
  q.gsc = take(q.cap * 4);
  q.bsum = take(q.nblocks * 8);
  q.mloc = take(q.cap * 4);
  q.mglob = take(q.cap * 4);
  q.sbuf = take(q.cap * 8);  // [s | z_t copy]: one SUM all-reduce of both
  q.hc = take(static_cast<size_t>(q.cap * D * 2));
  q.region = off;
  const size_t fwd = static_cast<size_t>(2 * q.n_tiles * q.cap * 4) + 1024;
  q.pm = q.region;
  q.ps = q.region + static_cast<size_t>(round_up(q.n_tiles * q.cap * 4, 1024));
  q.g = q.region;
  q.dh = q.region + static_cast<size_t>(round_up(q.cap * q.Vc * 2, 1024));
  const size_t bwd = (q.dh - q.region) + static_cast<size_t>(q.cap * D * 4);
  q.total = q.region + (fwd > bwd ? fwd : bwd);
  *pl = q;
  return true;
}

// Fused fwd+bwd (lce_forward_backward): row chunks of Nc compacted tokens keep
// q = exp(z - m_tile) in bf16 [Nc, ldv], turned into G in place (R24): 2 bytes
// per element bounded by the budget (default 2 GiB), never N x V_l.  The KD
// path keeps fp32 logits for student and teacher (see KdPlan).
constexpr int64_t kDefaultFusedBudget = 2ll << 30;
constexpr int64_t kDefaultKdBudget = 4ll << 30;
constexpr int64_t kTwoChunkBudget = 4ll << 30;
// Workspace sizes are host-pure, so the plan assumes a full B200 (148 SMs) when
// it reserves the dH split-K slabs; at launch the split factor and tile shape
// are re-derived from the current device's SM count (fit_plan_to_device),
// capped by the slab space reserved here.
constexpr int kPlanSms = 148;
// dH / dW GEMMs use 512 x 256 wide pair tiles when the token rows they reduce
// over (the fused row chunk, or all tokens in the recompute path) number at
// least this many: shorter k-ranges leave the epilogue of the wide kernel's
// single accumulator exposed (measured: DESIGN.md section 5)
constexpr int64_t kWideMinRows = 8192;
constexpr int64_t kWideMinDhK = 12288;

struct FusedPlan {
  int64_t N, D, Vl, cap, ldv, n_tiles, Nc, n_chunks;
  int split;                       // split-K factor of the chunk's dH GEMM
  int split_cap;                   // largest split the reserved slab space holds
  int wide_dh, wide_dw;            // 512 x 256 tiles for the chunk's dH / dW GEMMs
  size_t hdr, idx, yc, zt, lsec, gsc, ltok, hc, pm, ps, z, g, slab;
  size_t vmloc, vmglob, vsz, vdh;  // vocab-parallel chunk exchange buffers
  size_t qref, coef, hs, qflag;    // scaled-q mode (R25): per-row reference, dH row factors, scaled H chunk, flags
  bool chunk_hc;                   // CE fused path: H_c holds one row chunk (gathered per chunk), not the batch
  size_t total;
};

// LCE_FUSED_SCALED=0 selects the fused path's tile-max fix-up form (R24).
bool fused_scaled_env() { return !(getenv("LCE_FUSED_SCALED") && atoi(getenv("LCE_FUSED_SCALED")) == 0); }

int use_pair_units(int sms);
int use_wide(int cls, int dflt);
bool use_pair();

// Split-K factor of the fused path's dH GEMM: the smallest split in 1..8 whose
// work items fill the persistent grid's last wave to >= 97% (else the best).
// `max_split` bounds it where the fp32 slabs alias another buffer.
int dh_split(int64_t Nc, int64_t D, int max_split, int sms, int64_t rows) {
  if (const char* e = getenv("LCE_DH_SPLIT")) {  // tuning override
    const int v = atoi(e);
    return v < 1 ? 1 : (v > max_split ? max_split : v);
  }
  const int64_t units = use_pair_units(sms);
  const int64_t tiles = ceil_div(Nc, rows) * ceil_div(D, BN);
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 8 && s <= max_split; ++s) {
    const int64_t items = tiles * s;
    const double eff = static_cast<double>(items) / (ceil_div(items, units) * units);
    if (eff > best_eff + 1e-9) {
      best = s;
      best_eff = eff;
    }
    if (eff >= 0.97) break;
  }
  return best;
}

// Tile shape and split-K factor of a fused row chunk's dH GEMM (and the dW
// tile shape) for a grid of `sms` SMs.
void choose_dh(FusedPlan* q, int max_split, int sms) {
  const int split_wide = dh_split(q->Nc, q->D, max_split, sms, kWideBM);
  q->wide_dh = use_pair() && use_wide(LCE_K_BWD_DH, (q->Nc >= kWideMinRows && q->Vl / split_wide >= kWideMinDhK) ? 1 : 0);
  q->wide_dw = use_pair() && use_wide(LCE_K_BWD_DW, q->Nc >= kWideMinRows ? 1 : 0);
  q->split = dh_split(q->Nc, q->D, max_split, sms, !use_pair() ? BM : (q->wide_dh ? kWideBM : kPairBM));
}

// The plan was made for kPlanSms; re-derive the dH schedule for this device.
void fit_plan_to_device(FusedPlan* q, int sms) {
  if (sms != kPlanSms) choose_dh(q, q->split_cap, sms);
}

// kd: student chunk keeps fp32 Z + bf16 G (6 bytes per element), the dH
// split-K slabs alias Z; otherwise the CE layout above with its own slabs.
bool make_fused_plan(const lce_problem_t* p, FusedPlan* fp, bool kd = false) {
  Plan base;
  if (!make_plan(p, &base)) return false;
  FusedPlan q{};
  q.N = base.N;
  q.D = base.D;
  q.Vl = base.Vl;
  q.cap = base.cap;
  q.ldv = round_up(q.Vl, BN);
  q.n_tiles = ceil_div(q.Vl, BN);
  const int64_t per_elem = kd ? 6 : 2;
  int64_t budget = p->chunk_budget_bytes > 0 ? p->chunk_budget_bytes : kDefaultFusedBudget;
  // Default for CE: the fewest chunks the two-chunk rule allows (N_c = N / 2)
  // while such a chunk stays <= kTwoChunkBudget.  Every non-empty chunk pays a
  // full pass over W in the forward and dH GEMMs and a full fp32 pass over dW
  // (store, then reduce-adds), whatever its row count; with padded batches the
  // valid rows (compacted first) then often fit one chunk (packed Qwen: N_v =
  // 7,177 of 16,384 rows: 5,632 + 1,545-row chunks at 2 GiB, one 8,192-row
  // chunk here, 20.6 -> 18.7 ms per step, +1.5 GB; profiles/round2c_budget.log)
  if (!kd && p->chunk_budget_bytes <= 0) {
    const int64_t half = per_elem * q.ldv * round_up(ceil_div(q.cap, 2), kPairBM);
    if (half > budget && half <= kTwoChunkBudget) budget = half;
  }
  int64_t nc_max = (budget / (per_elem * q.ldv)) / kPairBM * kPairBM;
  // the chunk's row buffers that scale with N_c * D (H_c and the scaled H
  // chunk in bf16, the vocab-parallel fp32 dH chunk: 8 bytes per element) stay
  // within the budget as well -- only binding for small vocabularies (V_l <
  // 4 D), where the q chunk alone would allow very tall chunks
  if (!kd) {
    const int64_t nc_rows = (budget / (8 * q.D)) / kPairBM * kPairBM;
    if (nc_max > nc_rows) nc_max = nc_rows;
  }
  if (nc_max < kPairBM) nc_max = kPairBM;
  if (nc_max > q.cap) nc_max = q.cap;
  // at least two row chunks: the chunk buffer never holds all N x V_l
  // probabilities ("the dense [B, S, V] tensor is never materialized")
  if (q.cap > kPairBM && nc_max > round_up(ceil_div(q.cap, 2), kPairBM)) nc_max = round_up(ceil_div(q.cap, 2), kPairBM);
  q.n_chunks = ceil_div(q.cap, nc_max);
  q.Nc = round_up(ceil_div(q.cap, q.n_chunks), kPairBM);  // balanced chunks
  // wide tiles pay off once a dW work item's K (= the chunk's rows) is long
  // enough to hide the epilogue of the unbuffered accumulator
  // ... and, for dH (K = V_l, split-K), when each work item still reduces over
  // >= kWideMinDhK vocab columns (vocab-parallel shards are short; per-rank 8B
  // step on one GPU, scripts/bench_shard.py: at P = 8 (8,016 columns per item)
  // pair tiles were 5% faster per step, at P = 4 (16,032) and P = 2 (32,064)
  // wide tiles 1-4% faster)
  const int max_split = kd ? static_cast<int>(q.ldv / q.D) : 8;
  choose_dh(&q, max_split, kPlanSms);
  q.split_cap = kd ? max_split : q.split;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = static_cast<size_t>(round_up(static_cast<int64_t>(off + bytes), 1024));
    return o;
  };
  q.hdr = take(sizeof(Header));
  q.idx = take(q.cap * 4);
  q.yc = take(q.cap * 4);
  q.zt = take(q.cap * 4);
  q.lsec = take(q.cap * 4);
  q.gsc = take(q.cap * 4);
  q.ltok = take(q.cap * 4);
  // the CE fused path gathers one row chunk of H at a time (gather_chunk_kernel);
  // KD keeps the batch's compacted rows
  q.chunk_hc = !kd;
  q.hc = take(static_cast<size_t>((q.chunk_hc ? 1 : q.n_chunks) * q.Nc * q.D * 2));
  q.pm = take(static_cast<size_t>(q.n_tiles * q.Nc * 4));
  q.ps = take(static_cast<size_t>(q.n_tiles * q.Nc * 4));
  q.z = kd ? take(static_cast<size_t>(q.Nc * q.ldv * 4)) : 0;
  q.g = take(static_cast<size_t>(q.Nc * q.ldv * 2));
  q.slab = kd ? q.z : take(q.split > 1 ? static_cast<size_t>(q.split * q.Nc * q.D * 4) : 0);
  q.vmloc = take(static_cast<size_t>(q.Nc * 4));
  q.vmglob = take(static_cast<size_t>(q.Nc * 4));
  q.vsz = take(static_cast<size_t>(q.Nc * 8));
  q.vdh = take(static_cast<size_t>(q.Nc * q.D * 4));  // fp32 dH chunk (vocab-parallel only)
  if (!kd) {  // the KD path keeps fp32 logits and never uses the scaled-q form
    q.qref = take(static_cast<size_t>(q.n_chunks * q.Nc * 4));
    q.coef = take(static_cast<size_t>(q.Nc * 4));
    q.hs = take(static_cast<size_t>(q.Nc * q.D * 2));
    q.qflag = take(2 * sizeof(int32_t));
  }
  q.total = off;
  *fp = q;
  return true;
}

// Linear KD (NEXT-4): the fused layout plus the teacher's rows, partials and
// fp32 logit chunk; 10 bytes per chunk element (Z_S, Z_T fp32 + G bf16).
struct KdPlan {
  FusedPlan f;  // student (z = Z_S), G, partials, header/index sections
  int64_t Dt;
  size_t hct, pmt, pst, zt2, lset, total;
};

bool make_kd_plan(const lce_problem_t* p, int64_t teacher_dim, KdPlan* kp) {
  if (teacher_dim <= 0 || teacher_dim % 8 != 0 || teacher_dim >= (1ll << 31)) return false;
  lce_problem_t q = *p;
  // the student plan sized for 10 bytes per element instead of 6
  const int64_t budget = p->chunk_budget_bytes > 0 ? p->chunk_budget_bytes : kDefaultKdBudget;
  q.chunk_budget_bytes = budget * 6 / 10;
  KdPlan k{};
  if (!make_fused_plan(&q, &k.f, true)) return false;
  k.Dt = teacher_dim;
  size_t off = k.f.total;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = static_cast<size_t>(round_up(static_cast<int64_t>(off + bytes), 1024));
    return o;
  };
  k.hct = take(static_cast<size_t>(k.f.n_chunks * k.f.Nc * teacher_dim * 2));
  k.pmt = take(static_cast<size_t>(k.f.n_tiles * k.f.Nc * 4));
  k.pst = take(static_cast<size_t>(k.f.n_tiles * k.f.Nc * 4));
  k.zt2 = take(static_cast<size_t>(k.f.Nc * k.f.ldv * 4));
  k.lset = take(static_cast<size_t>(k.f.cap * 4));
  k.total = off;
  *kp = k;
  return true;
}

// ------------------------------------------------------------------ device / driver
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  });
  return fn;
}

struct DevInfo {
  bool ok;
  int sms;
};

lce_status_t device_info(DevInfo* out) {
  int dev = 0;
  LCE_CUDA(cudaGetDevice(&dev));
  static DevInfo cache[64];
  static bool have[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  // LCE_SMS=n (tests, A/B): run every grid on n < #SMs SMs, as on a partial
  // part (MIG, a reserved slice); the plan's split-K is re-derived for it
  auto limit = [](DevInfo* d) {
    const char* e = getenv("LCE_SMS");
    const int v = e ? atoi(e) : 0;
    if (v >= 2 && v < d->sms) d->sms = v & ~1;
  };
  if (dev < 64 && have[dev]) {
    *out = cache[dev];
    limit(out);
    return out->ok ? LCE_OK : LCE_ERR_DEVICE;
  }
  int major = 0, minor = 0, sms = 0;
  LCE_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  LCE_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  LCE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DevInfo d{major == 10 && minor == 0, sms};
  if (d.ok) {
    // opt in to the dynamic shared memory every GEMM instantiation needs
#define LCE_SMEM_ATTR(A, B, E)                                                                                 \
  LCE_CUDA(cudaFuncSetAttribute(gemm_kernel<A, B, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes)); \
  LCE_CUDA(cudaFuncSetAttribute(gemm_pair_kernel<A, B, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmemBytes)); \
  LCE_CUDA(cudaFuncSetAttribute(gemm_wide_kernel<A, B, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWideSmemBytes))
    LCE_SMEM_ATTR(false, false, EpiLse);
    LCE_SMEM_ATTR(false, false, EpiG);
    LCE_SMEM_ATTR(false, true, EpiDH);
    LCE_SMEM_ATTR(true, true, EpiDW);
    LCE_SMEM_ATTR(true, true, EpiAdamW);
    LCE_SMEM_ATTR(false, false, EpiStore);
    LCE_SMEM_ATTR(false, true, EpiStore);
    LCE_SMEM_ATTR(true, false, EpiStore);
    LCE_SMEM_ATTR(true, true, EpiStore);
    LCE_SMEM_ATTR(false, false, EpiDW);  // lce_debug_gemm under LCE_DEBUG_GEMM_TMA
    LCE_SMEM_ATTR(false, true, EpiDW);
    LCE_SMEM_ATTR(true, false, EpiDW);
#undef LCE_SMEM_ATTR
  }
  if (dev < 64) {
    cache[dev] = d;
    have[dev] = true;
  }
  *out = d;
  limit(out);
  return d.ok ? LCE_OK : LCE_ERR_DEVICE;
}

// 2-D bf16 tensor map over a row-major [rows, inner] array with row pitch
// `pitch` elements, box {64, box_rows}, 128-byte swizzle, zero OOB fill.
lce_status_t encode_map(CUtensorMap* m, const void* base, int64_t inner, int64_t rows, int64_t pitch,
                        int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return LCE_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (getenv("LCE_DEBUG"))
      fprintf(stderr, "lce: cuTensorMapEncodeTiled(%lld x %lld, pitch %lld, box %d) -> %d\n", (long long)inner,
              (long long)rows, (long long)pitch, box_rows, (int)r);
    return LCE_ERR_CUDA;
  }
  return LCE_OK;
}

// fp32 row-major [rows, inner] (pitch `pitch` floats) for TMA stores of
// 32 x 32 boxes (128-byte inner extent, 128-byte swizzle).
lce_status_t map_f32_store(CUtensorMap* m, const void* base, int64_t inner, int64_t rows, int64_t pitch) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return LCE_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch * 4)};
  cuuint32_t box[2] = {32u, 32u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? LCE_OK : LCE_ERR_CUDA;
}

// K-major operand stored [rows, K]: box {64 of K, box_rows}.
lce_status_t map_kmajor(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int64_t pitch, int box_rows) {
  return encode_map(m, base, K, rows, pitch, box_rows);
}
// MN-major operand stored [K, MN]: boxes {64 of MN, BK rows of K}.
lce_status_t map_mnmajor(CUtensorMap* m, const void* base, int64_t K, int64_t MN, int64_t pitch) {
  return encode_map(m, base, MN, K, pitch, BK);
}

// ------------------------------------------------------------------ profiler
struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  int slot;  // clock-probe slot of a GEMM launch, -1 otherwise
};
// clock probes of profiled GEMM launches: {t0 ns, clock0, t1 ns, clock1}
constexpr int kProbeSlots = 4096;
__device__ unsigned long long g_probe[kProbeSlots][4];
struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  int next_slot = 0;
  unsigned long long* probe_base = nullptr;
  // next probe slot (wraps; profile_read is expected well before 4096 GEMMs)
  unsigned long long* take_slot(int* slot) {
    if (!probe_base && cudaGetSymbolAddress(reinterpret_cast<void**>(&probe_base), g_probe) != cudaSuccess) {
      probe_base = nullptr;
      *slot = -1;
      return nullptr;
    }
    *slot = next_slot;
    next_slot = (next_slot + 1) % kProbeSlots;
    return probe_base + 4 * *slot;
  }
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
} g_prof;

// NVTX (header-only NVTX3; a no-op unless a tool such as nsys or ncu
// --nvtx is attached): one range per API call (NvtxCall) and one per kernel
// launch named by its step class (LaunchScope), so a timeline shows S0-S7.
constexpr const char* kClassName[LCE_K_COUNT] = {"S0 prep",         "S0 gather", "S1+S2 forward GEMM + LSE",
                                                 "S3 combine",      "S4 G",      "S6 dH GEMM",
                                                 "S5 dW GEMM",      "S7 dH finalize", "NCCL"};
struct NvtxCall {
  explicit NvtxCall(const char* name) { nvtxRangePushA(name); }
  ~NvtxCall() { nvtxRangePop(); }
  NvtxCall(const NvtxCall&) = delete;
  NvtxCall& operator=(const NvtxCall&) = delete;
};

struct LaunchScope {
  int cls;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  int slot = -1;
  NvtxCall range;
  LaunchScope(int c, cudaStream_t st) : cls(c), s(st), range(kClassName[c]) {
    if (g_prof.on) {
      a = g_prof.get();
      b = g_prof.get();
      cudaEventRecord(a, s);
    }
  }
  // GEMM launches: the clock-probe record for this launch (null when not profiling)
  unsigned long long* probe() { return a ? g_prof.take_slot(&slot) : nullptr; }
  ~LaunchScope() {
    g_launches.fetch_add(cls == LCE_K_COMM ? 0 : 1);
    if (a) {
      cudaEventRecord(b, s);
      g_prof.recs.push_back({cls, a, b, slot});
    }
  }
};

inline lce_status_t last_error() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (getenv("LCE_DEBUG")) fprintf(stderr, "lce: launch error %s\n", cudaGetErrorString(e));
    return LCE_ERR_CUDA;
  }
  return LCE_OK;
}

// GEMM variant: CTA pairs (tcgen05 cta_group::2, 256x256 tiles) by default;
// LCE_GEMM=single selects the one-CTA 128x256 mainloop (A/B comparisons).
bool use_pair() {
  const char* e = getenv("LCE_GEMM");
  return !(e && strcmp(e, "single") == 0);
}
// persistent work units of the GEMM grid: CTA pairs, or single CTAs
int use_pair_units(int sms) { return use_pair() ? sms / 2 : sms; }
// Fused path: the fp32 logit chunk leaves the forward epilogue through TMA
// stores (128B-swizzled 32x32 staging tiles) instead of per-thread row stores;
// the split path's bf16 G chunk likewise (64x32 boxes).  LCE_ZSTORE=direct
// selects the st.global path for both (A/B comparisons).
int z_tma() {
  const char* e = getenv("LCE_ZSTORE");
  return (e && strcmp(e, "direct") == 0) ? 0 : 1;
}
// dW epilogue: fp32 rows staged in shared memory and written with TMA stores /
// reduce-adds (default), or (LCE_DW_STORE=direct) straight from registers
// (16-byte st.global / red.global.add.v4.f32).  Measured on B200 (8B / 1B /
// 70B fused, 8B split): the direct path was 1-6% slower per dW launch.
int dw_tma() {
  const char* e = getenv("LCE_DW_STORE");
  return (e && strcmp(e, "direct") == 0) ? 0 : 1;
}
// Diagnostics (A/B only): LCE_DBG_EPI=1 makes the dW epilogue skip its global
// writes, =2 also its TMEM reads (the mainloop alone); results are then wrong.
int dbg_epi() {
  const char* e = getenv("LCE_DBG_EPI");
  return e ? atoi(e) : 0;
}

// Rows of the TMA box of a K-major B operand: each CTA of a pair stages half of
// the 256-column tile.
int b_box_rows() { return use_pair() ? BN / 2 : BN; }

// Raster group (M-blocks per N sweep) of a GEMM class: the caller's choice,
// overridable per class with LCE_GROUP_M_<class index> or globally with
// LCE_GROUP_M (tuning experiments).
int group_override(int cls, int dflt) {
  char name[32];
  snprintf(name, sizeof(name), "LCE_GROUP_M_%d", cls);
  const char* e = getenv(name);
  if (!e) e = getenv("LCE_GROUP_M");
  return e ? atoi(e) : dflt;
}

int hint_override(int cls, char which, int dflt) {
  char name[32];
  snprintf(name, sizeof(name), "LCE_HINT_%c_%d", which, cls);
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Wide (512 x 256) pair tiles: chosen per call site (launch_gemm's wide_pref:
// the fused path's dH / dW and the recompute path's dW when there are enough
// token rows, kWideMinRows).  LCE_WIDE_<class index> or LCE_WIDE (1 on, 0 off)
// override; LCE_GEMM=pair / wide force one tile shape for every GEMM.
int use_wide(int cls, int dflt) {
  char name[32];
  snprintf(name, sizeof(name), "LCE_WIDE_%d", cls);
  const char* e = getenv(name);
  if (!e) e = getenv("LCE_WIDE");
  if (e) return atoi(e);
  const char* g = getenv("LCE_GEMM");
  if (g && strcmp(g, "pair") == 0) return 0;
  if (g && strcmp(g, "wide") == 0) return 1;
  return dflt;
}

// K-lockstep of the persistent GEMM grids (gemm.cuh lockstep_gate /
// lockstep_monitor): one progress word per cluster in a device-global array;
// every launch gets a new generation tag, so words left by earlier launches
// read as "not started" (a CUDA-graph replay reuses its captured tag: until
// every monitor has published again, words left by the previous replay read
// as "done" and gate nothing -- timing only).  Measured (one B200, in-step,
// medians of 3-4, monitor polling every 2 us; DESIGN.md section 5 "Power"):
// the dH / dW GEMMs' DRAM reads drop from 12.6 / 13.9 to 6.2 / 6.7 GB per 8B
// chunk (cold-cache ncu); step +1.1-5.1% (8B fused), +6.2% (70B fused),
// +0.4-2.5% (8B split) over no lockstep, the more the box is power-limited.
// Short-K pair-tile launches (1B / packed-Qwen dH, dW; forward and G at
// D < 4096) lose more to the gate's stalls than they save (1B pair dW -15%),
// so they run without it.  LCE_LOCK[_<class>]
// = 0 / 1 overrides, LCE_LOCK_D[_<class>] sets the allowed drift in k-block steps.
__device__ unsigned long long g_lock_prog[128];
constexpr int kLockMinPairK = 4096;
constexpr int kLockD = 16, kLockDPair = 32;  // k-blocks: 16 wide (1024-cycle) steps, 32 pair (512-cycle) steps
void lockstep_config(GemmDims& d, int cls, bool wide) {
  static std::atomic<uint32_t> gen{0x5a5a0000u};
  char name[32];
  snprintf(name, sizeof(name), "LCE_LOCK_%d", cls);
  const char* env = getenv(name);
  if (!env) env = getenv("LCE_LOCK");
  // default: every wide-tile launch, and the pair-tile forward / G-recompute
  // GEMMs when their K (= D) is long (>= 4096: 8B, 70B; the 1B / packed-Qwen
  // heads measured -0.5 to -1.8%); never the short-K pair dH / dW launches
  const bool dflt = wide || ((cls == LCE_K_FWD || cls == LCE_K_BWD_G) && !d.k_dev && d.k_static >= kLockMinPairK);
  if (!(env ? atoi(env) != 0 : dflt)) return;
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, g_lock_prog) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  snprintf(name, sizeof(name), "LCE_LOCK_D_%d", cls);
  const char* de = getenv(name);
  if (!de) de = getenv("LCE_LOCK_D");
  const int dd = de ? atoi(de) : (wide ? kLockD : kLockDPair);
  d.lock_prog = static_cast<unsigned long long*>(p);
  d.lock_gen = ++gen;
  d.lock_d = dd < 0 ? 0 : dd;
}

// wide_pref: this call site's tile shape (0: 256 x 256 pair tiles, 1: 512 x 256
// wide tiles); environment overrides win.
template <bool A_MN, bool B_MN, class Epi>
lce_status_t launch_gemm(int cls, const CUtensorMap& a, const CUtensorMap& b, const GemmDims& d_in,
                         const typename Epi::Params& ep, int sms, cudaStream_t s, int wide_pref = 0) {
  GemmDims d = d_in;
  // dH / dW have few N tiles (N = D) and long K: an N-fastest raster
  // (group_m = 1) lets the concurrently resident tiles of one A row block
  // read each A k-slab once; the forward / recompute GEMMs (N = V) keep
  // 16-row-block groups so the H_c group stays in L2 while W streams.
  if (d.group_m == 0) d.group_m = (cls == LCE_K_BWD_DH || cls == LCE_K_BWD_DW) ? 1 : kGroupM;
  d.group_m = group_override(cls, d.group_m);
  // L2 policy: in the forward / recompute GEMMs the A group (rows of H_c) is
  // reused by every vocab tile of the sweep while each W tile is used once per
  // group -> keep H_c, stream W.  Overridable: LCE_HINT_A_<cls> / LCE_HINT_B_<cls>.
  // (Measured on B200: every combination within the +-2% run-to-run noise of
  // these power-capped, MMA-bound kernels, evict_first on either operand
  // 2-12% slower; default normal.)
  d.a_hint = hint_override(cls, 'A', 0);
  d.b_hint = hint_override(cls, 'B', 0);
  d.st_hint = hint_override(cls, 'S', 0);
  LaunchScope sc(cls, s);
  d.probe = sc.probe();
  if (!use_pair()) {
    gemm_kernel<A_MN, B_MN, Epi><<<sms, kThreads, kSmemBytes, s>>>(a, b, d, ep);
    return last_error();
  }
  const bool wide = use_wide(cls, wide_pref) != 0;
  if ((sms >> 1) <= 128) lockstep_config(d, cls, wide);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(sms & ~1));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kPairSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (wide) cfg.dynamicSmemBytes = kWideSmemBytes;
  cudaError_t e = wide ? cudaLaunchKernelEx(&cfg, gemm_wide_kernel<A_MN, B_MN, Epi>, a, b, d, ep)
                       : cudaLaunchKernelEx(&cfg, gemm_pair_kernel<A_MN, B_MN, Epi>, a, b, d, ep);
  if (e != cudaSuccess) {
    if (getenv("LCE_DEBUG")) fprintf(stderr, "lce: cudaLaunchKernelEx -> %s\n", cudaGetErrorString(e));
    return LCE_ERR_CUDA;
  }
  return last_error();
}

// ------------------------------------------------------------------ NCCL (loaded at run time)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*groupStart)();
  ncclResult_t (*groupEnd)();
  ncclResult_t (*getAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
};

NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.getAsyncError = reinterpret_cast<decltype(api.getAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce;
  });
  return api.ok ? &api : nullptr;
}

}  // namespace

// NVLS state of a vocab-parallel communicator (LCE_NVLS=1): one multicast
// object over every rank's GPU, bound to a local fp32 buffer on each, mapped
// twice -- the multicast VA (the dH epilogue's multimem.red.add target: the
// switch adds into every GPU's copy) and the local unicast VA (read back by
// the cast / scatter).  The last 4 KB hold the NVLS barrier counter.
struct NvlsBuf {
  bool ready = false;
  size_t bytes = 0, size = 0;
  CUmemGenericAllocationHandle mc = 0, phys = 0;
  CUdeviceptr uc = 0, mcva = 0;
  uint32_t barriers = 0;  // barriers issued so far on this buffer
  int dev = -1;
  bool unicast = false;   // LCE_NVLS=2 on a one-rank communicator: cudaMalloc'd stand-in
};

struct lce_comm_s {
  ncclComm_t comm;
  int nranks, rank;
  int mode;  // lce_parallel_t
  cudaStream_t side;          // runs the dH all-reduce concurrently with the last dW GEMM
  cudaEvent_t dh_ready, dh_reduced;
  NvlsBuf nvls;
  void* scratch = nullptr;    // 256 B of device memory for the NVLS setup exchange
};

namespace {

// SMs a GEMM leaves free while an NCCL collective runs concurrently on the
// communicator's side stream (vocab-parallel dH all-reduce overlapped with the
// dW GEMM): the persistent GEMM grid otherwise fills every SM (one
// CTA per SM, ~227 KB of shared memory each) and the collective's kernel could
// only start after it.  LCE_VP_RESERVE_SMS overrides (even, 0 = no reservation).
// (LCE_VP_RESERVE_TEST=1 applies the reservation on a one-rank communicator
// too, so the reduced-grid launches are covered by the one-GPU tests.)
int overlap_sms(lce_comm_t comm, int sms) {
  if (!comm || (comm->nranks < 2 && !getenv("LCE_VP_RESERVE_TEST"))) return sms;
  const char* e = getenv("LCE_VP_RESERVE_SMS");
  int r = e ? atoi(e) : 16;
  r = r < 0 ? 0 : (r > sms / 2 ? sms / 2 : r);
  return (sms - r) & ~1;
}


// ------------------------------------------------------------------ NVLS (in-switch dH reduction)
// LCE_NVLS=1 with a vocab-parallel communicator: the dH partials are added into
// a multicast buffer by the dH GEMM's epilogue (multimem.red.add.v4.f32) instead
// of an NCCL all-reduce afterwards -- the GEMM and its collective are one
// kernel, no SMs are held back for NCCL, and the partials never make a second
// trip through HBM.  Gated on CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED on every
// rank.  Summation order inside the switch is not fixed, so dH is not bitwise
// reproducible in this mode (the NCCL path is).
struct DrvApi {
  bool ok = false;
  PFN_cuMulticastCreate mcCreate;
  PFN_cuMulticastAddDevice mcAdd;
  PFN_cuMulticastBindMem mcBind;
  PFN_cuMulticastUnbind mcUnbind;
  PFN_cuMulticastGetGranularity mcGran;
  PFN_cuMemCreate memCreate;
  PFN_cuMemRelease memRelease;
  PFN_cuMemAddressReserve addrReserve;
  PFN_cuMemAddressFree addrFree;
  PFN_cuMemMap memMap;
  PFN_cuMemUnmap memUnmap;
  PFN_cuMemSetAccess setAccess;
  PFN_cuMemExportToShareableHandle exportH;
  PFN_cuMemImportFromShareableHandle importH;
  PFN_cuDeviceGet devGet;
  PFN_cuDeviceGetAttribute devAttr;
};

DrvApi* drv() {
  static DrvApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    auto get = [&](const char* name, auto& fn) {
      void* ptr = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        ok = false;
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(ptr);
    };
    get("cuMulticastCreate", api.mcCreate);
    get("cuMulticastAddDevice", api.mcAdd);
    get("cuMulticastBindMem", api.mcBind);
    get("cuMulticastUnbind", api.mcUnbind);
    get("cuMulticastGetGranularity", api.mcGran);
    get("cuMemCreate", api.memCreate);
    get("cuMemRelease", api.memRelease);
    get("cuMemAddressReserve", api.addrReserve);
    get("cuMemAddressFree", api.addrFree);
    get("cuMemMap", api.memMap);
    get("cuMemUnmap", api.memUnmap);
    get("cuMemSetAccess", api.setAccess);
    get("cuMemExportToShareableHandle", api.exportH);
    get("cuMemImportFromShareableHandle", api.importH);
    get("cuDeviceGet", api.devGet);
    get("cuDeviceGetAttribute", api.devAttr);
    api.ok = ok;
  });
  return api.ok ? &api : nullptr;
}

// 1: NVLS; 2: its one-rank emulation (a unicast buffer and plain reductions:
// the same zero / add / barrier / read-back sequence, for boxes whose driver
// refuses multicast objects -- tests only)
int nvls_requested() {
  const char* e = getenv("LCE_NVLS");
  const int v = e ? atoi(e) : 0;
  return (v == 1 || v == 2) ? v : 0;
}

#define LCE_CU(expr)                                                                           \
  do {                                                                                         \
    CUresult r_ = (expr);                                                                      \
    if (r_ != CUDA_SUCCESS) {                                                                  \
      if (getenv("LCE_DEBUG")) fprintf(stderr, "lce: %s -> CUresult %d\n", #expr, (int)r_);    \
      return LCE_ERR_CUDA;                                                                     \
    }                                                                                          \
  } while (0)

void nvls_release(lce_comm_t c) {
  NvlsBuf& b = c->nvls;
  if (b.unicast) {
    cudaFree(reinterpret_cast<void*>(b.uc));
    b = NvlsBuf{};
    return;
  }
  DrvApi* d = drv();
  if (d) {
    if (b.mcva) {
      d->memUnmap(b.mcva, b.size);
      d->addrFree(b.mcva, b.size);
    }
    if (b.uc) {
      d->memUnmap(b.uc, b.size);
      d->addrFree(b.uc, b.size);
    }
    if (b.mc && b.phys) {
      CUdevice cud;
      if (d->devGet(&cud, b.dev) == CUDA_SUCCESS) d->mcUnbind(b.mc, cud, 0, b.size);
    }
    if (b.phys) d->memRelease(b.phys);
    if (b.mc) d->memRelease(b.mc);
  }
  b = NvlsBuf{};
}

// Host-synchronous collective setup (first use, or a larger problem): every
// rank of the communicator must call it with the same `bytes`.
lce_status_t nvls_ensure(lce_comm_t c, size_t bytes, cudaStream_t s) {
  NvlsBuf& b = c->nvls;
  const bool emulate = nvls_requested() == 2;
  if (b.ready && b.bytes >= bytes && b.unicast == emulate) return LCE_OK;
  if (emulate) {  // one rank only: a unicast stand-in for the multicast buffer
    if (c->nranks != 1) return LCE_ERR_COMM;
    nvls_release(c);
    b.size = (bytes + 4096 + 4095) / 4096 * 4096;
    void* p = nullptr;
    LCE_CUDA(cudaMalloc(&p, b.size));
    LCE_CUDA(cudaMemsetAsync(p, 0, b.size, s));
    b.uc = b.mcva = reinterpret_cast<CUdeviceptr>(p);
    b.unicast = true;
    b.bytes = bytes;
    b.ready = true;
    return LCE_OK;
  }
  DrvApi* d = drv();
  NcclApi* nc = nccl();
  if (!d || !nc || !nc->broadcast) return LCE_ERR_CUDA;
  nvls_release(c);
  int dev = 0;
  LCE_CUDA(cudaGetDevice(&dev));
  CUdevice cud;
  LCE_CU(d->devGet(&cud, dev));
  int mc_ok = 0;
  LCE_CU(d->devAttr(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cud));
  if (!c->scratch) LCE_CUDA(cudaMalloc(&c->scratch, 256));
  // every rank must support multicast (MIN over ranks)
  int32_t* sc = static_cast<int32_t*>(c->scratch);
  LCE_CUDA(cudaMemcpyAsync(sc, &mc_ok, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (nc->allReduce(sc, sc, 1, ncclInt32, ncclMin, c->comm, s) != ncclSuccess) return LCE_ERR_NCCL;
  LCE_CUDA(cudaMemcpyAsync(&mc_ok, sc, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  LCE_CUDA(cudaStreamSynchronize(s));
  if (!mc_ok) return LCE_ERR_DEVICE;
  CUmulticastObjectProp prop{};
  prop.numDevices = static_cast<unsigned>(c->nranks);
  prop.handleTypes = c->nranks > 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  size_t gran = 0;
  prop.size = bytes + 4096;
  LCE_CU(d->mcGran(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (bytes + 4096 + gran - 1) / gran * gran;
  prop.size = size;
  // rank 0 creates the multicast object; the others import it by duplicating
  // rank 0's file descriptor (pidfd_getfd); {pid, fd} travel by ncclBroadcast
  struct {
    int32_t pid, fd;
  } ex{static_cast<int32_t>(getpid()), -1};
  if (c->rank == 0) {
    // a driver / partition without multicast objects (e.g. a container that
    // sees one GPU of the NVSwitch fabric) refuses here: LCE_ERR_DEVICE
    // (a one-rank communicator has no peer to wait for it; with more ranks
    // the others then fail in the broadcast below -- NCCL path recommended)
    const CUresult r = d->mcCreate(&b.mc, &prop);
    if (r != CUDA_SUCCESS) {
      if (getenv("LCE_DEBUG")) fprintf(stderr, "lce: cuMulticastCreate -> CUresult %d\n", (int)r);
      b.mc = 0;
      if (c->nranks == 1) return LCE_ERR_DEVICE;
      ex.fd = -2;  // tell the other ranks
    }
    if (c->nranks > 1 && b.mc) {
      int fd = -1;
      LCE_CU(d->exportH(&fd, b.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
      ex.fd = fd;
    }
  }
  if (c->nranks > 1) {
    LCE_CUDA(cudaMemcpyAsync(sc, &ex, sizeof(ex), cudaMemcpyHostToDevice, s));
    if (nc->broadcast(sc, sc, sizeof(ex), ncclUint8, 0, c->comm, s) != ncclSuccess) return LCE_ERR_NCCL;
    LCE_CUDA(cudaMemcpyAsync(&ex, sc, sizeof(ex), cudaMemcpyDeviceToHost, s));
    LCE_CUDA(cudaStreamSynchronize(s));
    if (ex.fd == -2) return LCE_ERR_DEVICE;  // rank 0 could not create the multicast object
    if (c->rank != 0) {
      const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, ex.pid, 0));
      if (pidfd < 0) return LCE_ERR_CUDA;
      const int fd = static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, ex.fd, 0));
      close(pidfd);
      if (fd < 0) return LCE_ERR_CUDA;
      const CUresult r = d->importH(&b.mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      close(fd);
      LCE_CU(r);
    }
  }
  LCE_CU(d->mcAdd(b.mc, cud));
  // every device is added before anyone binds memory: a barrier over NCCL
  if (c->nranks > 1) {
    if (nc->allReduce(sc, sc, 1, ncclInt32, ncclSum, c->comm, s) != ncclSuccess) return LCE_ERR_NCCL;
    LCE_CUDA(cudaStreamSynchronize(s));
  }
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  LCE_CU(d->memCreate(&b.phys, size, &ap, 0));
  b.size = size;
  b.dev = dev;
  LCE_CU(d->mcBind(b.mc, 0, b.phys, 0, size, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  LCE_CU(d->addrReserve(&b.uc, size, gran, 0, 0));
  LCE_CU(d->memMap(b.uc, size, 0, b.phys, 0));
  LCE_CU(d->setAccess(b.uc, size, &acc, 1));
  LCE_CU(d->addrReserve(&b.mcva, size, gran, 0, 0));
  LCE_CU(d->memMap(b.mcva, size, 0, b.mc, 0));
  LCE_CU(d->setAccess(b.mcva, size, &acc, 1));
  LCE_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(b.uc), 0, size, s));
  LCE_CUDA(cudaStreamSynchronize(s));
  if (c->nranks > 1) {  // every copy (and its barrier counter) is zero before first use
    if (nc->allReduce(sc, sc, 1, ncclInt32, ncclSum, c->comm, s) != ncclSuccess) return LCE_ERR_NCCL;
    LCE_CUDA(cudaStreamSynchronize(s));
  }
  b.bytes = bytes;
  b.barriers = 0;
  b.ready = true;
  return LCE_OK;
}

// The NVLS fp32 dH buffer of `comm` for this call, or null (NCCL path).
float* nvls_buffer(lce_comm_t comm, size_t bytes, cudaStream_t s, lce_status_t* st) {
  *st = LCE_OK;
  if (!comm || comm->mode != LCE_PAR_VOCAB || !nvls_requested()) return nullptr;
  *st = nvls_ensure(comm, bytes, s);
  return *st == LCE_OK ? reinterpret_cast<float*>(comm->nvls.mcva) : nullptr;
}

// Zero this rank's copy of the first `bytes`, then a barrier so that no rank
// adds into a copy another rank has not cleared yet.
lce_status_t nvls_begin(lce_comm_t c, size_t bytes, cudaStream_t s);
// Barrier over every rank's GPU through the multicast counter (stream-ordered).
lce_status_t nvls_barrier(lce_comm_t c, cudaStream_t s) {
  NvlsBuf& b = c->nvls;
  const uint32_t target = ++b.barriers * static_cast<uint32_t>(c->nranks);
  uint32_t* mcf = reinterpret_cast<uint32_t*>(b.mcva + b.size - 4096);
  const uint32_t* ucf = reinterpret_cast<const uint32_t*>(b.uc + b.size - 4096);
  LaunchScope sc(LCE_K_COMM, s);
  nvls_barrier_kernel<<<1, 32, 0, s>>>(mcf, ucf, target, b.unicast ? 1 : 0);
  return last_error();
}
lce_status_t nvls_begin(lce_comm_t c, size_t bytes, cudaStream_t s) {
  LCE_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(c->nvls.uc), 0, bytes, s));
  return nvls_barrier(c, s);
}
// This rank's copy of the reduced buffer (read after the closing barrier).
float* nvls_local(lce_comm_t c) { return reinterpret_cast<float*>(c->nvls.uc); }

lce_status_t allreduce(lce_comm_t c, void* buf, size_t count, ncclRedOp_t op, cudaStream_t s) {
  NcclApi* api = nccl();
  if (!api) return LCE_ERR_NCCL;
  LaunchScope sc(LCE_K_COMM, s);
  if (api->allReduce(buf, buf, count, ncclFloat32, op, c->comm, s) != ncclSuccess) return LCE_ERR_NCCL;
  return LCE_OK;
}

lce_status_t allreduce_i32(lce_comm_t c, void* buf, size_t count, cudaStream_t s) {
  NcclApi* api = nccl();
  if (!api) return LCE_ERR_NCCL;
  LaunchScope sc(LCE_K_COMM, s);
  if (api->allReduce(buf, buf, count, ncclInt32, ncclSum, c->comm, s) != ncclSuccess) return LCE_ERR_NCCL;
  return LCE_OK;
}

// The vocab-parallel / token-parallel communicator behind `c` (null if none).
lce_comm_t vocab_comm(lce_comm_t c) { return (c && c->mode == LCE_PAR_VOCAB) ? c : nullptr; }
lce_comm_t token_comm(lce_comm_t c) { return (c && c->mode == LCE_PAR_TOKEN) ? c : nullptr; }

// Token parallelism, after prep: all-reduce (N_v, bad-label flag) and rescale
// the MEAN divisor / gradient scale to the global N_v.
lce_status_t tp_sync(lce_comm_t tp, Header* hdr, const float* grad_loss, int reduction, cudaStream_t s) {
  if (!tp) return LCE_OK;
  LCE_TRY(allreduce_i32(tp, &hdr->tp_nv, 2, s));
  LaunchScope sc(LCE_K_PREP, s);
  tp_scale_kernel<<<1, 1, 0, s>>>(hdr, grad_loss, reduction);
  return last_error();
}
// Token parallelism: the rank's loss share (sum_i loss_i / N_v_global for
// MEAN, sum_i loss_i otherwise) summed over ranks.
lce_status_t tp_loss(lce_comm_t tp, float* loss, cudaStream_t s) {
  return tp ? allreduce(tp, loss, 1, ncclSum, s) : LCE_OK;
}
// Token parallelism, a rank with no tokens: still joins both exchanges.
lce_status_t tp_empty_rank(lce_comm_t tp, const lce_problem_t* p, Header* hdr, const float* grad_loss,
                           float* loss, int32_t* n_valid, cudaStream_t s) {
  {
    LaunchScope sc(LCE_K_PREP, s);
    prep_kernel<<<1, 1024, 0, s>>>(nullptr, 0, p->ignore_index, p->vocab_total, nullptr, nullptr, nullptr, nullptr,
                                   nullptr, hdr, grad_loss, p->reduction);
    LCE_TRY(last_error());
  }
  LCE_TRY(tp_sync(tp, hdr, grad_loss, p->reduction, s));
  if (loss) {
    LCE_CUDA(cudaMemsetAsync(loss, 0, sizeof(float), s));
    LCE_TRY(tp_loss(tp, loss, s));
  }
  if (n_valid) LCE_CUDA(cudaMemcpyAsync(n_valid, &hdr->mean_div, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  return LCE_OK;
}

lce_status_t validate(const lce_problem_t* p, lce_comm_t comm, size_t ws_bytes, const void* ws, Plan* pl) {
  if (!p) return LCE_ERR_NULL;
  if (p->reduction != LCE_MEAN && p->reduction != LCE_SUM && p->reduction != LCE_NONE) return LCE_ERR_REDUCTION;
  if (!make_plan(p, pl)) return LCE_ERR_SHAPE;
  if (!ws) return LCE_ERR_NULL;
  if (!aligned16(ws)) return LCE_ERR_ALIGN;
  if (ws_bytes < pl->total) return LCE_ERR_WORKSPACE;
  if (!vocab_comm(comm) && (p->vocab_start != 0 || p->vocab_local != p->vocab_total)) return LCE_ERR_COMM;
  return LCE_OK;
}


}  // namespace

// ====================================================================== C ABI
extern "C" {

int lce_abi_version(void) { return LCE_ABI_VERSION; }

uint64_t lce_launch_count(void) { return g_launches.load(); }

const char* lce_status_string(lce_status_t s) {
  switch (s) {
    case LCE_OK: return "ok";
    case LCE_ERR_NULL: return "null pointer";
    case LCE_ERR_SHAPE: return "invalid shape";
    case LCE_ERR_ALIGN: return "pointer not 16-byte aligned";
    case LCE_ERR_REDUCTION: return "invalid reduction";
    case LCE_ERR_WORKSPACE: return "workspace too small";
    case LCE_ERR_LABEL_RANGE: return "label out of range";
    case LCE_ERR_DEVICE: return "device is not sm_100 (B200)";
    case LCE_ERR_CUDA: return "CUDA error";
    case LCE_ERR_NCCL: return "NCCL error or NCCL unavailable";
    case LCE_ERR_COMM: return "communicator does not match problem";
    case LCE_ERR_ARG: return "unsupported flag combination";
    case LCE_ERR_UPSTREAM: return "upstream gradient differs from the one the fused call assumed";
  }
  return "unknown status";
}

size_t lce_workspace_bytes(const lce_problem_t* p) {
  Plan pl;
  if (!make_plan(p, &pl)) return 0;
  return pl.total;
}

lce_status_t lce_forward(const lce_problem_t* p, lce_comm_t comm_in, const uint16_t* hidden, const uint16_t* weight,
                         const int32_t* labels, float* loss, float* lse, float* token_loss, int32_t* n_valid,
                         void* workspace, size_t workspace_bytes, void* stream) {
  NvtxCall nvtx_call("lce_forward");
  Plan pl;
  LCE_TRY(validate(p, comm_in, workspace_bytes, workspace, &pl));
  lce_comm_t comm = vocab_comm(comm_in), tp = token_comm(comm_in);
  if (!weight || !loss) return LCE_ERR_NULL;
  if (pl.N > 0 && (!hidden || !labels || !lse)) return LCE_ERR_NULL;
  const void* ptrs[] = {hidden, weight, labels, loss, lse, token_loss, n_valid};
  for (const void* q : ptrs)
    if (q && !aligned16(q)) return LCE_ERR_ALIGN;
  DevInfo dev;
  LCE_TRY(device_info(&dev));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  Header* hdr = reinterpret_cast<Header*>(ws + pl.hdr);

  if (pl.N == 0) {  // empty batch: loss 0, N_v 0, nothing to project
    if (tp) return tp_empty_rank(tp, p, hdr, nullptr, loss, n_valid, s);
    LCE_CUDA(cudaMemsetAsync(loss, 0, sizeof(float), s));
    if (n_valid) LCE_CUDA(cudaMemsetAsync(n_valid, 0, sizeof(int32_t), s));
    return LCE_OK;
  }
  const int N = static_cast<int>(pl.N);
  int32_t* idx = reinterpret_cast<int32_t*>(ws + pl.idx);
  int32_t* yc = reinterpret_cast<int32_t*>(ws + pl.yc);
  float* zt = reinterpret_cast<float*>(ws + pl.zt);
  uint16_t* hc = reinterpret_cast<uint16_t*>(ws + pl.hc);
  float* pm = reinterpret_cast<float*>(ws + pl.pm);
  float* ps = reinterpret_cast<float*>(ws + pl.ps);
  double* bsum = reinterpret_cast<double*>(ws + pl.bsum);
  float* mloc = reinterpret_cast<float*>(ws + pl.mloc);
  float* mglob = reinterpret_cast<float*>(ws + pl.mglob);
  float* sbuf = reinterpret_cast<float*>(ws + pl.sbuf);

  {  // S0: label scan + compaction
    LaunchScope sc(LCE_K_PREP, s);
    prep_kernel<<<1, 1024, 0, s>>>(labels, N, p->ignore_index, p->vocab_total, idx, yc, zt, lse, token_loss, hdr,
                                   nullptr, p->reduction);
    LCE_TRY(last_error());
  }
  LCE_TRY(tp_sync(tp, hdr, nullptr, p->reduction, s));
  {  // S0: gather valid rows of H
    LaunchScope sc(LCE_K_GATHER, s);
    gather_kernel<<<static_cast<unsigned>(pl.cap), 128, 0, s>>>(hidden, pl.D, N, idx, hdr, hc, nullptr, nullptr,
                                                               nullptr, nullptr, labels, p->ignore_index,
                                                               p->vocab_total, nullptr);
    LCE_TRY(last_error());
  }
  // S1+S2: logits tile by tile in TMEM, online LSE epilogue
  CUtensorMap ta, tb;
  LCE_TRY(map_kmajor(&ta, hc, pl.cap, pl.D, pl.D, BM));
  LCE_TRY(map_kmajor(&tb, weight, pl.Vl, pl.D, pl.D, b_box_rows()));
  GemmDims d{&hdr->n_valid, 0, nullptr, static_cast<int32_t>(pl.D), static_cast<int32_t>(pl.Vl)};
  EpiLse::Params ep{yc, static_cast<int32_t>(p->vocab_start), static_cast<int32_t>(pl.Vl), pm, ps, pl.cap, zt, 0, nullptr, 0};
  LCE_TRY((launch_gemm<false, false, EpiLse>(LCE_K_FWD, ta, tb, d, ep, dev.sms, s)));

  const unsigned cblocks = static_cast<unsigned>(pl.nblocks);
  const int nt = static_cast<int>(pl.n_tiles);
  if (!comm) {  // S3 on one GPU: one fused combine + loss kernel
    LaunchScope sc(LCE_K_COMBINE, s);
    combine_kernel<<<cblocks, 256, 0, s>>>(0, pm, ps, nt, pl.cap, mloc, mglob, sbuf, zt, idx, hdr, lse, token_loss,
                                           bsum, loss, n_valid, p->reduction);
    LCE_TRY(last_error());
    return tp_loss(tp, loss, s);
  }
  {  // with a communicator (any size, including 1): local merge first
    LaunchScope sc(LCE_K_COMBINE, s);
    combine_kernel<<<cblocks, 256, 0, s>>>(1, pm, ps, nt, pl.cap, mloc, mglob, sbuf, zt, idx, hdr, lse, token_loss,
                                           bsum, loss, n_valid, p->reduction);
    LCE_TRY(last_error());
  }
  // vocab-parallel exchange: MAX of m, then SUM of (s * e^{m - M}, z_target)
  float* sz = sbuf;                  // [cap] s followed by [cap] target logits
  float* ztc = sbuf + pl.cap;
  LCE_CUDA(cudaMemcpyAsync(ztc, zt, pl.cap * sizeof(float), cudaMemcpyDeviceToDevice, s));
  LCE_TRY(allreduce(comm, mglob, pl.cap, ncclMax, s));
  {
    LaunchScope sc(LCE_K_COMBINE, s);
    combine_kernel<<<cblocks, 256, 0, s>>>(2, pm, ps, nt, pl.cap, mloc, mglob, sbuf, zt, idx, hdr, lse, token_loss,
                                           bsum, loss, n_valid, p->reduction);
    LCE_TRY(last_error());
  }
  LCE_TRY(allreduce(comm, sz, 2 * pl.cap, ncclSum, s));
  {
    LaunchScope sc(LCE_K_COMBINE, s);
    combine_kernel<<<cblocks, 256, 0, s>>>(3, pm, ps, nt, pl.cap, mloc, mglob, sbuf, ztc, idx, hdr, lse,
                                           token_loss, bsum, loss, n_valid, p->reduction);
    LCE_TRY(last_error());
  }
  return LCE_OK;
}

}  // extern "C"

namespace {

// In-backward AdamW state for lce_backward_adamw (NEXT-2); null for lce_backward.
struct AdamArgs {
  float* theta;
  float* exp_avg;
  float* exp_avg_sq;
  uint16_t* w;
  lce_adamw_t hp;
};

lce_status_t backward_impl(const lce_problem_t* p, lce_comm_t comm_in, const uint16_t* hidden, const uint16_t* weight,
                           const int32_t* labels, const float* lse, const float* grad_loss, uint16_t* dhidden,
                           void* dweight_out, int dweight_flags, const AdamArgs* adam, void* workspace,
                           size_t workspace_bytes, void* stream) {
  Plan pl;
  LCE_TRY(validate(p, comm_in, workspace_bytes, workspace, &pl));
  lce_comm_t comm = vocab_comm(comm_in), tp = token_comm(comm_in);
  if (tp && adam) return LCE_ERR_COMM;  // the in-backward step needs the full-batch dW
  if ((dweight_flags & ~(LCE_DW_ACCUMULATE | LCE_DW_BF16)) ||
      ((dweight_flags & LCE_DW_BF16) && (dweight_flags & LCE_DW_ACCUMULATE)))
    return LCE_ERR_ARG;
  const bool accumulate_dweight = (dweight_flags & LCE_DW_ACCUMULATE) != 0;
  const bool dw_bf16 = (dweight_flags & LCE_DW_BF16) != 0;
  float* dweight = dw_bf16 ? nullptr : static_cast<float*>(dweight_out);
  uint16_t* dweight_h = dw_bf16 ? static_cast<uint16_t*>(dweight_out) : nullptr;
  if (!weight || (!dweight_out && !adam)) return LCE_ERR_NULL;
  if (pl.N > 0 && (!hidden || !labels || !lse || !dhidden)) return LCE_ERR_NULL;
  const void* ptrs[] = {hidden, weight, labels, lse, grad_loss, dhidden, dweight_out};
  for (const void* q : ptrs)
    if (q && !aligned16(q)) return LCE_ERR_ALIGN;
  DevInfo dev;
  LCE_TRY(device_info(&dev));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  Header* hdr = reinterpret_cast<Header*>(ws + pl.hdr);

  if (pl.N == 0 && !adam) {
    if (!accumulate_dweight)
      LCE_CUDA(cudaMemsetAsync(dweight_out, 0, pl.Vl * pl.D * (dw_bf16 ? sizeof(uint16_t) : sizeof(float)), s));
    if (tp) return tp_empty_rank(tp, p, hdr, grad_loss, nullptr, nullptr, s);
    return LCE_OK;
  }
  if (pl.N == 0) {  // empty batch, in-backward AdamW: the step still runs with g = 0
    LCE_CUDA(cudaMemsetAsync(hdr, 0, sizeof(Header), s));
    CUtensorMap t_any;
    LCE_TRY(map_mnmajor(&t_any, weight, pl.Vl, pl.D, pl.D));
    const lce_adamw_t& h = adam->hp;
    const double bc1 = 1.0 - pow(static_cast<double>(h.beta1), static_cast<double>(h.step));
    const double bc2 = 1.0 - pow(static_cast<double>(h.beta2), static_cast<double>(h.step));
    GemmDims d{nullptr, static_cast<int32_t>(pl.Vl), nullptr, 0, static_cast<int32_t>(pl.D)};
    EpiAdamW::Params ep{adam->theta, adam->exp_avg, adam->exp_avg_sq, adam->w, pl.D, hdr, h.lr, h.beta1, h.beta2,
                        h.eps, 1.f - h.lr * h.weight_decay, static_cast<float>(h.lr / bc1),
                        static_cast<float>(sqrt(bc2))};
    return launch_gemm<true, true, EpiAdamW>(LCE_K_BWD_DW, t_any, t_any, d, ep, dev.sms, s);
  }
  const int N = static_cast<int>(pl.N);
  int32_t* idx = reinterpret_cast<int32_t*>(ws + pl.idx);
  int32_t* yc = reinterpret_cast<int32_t*>(ws + pl.yc);
  float* zt = reinterpret_cast<float*>(ws + pl.zt);
  float* lsec = reinterpret_cast<float*>(ws + pl.lsec);
  float* gsc = reinterpret_cast<float*>(ws + pl.gsc);
  // reduction NONE: grad_loss is [N] per-token upstream gradients, folded into G per row
  const float* row_grad = p->reduction == LCE_NONE ? grad_loss : nullptr;
  uint16_t* hc = reinterpret_cast<uint16_t*>(ws + pl.hc);
  uint16_t* G = reinterpret_cast<uint16_t*>(ws + pl.g);
  float* dh = reinterpret_cast<float*>(ws + pl.dh);
  const bool multi = comm && comm->nranks >= 1;
  // dH chunks accumulate through TMA stores / reduce-adds (then one finalize
  // pass) instead of an SM read-modify-write per chunk; LCE_DH_TMA=0 selects
  // the read-modify-write epilogue (A/B)
  const bool dh_tma = z_tma() && !(getenv("LCE_DH_TMA") && atoi(getenv("LCE_DH_TMA")) == 0);

  {
    LaunchScope sc(LCE_K_PREP, s);
    prep_kernel<<<1, 1024, 0, s>>>(labels, N, p->ignore_index, p->vocab_total, idx, yc, zt, nullptr, nullptr, hdr,
                                   grad_loss, p->reduction);
    LCE_TRY(last_error());
  }
  LCE_TRY(tp_sync(tp, hdr, grad_loss, p->reduction, s));
  {
    LaunchScope sc(LCE_K_GATHER, s);
    gather_kernel<<<static_cast<unsigned>(pl.cap), 128, 0, s>>>(hidden, pl.D, N, idx, hdr, hc, lse, lsec, row_grad,
                                                               gsc, labels, p->ignore_index, p->vocab_total, dhidden);
    LCE_TRY(last_error());
  }
  // NVLS (LCE_NVLS=1): every vocab chunk's dH epilogue adds into the multicast
  // buffer, which the switch sums over ranks; one barrier after the last dW
  lce_status_t nst;
  float* nvls_mc = multi ? nvls_buffer(comm, static_cast<size_t>(pl.cap * pl.D * 4), s, &nst) : nullptr;
  if (multi) LCE_TRY(nst);
  if (nvls_mc) LCE_TRY(nvls_begin(comm, static_cast<size_t>(pl.cap * pl.D * 4), s));
  CUtensorMap t_hc_k, t_hc_mn, t_g_k, t_g_mn;
  LCE_TRY(map_kmajor(&t_hc_k, hc, pl.cap, pl.D, pl.D, BM));
  LCE_TRY(map_mnmajor(&t_hc_mn, hc, pl.cap, pl.D, pl.D));
  LCE_TRY(map_kmajor(&t_g_k, G, pl.cap, pl.Vc, pl.Vc, BM));
  LCE_TRY(map_mnmajor(&t_g_mn, G, pl.cap, pl.Vc, pl.Vc));

  for (int64_t k = 0; k < pl.n_chunks; ++k) {
    const int64_t v0 = k * pl.Vc;
    const int64_t vc = (pl.Vl - v0) < pl.Vc ? (pl.Vl - v0) : pl.Vc;
    const uint16_t* wc = weight + v0 * pl.D;
    CUtensorMap t_w_k, t_w_mn;
    LCE_TRY(map_kmajor(&t_w_k, wc, vc, pl.D, pl.D, b_box_rows()));
    LCE_TRY(map_mnmajor(&t_w_mn, wc, vc, pl.D, pl.D));
    // S4: recompute logits of the chunk, G_c = softmax - onehot (bf16)
    {
      GemmDims d{&hdr->n_valid, 0, nullptr, static_cast<int32_t>(pl.D), static_cast<int32_t>(vc)};
      EpiG::Params ep{yc, lsec, static_cast<int32_t>(p->vocab_start + v0), static_cast<int32_t>(vc), G, pl.Vc,
                      row_grad ? gsc : nullptr};
      ep.use_gmap = z_tma();
      if (ep.use_gmap) LCE_TRY(encode_map(&ep.gmap, G, pl.Vc, pl.cap, pl.Vc, 32));
      LCE_TRY((launch_gemm<false, false, EpiG>(LCE_K_BWD_G, t_hc_k, t_w_k, d, ep, dev.sms, s)));
    }
    // S6: dH (+)= G_c W_c   (A = G_c K-major over vocab, B = W_c MN-major)
    {
      GemmDims d{&hdr->n_valid, 0, nullptr, static_cast<int32_t>(vc), static_cast<int32_t>(pl.D)};
      EpiDH::Params ep{dh, pl.D, k == 0, (!multi && !dh_tma && k == pl.n_chunks - 1) ? 1 : 0, hdr, dhidden, idx,
                       0, 1};
      ep.use_map = (dh_tma && !nvls_mc) ? 1 : 0;
      if (ep.use_map) LCE_TRY(map_f32_store(&ep.map, dh, pl.D, pl.cap, pl.D));
      ep.mc_out = nvls_mc;  // unscaled chunk sums into the switch-reduced buffer
      ep.mc_unicast = (nvls_mc && comm->nvls.unicast) ? 1 : 0;
      // the TMA epilogue is short enough for wide tiles; the read-modify-write
      // one (LCE_DH_TMA=0) is not
      LCE_TRY((launch_gemm<false, true, EpiDH>(LCE_K_BWD_DH, t_g_k, t_w_mn, d, ep, dev.sms, s,
                                               (dh_tma && pl.cap >= kWideMinRows) ? 1 : 0)));
    }
    // S7 (vocab-parallel): once the last chunk's dH partial is complete, its
    // all-reduce runs on the communicator's side stream while the last dW GEMM
    // (which does not read dH) runs here.
    if (multi && !nvls_mc && k == pl.n_chunks - 1) {
      LCE_CUDA(cudaEventRecord(comm->dh_ready, s));
      LCE_CUDA(cudaStreamWaitEvent(comm->side, comm->dh_ready, 0));
      LCE_TRY(allreduce(comm, dh, static_cast<size_t>(pl.N * pl.D), ncclSum, comm->side));
      LCE_CUDA(cudaEventRecord(comm->dh_reduced, comm->side));
    }
    // S5: dW_c = c G_c^T H   (A = G_c MN-major, B = H_c MN-major, K = N_v)
    {
      GemmDims d{nullptr, static_cast<int32_t>(vc), &hdr->n_valid, 0, static_cast<int32_t>(pl.D)};
      if (!adam) {
        EpiDW::Params ep{dw_bf16 ? nullptr : dweight + v0 * pl.D, pl.D, accumulate_dweight ? 1 : 0, hdr, 1};
        // bf16 rows are written straight from registers (the direct epilogue)
        ep.use_map = dw_bf16 ? 0 : dw_tma();
        ep.dw_bf16 = dw_bf16 ? dweight_h + v0 * pl.D : nullptr;
        ep.dbg = dbg_epi();
        if (ep.use_map) LCE_TRY(map_f32_store(&ep.map, dweight + v0 * pl.D, pl.D, vc, pl.D));
        ep.prefetch = 0;  // each dW row block is written once here (K = all tokens)
        // the last chunk's dW runs beside the dH all-reduce (vocab-parallel)
        const int g_sms = (multi && !nvls_mc && k == pl.n_chunks - 1) ? overlap_sms(comm, dev.sms) : dev.sms;
        LCE_TRY((launch_gemm<true, true, EpiDW>(LCE_K_BWD_DW, t_g_mn, t_hc_mn, d, ep, g_sms, s,
                                                 pl.cap >= kWideMinRows ? 1 : 0)));
      } else {  // NEXT-2: the AdamW step of these W rows happens in the dW epilogue
        const lce_adamw_t& h = adam->hp;
        const double bc1 = 1.0 - pow(static_cast<double>(h.beta1), static_cast<double>(h.step));
        const double bc2 = 1.0 - pow(static_cast<double>(h.beta2), static_cast<double>(h.step));
        const int64_t o = v0 * pl.D;
        EpiAdamW::Params ep{adam->theta + o, adam->exp_avg + o, adam->exp_avg_sq + o, adam->w + o, pl.D, hdr,
                            h.lr, h.beta1, h.beta2, h.eps, 1.f - h.lr * h.weight_decay,
                            static_cast<float>(h.lr / bc1), static_cast<float>(sqrt(bc2))};
        // pair tiles: the optimizer epilogue (26 bytes of state traffic per
        // element) is too long to hide behind the wide kernel's other half
        const int g_sms = (multi && !nvls_mc && k == pl.n_chunks - 1) ? overlap_sms(comm, dev.sms) : dev.sms;
        LCE_TRY((launch_gemm<true, true, EpiAdamW>(LCE_K_BWD_DW, t_g_mn, t_hc_mn, d, ep, g_sms, s, 0)));
      }
    }
  }
  if (nvls_mc) {  // every rank's adds have landed in every copy: scale, cast, scatter this rank's copy
    LCE_TRY(nvls_barrier(comm, s));
    LaunchScope sc(LCE_K_FINAL, s);
    finalize_dh_kernel<<<static_cast<unsigned>(pl.N), 256, 0, s>>>(nvls_local(comm), pl.D, idx, hdr, dhidden);
    LCE_TRY(last_error());
  } else if (multi || dh_tma) {
    // S7: dH summed over the vocab shards, then scaled, cast, scattered
    if (multi) LCE_CUDA(cudaStreamWaitEvent(s, comm->dh_reduced, 0));
    LaunchScope sc(LCE_K_FINAL, s);
    finalize_dh_kernel<<<static_cast<unsigned>(pl.N), 256, 0, s>>>(dh, pl.D, idx, hdr, dhidden);
    LCE_TRY(last_error());
  }
  return LCE_OK;
}

// S6 + S5 (+ S7 under vocab parallel) of one row chunk of the fused paths (CE
// and KD), from the chunk's bf16 G: dH rows = G_q W (K = V_l; split-K into fp32
// slabs that reuse the dead logit chunk Z, so the persistent grid sees whole
// waves), written straight to dhidden -- or, with a communicator, summed in
// fp32 and all-reduced on the side stream while the dW GEMM runs, then cast and
// scattered; dW (+)= G_q^T H_q (K = chunk rows).
lce_status_t chunk_grads(const FusedPlan& fp, lce_comm_t comm, int sms, cudaStream_t s, Header* hdr,
                         const CUtensorMap& t_g_k, const CUtensorMap& t_w_mn, const CUtensorMap& t_g_mn,
                         const CUtensorMap& t_h_mn, int32_t r0, float* slab, float* vdh, const int32_t* idx,
                         uint16_t* dhidden, float* dweight, bool accumulate, const float* row_coef = nullptr,
                         float* nvls_mc = nullptr) {
  const int32_t Nc = static_cast<int32_t>(fp.Nc), Vl = static_cast<int32_t>(fp.Vl), D = static_cast<int32_t>(fp.D);
  const int split = fp.split;
  if (nvls_mc) {
    // NVLS: the dH GEMM's epilogue adds its (split-K) partials of the chunk rows
    // into the multicast buffer -- summed over ranks in the switch -- while the
    // GEMM runs; no slabs, no NCCL kernel, no SMs held back for one
    const size_t bytes = static_cast<size_t>(fp.Nc * fp.D * 4);
    LCE_TRY(nvls_begin(comm, bytes, s));
    {
      GemmDims d{&hdr->n_valid, 0, nullptr, Vl, D, r0, Nc, 0, 0, split};
      EpiDH::Params ep{nullptr, fp.D, 1, 1, hdr, dhidden, idx, r0, 0, nullptr, 0};
      ep.row_coef = row_coef;
      ep.mc_out = nvls_mc;
      ep.mc_unicast = comm->nvls.unicast ? 1 : 0;
      LCE_TRY((launch_gemm<false, true, EpiDH>(LCE_K_BWD_DH, t_g_k, t_w_mn, d, ep, sms, s, fp.wide_dh)));
    }
    {
      GemmDims d{nullptr, Vl, &hdr->n_valid, 0, D, 0, 0, r0, Nc};
      EpiDW::Params ep{dweight, fp.D, accumulate ? 1 : 0, hdr, 0};
      ep.use_map = dw_tma();
      if (ep.use_map) LCE_TRY(map_f32_store(&ep.map, dweight, fp.D, fp.Vl, fp.D));
      LCE_TRY((launch_gemm<true, true, EpiDW>(LCE_K_BWD_DW, t_g_mn, t_h_mn, d, ep, sms, s, fp.wide_dw)));
    }
    LCE_TRY(nvls_barrier(comm, s));  // every rank's partials have landed in every copy
    LaunchScope sc(LCE_K_FINAL, s);
    reduce_dh_kernel<<<static_cast<unsigned>(fp.Nc), 256, 0, s>>>(nvls_local(comm), 1, fp.Nc * fp.D, fp.D, r0, Nc, idx,
                                                                 hdr, dhidden);
    return last_error();
  }
  {
    GemmDims d{&hdr->n_valid, 0, nullptr, Vl, D, r0, Nc, 0, 0, split};
    float* part = split > 1 ? slab : (comm ? vdh : nullptr);
    EpiDH::Params ep{nullptr, fp.D, 1, 1, hdr, dhidden, idx, r0, 0, part, fp.Nc * fp.D};
    ep.row_coef = row_coef;
    // split-K slabs through TMA stores (LCE_DH_SLAB_TMA=0: per-row 16-byte stores)
    if (part && !(getenv("LCE_DH_SLAB_TMA") && atoi(getenv("LCE_DH_SLAB_TMA")) == 0)) {
      ep.use_map = 1;
      LCE_TRY(map_f32_store(&ep.map, part, fp.D, (split > 1 ? split : 1) * fp.Nc, fp.D));
    }
    LCE_TRY((launch_gemm<false, true, EpiDH>(LCE_K_BWD_DH, t_g_k, t_w_mn, d, ep, sms, s, fp.wide_dh)));
  }
  if (split > 1) {
    LaunchScope sc(LCE_K_FINAL, s);
    reduce_dh_kernel<<<static_cast<unsigned>(fp.Nc), 256, 0, s>>>(slab, split, fp.Nc * fp.D, fp.D, r0, Nc, idx, hdr,
                                                                 dhidden, comm ? vdh : nullptr);
    LCE_TRY(last_error());
  }
  if (comm) {
    LCE_CUDA(cudaEventRecord(comm->dh_ready, s));
    LCE_CUDA(cudaStreamWaitEvent(comm->side, comm->dh_ready, 0));
    LCE_TRY(allreduce(comm, vdh, static_cast<size_t>(fp.Nc * fp.D), ncclSum, comm->side));
    LCE_CUDA(cudaEventRecord(comm->dh_reduced, comm->side));
  }
  {
    GemmDims d{nullptr, Vl, &hdr->n_valid, 0, D, 0, 0, r0, Nc};
    EpiDW::Params ep{dweight, fp.D, accumulate ? 1 : 0, hdr, 0};
    ep.use_map = dw_tma();
    ep.dbg = dbg_epi();
    // L2 prefetch of the old dW rows before the reduce-adds: measured 0.5-1.3%
    // slower per step (8B / 70B fused), so off unless LCE_DW_PREFETCH=1
    ep.prefetch = getenv("LCE_DW_PREFETCH") && atoi(getenv("LCE_DW_PREFETCH")) == 1;
    if (ep.use_map) LCE_TRY(map_f32_store(&ep.map, dweight, fp.D, fp.Vl, fp.D));
    // runs beside this chunk's dH all-reduce under vocab parallelism
    LCE_TRY((launch_gemm<true, true, EpiDW>(LCE_K_BWD_DW, t_g_mn, t_h_mn, d, ep, overlap_sms(comm, sms), s,
                                            fp.wide_dw)));
  }
  if (comm) {  // cast + scatter the reduced dH rows of the chunk (c already in G)
    LCE_CUDA(cudaStreamWaitEvent(s, comm->dh_reduced, 0));
    LaunchScope sc(LCE_K_FINAL, s);
    reduce_dh_kernel<<<static_cast<unsigned>(fp.Nc), 256, 0, s>>>(vdh, 1, fp.Nc * fp.D, fp.D, r0, Nc, idx, hdr,
                                                                 dhidden);
    LCE_TRY(last_error());
  }
  return LCE_OK;
}

}  // namespace

extern "C" {

lce_status_t lce_backward(const lce_problem_t* p, lce_comm_t comm, const uint16_t* hidden, const uint16_t* weight,
                          const int32_t* labels, const float* lse, const float* grad_loss, uint16_t* dhidden,
                          void* dweight, int dweight_flags, void* workspace, size_t workspace_bytes,
                          void* stream) {
  NvtxCall nvtx_call("lce_backward");
  return backward_impl(p, comm, hidden, weight, labels, lse, grad_loss, dhidden, dweight, dweight_flags, nullptr,
                       workspace, workspace_bytes, stream);
}

lce_status_t lce_backward_adamw(const lce_problem_t* p, lce_comm_t comm, const uint16_t* hidden, uint16_t* weight,
                                const int32_t* labels, const float* lse, const float* grad_loss, uint16_t* dhidden,
                                float* master_weight, float* exp_avg, float* exp_avg_sq, const lce_adamw_t* hp,
                                void* workspace, size_t workspace_bytes, void* stream) {
  NvtxCall nvtx_call("lce_backward_adamw");
  if (!hp || !master_weight || !exp_avg || !exp_avg_sq || !weight) return LCE_ERR_NULL;
  if (hp->step < 1 || !(hp->beta1 >= 0.f && hp->beta1 < 1.f) || !(hp->beta2 >= 0.f && hp->beta2 < 1.f) ||
      !(hp->eps > 0.f) || !(hp->lr >= 0.f) || !(hp->weight_decay >= 0.f))
    return LCE_ERR_SHAPE;
  if (!aligned16(master_weight) || !aligned16(exp_avg) || !aligned16(exp_avg_sq)) return LCE_ERR_ALIGN;
  AdamArgs a{master_weight, exp_avg, exp_avg_sq, weight, *hp};
  return backward_impl(p, comm, hidden, weight, labels, lse, grad_loss, dhidden, nullptr, 0, &a, workspace,
                       workspace_bytes, stream);
}

size_t lce_fused_workspace_bytes(const lce_problem_t* p) {
  FusedPlan fp;
  if (!make_fused_plan(p, &fp)) return 0;
  return fp.total;
}

lce_status_t lce_forward_backward(const lce_problem_t* p, lce_comm_t comm_in, const uint16_t* hidden,
                                  const uint16_t* weight, const int32_t* labels, const float* grad_loss,
                                  float* loss, float* lse, float* token_loss, int32_t* n_valid, uint16_t* dhidden,
                                  float* dweight, int dweight_flags, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  NvtxCall nvtx_call("lce_forward_backward");
  if (!p) return LCE_ERR_NULL;
  if (dweight_flags & ~LCE_DW_ACCUMULATE) return LCE_ERR_ARG;  // fp32 only: dW is summed over row chunks
  const bool accumulate_dweight = dweight_flags != 0;
  if (p->reduction != LCE_MEAN && p->reduction != LCE_SUM && p->reduction != LCE_NONE) return LCE_ERR_REDUCTION;
  FusedPlan fp;
  if (!make_fused_plan(p, &fp)) return LCE_ERR_SHAPE;
  lce_comm_t comm = vocab_comm(comm_in), tp = token_comm(comm_in);
  if (!comm && (p->vocab_start != 0 || p->vocab_local != p->vocab_total)) return LCE_ERR_COMM;
  if (!workspace || !weight || !loss || !dweight) return LCE_ERR_NULL;
  if (fp.N > 0 && (!hidden || !labels || !lse || !dhidden)) return LCE_ERR_NULL;
  const void* ptrs[] = {hidden, weight, labels, grad_loss, loss, lse, token_loss, n_valid, dhidden, dweight, workspace};
  for (const void* q : ptrs)
    if (q && !aligned16(q)) return LCE_ERR_ALIGN;
  if (workspace_bytes < fp.total) return LCE_ERR_WORKSPACE;
  DevInfo dev;
  LCE_TRY(device_info(&dev));
  fit_plan_to_device(&fp, dev.sms);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  Header* hdr = reinterpret_cast<Header*>(ws + fp.hdr);
  if (fp.N == 0) {
    if (!accumulate_dweight) LCE_CUDA(cudaMemsetAsync(dweight, 0, fp.Vl * fp.D * sizeof(float), s));
    if (tp) return tp_empty_rank(tp, p, hdr, grad_loss, loss, n_valid, s);
    LCE_CUDA(cudaMemsetAsync(loss, 0, sizeof(float), s));
    if (n_valid) LCE_CUDA(cudaMemsetAsync(n_valid, 0, sizeof(int32_t), s));
    return LCE_OK;
  }
  const int N = static_cast<int>(fp.N);
  int32_t* idx = reinterpret_cast<int32_t*>(ws + fp.idx);
  int32_t* yc = reinterpret_cast<int32_t*>(ws + fp.yc);
  float* zt = reinterpret_cast<float*>(ws + fp.zt);
  float* lsec = reinterpret_cast<float*>(ws + fp.lsec);
  float* gsc = reinterpret_cast<float*>(ws + fp.gsc);
  float* ltok = reinterpret_cast<float*>(ws + fp.ltok);
  uint16_t* hc = reinterpret_cast<uint16_t*>(ws + fp.hc);
  float* pm = reinterpret_cast<float*>(ws + fp.pm);
  float* ps = reinterpret_cast<float*>(ws + fp.ps);
  uint16_t* G = reinterpret_cast<uint16_t*>(ws + fp.g);  // q of the chunk, then G in place
  float* slab = reinterpret_cast<float*>(ws + fp.slab);
  float* vmloc = reinterpret_cast<float*>(ws + fp.vmloc);
  float* vmglob = reinterpret_cast<float*>(ws + fp.vmglob);
  float* vsz = reinterpret_cast<float*>(ws + fp.vsz);
  float* vdh = reinterpret_cast<float*>(ws + fp.vdh);
  const float* row_grad = p->reduction == LCE_NONE ? grad_loss : nullptr;

  {
    LaunchScope sc(LCE_K_PREP, s);
    prep_kernel<<<1, 1024, 0, s>>>(labels, N, p->ignore_index, p->vocab_total, idx, yc, zt, lse, token_loss, hdr,
                                   grad_loss, p->reduction);
    LCE_TRY(last_error());
  }
  LCE_TRY(tp_sync(tp, hdr, grad_loss, p->reduction, s));
  {
    LaunchScope sc(LCE_K_GATHER, s);
    // per-row gathers and the zero dhidden rows of ignored tokens; the rows of
    // H themselves are gathered chunk by chunk below
    gather_kernel<<<static_cast<unsigned>(fp.cap), 128, 0, s>>>(hidden, fp.D, N, idx, hdr, nullptr, nullptr, nullptr,
                                                               row_grad, gsc, labels, p->ignore_index,
                                                               p->vocab_total, dhidden);
    LCE_TRY(last_error());
  }
  const int32_t Nc = static_cast<int32_t>(fp.Nc), Vl = static_cast<int32_t>(fp.Vl), D = static_cast<int32_t>(fp.D);
  CUtensorMap t_h_k, t_h_mn;  // the chunk's H_c rows (one chunk-sized buffer, refilled per chunk)
  LCE_TRY(map_kmajor(&t_h_k, hc, fp.Nc, fp.D, fp.D, BM));
  LCE_TRY(map_mnmajor(&t_h_mn, hc, fp.Nc, fp.D, fp.D));
  CUtensorMap t_w_k, t_w_mn, t_g_k, t_g_mn;
  LCE_TRY(map_kmajor(&t_w_k, weight, fp.Vl, fp.D, fp.D, b_box_rows()));
  LCE_TRY(map_mnmajor(&t_w_mn, weight, fp.Vl, fp.D, fp.D));
  LCE_TRY(map_kmajor(&t_g_k, G, fp.Nc, fp.ldv, fp.ldv, BM));
  LCE_TRY(map_mnmajor(&t_g_mn, G, fp.Nc, fp.ldv, fp.ldv));
  // Scaled-q form (R25): q relative to a per-row reference
  // (the target logit), so the row factors of G move into the dH epilogue and
  // the dW GEMM's B operand and the HBM-bound fix-up pass is skipped; chunks
  // with out-of-range rows redo their forward in the tile-max form on the GPU
  // (no host sync; under vocab parallelism each rank decides for its own
  // partials).  LCE_FUSED_SCALED=0 selects the fix-up form.
  const bool scaled = fused_scaled_env();
  float* qref = reinterpret_cast<float*>(ws + fp.qref);
  float* coef = reinterpret_cast<float*>(ws + fp.coef);
  uint16_t* hs = reinterpret_cast<uint16_t*>(ws + fp.hs);
  int32_t* qflag = reinterpret_cast<int32_t*>(ws + fp.qflag);
  int32_t* redo_rows = qflag + 1;
  CUtensorMap t_hs_mn;
  if (scaled) {
    LCE_TRY(map_mnmajor(&t_hs_mn, hs, fp.Nc, fp.D, fp.D));
    LaunchScope sc(LCE_K_GATHER, s);
    const int rows = static_cast<int>(fp.n_chunks * fp.Nc);
    target_dot_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(
        hidden, idx, weight, fp.D, yc, static_cast<int32_t>(p->vocab_start), Vl, hdr, rows, qref);
    LCE_TRY(last_error());
  }
  // vocab-parallel: the target row of W lives on one rank (the others add 0)
  if (scaled && comm) LCE_TRY(allreduce(comm, qref, static_cast<size_t>(fp.n_chunks * fp.Nc), ncclSum, s));
  lce_status_t nst;
  float* nvls_mc = nvls_buffer(comm, static_cast<size_t>(fp.Nc * fp.D * 4), s, &nst);  // LCE_NVLS=1
  LCE_TRY(nst);
  for (int64_t q = 0; q < fp.n_chunks; ++q) {
    const int32_t r0 = static_cast<int32_t>(q * fp.Nc);
    {  // S0 for the chunk: its compacted rows of H into the chunk-sized H_c
      LaunchScope sc(LCE_K_GATHER, s);
      gather_chunk_kernel<<<static_cast<unsigned>(fp.Nc), 128, 0, s>>>(hidden, fp.D, idx, hdr, r0, Nc, hc);
      LCE_TRY(last_error());
    }
    if (scaled) LCE_CUDA(cudaMemsetAsync(qflag, 0, sizeof(int32_t), s));
    // S1+S2 (+ keep q of the chunk in bf16): z = H_q W^T, LSE partials
    {
      GemmDims d{&hdr->n_valid, 0, nullptr, D, Vl, r0, Nc, 0, 0};
      EpiLse::Params ep{yc, static_cast<int32_t>(p->vocab_start), Vl, pm, ps, fp.Nc, zt, r0, nullptr, fp.ldv};
      ep.store_q = 1;
      ep.q_ref = scaled ? qref : nullptr;
      ep.q_flag = scaled ? qflag : nullptr;
      ep.dbg = getenv("LCE_DBG_FWD") ? atoi(getenv("LCE_DBG_FWD")) : 0;
      LCE_TRY(encode_map(&ep.zmap, G, fp.ldv, fp.Nc, fp.ldv, 32));
      LCE_TRY((launch_gemm<false, false, EpiLse>(LCE_K_FWD, t_h_k, t_w_k, d, ep, dev.sms, s)));
    }
    const unsigned cb = static_cast<unsigned>(fp.Nc / kRowsPerCta);
    if (!comm) {  // S3 for the chunk rows
      LaunchScope sc(LCE_K_COMBINE, s);
      combine_rows_kernel<<<cb, 256, 0, s>>>(pm, ps, static_cast<int>(fp.n_tiles), fp.Nc, r0, Nc, zt, idx, hdr, lse,
                                            token_loss, lsec, ltok, scaled ? qref : nullptr,
                                            scaled ? qflag : nullptr);
      LCE_TRY(last_error());
    } else {  // vocab-parallel S3: MAX of m, rescale, SUM of (s, z_t) over the chunk rows
      const int nt = static_cast<int>(fp.n_tiles);
      {
        LaunchScope sc(LCE_K_COMBINE, s);
        combine_chunk_vp_kernel<<<cb, 256, 0, s>>>(1, pm, ps, nt, fp.Nc, r0, Nc, zt, vmloc, vmglob, vsz, idx, hdr,
                                                   lse, token_loss, lsec, ltok);
        LCE_TRY(last_error());
      }
      LCE_TRY(allreduce(comm, vmglob, static_cast<size_t>(fp.Nc), ncclMax, s));
      {
        LaunchScope sc(LCE_K_COMBINE, s);
        combine_chunk_vp_kernel<<<cb, 256, 0, s>>>(2, pm, ps, nt, fp.Nc, r0, Nc, zt, vmloc, vmglob, vsz, idx, hdr,
                                                   lse, token_loss, lsec, ltok);
        LCE_TRY(last_error());
      }
      LCE_TRY(allreduce(comm, vsz, static_cast<size_t>(2 * fp.Nc), ncclSum, s));
      {
        LaunchScope sc(LCE_K_COMBINE, s);
        combine_chunk_vp_kernel<<<cb, 256, 0, s>>>(3, pm, ps, nt, fp.Nc, r0, Nc, zt, vmloc, vmglob, vsz, idx, hdr,
                                                   lse, token_loss, lsec, ltok, scaled ? qref : nullptr,
                                                   scaled ? qflag : nullptr);
        LCE_TRY(last_error());
      }
    }
    if (scaled) {  // row factors, scaled H chunk, target column; fallback extent
      {
        LaunchScope sc(LCE_K_BWD_G, s);
        scaled_prep_kernel<<<static_cast<unsigned>(fp.Nc), 256, 0, s>>>(
            G, fp.ldv, r0, Nc, hidden, idx, fp.D, yc, static_cast<int32_t>(p->vocab_start), Vl, lsec, zt, qref,
            row_grad ? gsc : nullptr, hdr, qflag, redo_rows, coef, hs);
        LCE_TRY(last_error());
      }
      // fallback (device-decided, empty unless a row was out of range): the
      // forward again with tile-max q, then the fix-up below
      GemmDims d{redo_rows, 0, nullptr, D, Vl, r0, Nc, 0, 0};
      EpiLse::Params ep{yc, static_cast<int32_t>(p->vocab_start), Vl, pm, ps, fp.Nc, zt, r0, nullptr, fp.ldv};
      ep.store_q = 1;
      LCE_TRY(encode_map(&ep.zmap, G, fp.ldv, fp.Nc, fp.ldv, 32));
      LCE_TRY((launch_gemm<false, false, EpiLse>(LCE_K_BWD_G, t_h_k, t_w_k, d, ep, dev.sms, s)));
    }
    {  // S4 without recompute: G = s_i (softmax - onehot) from the kept q, in place
      // (scaled form: only on the fallback)
      LaunchScope sc(LCE_K_BWD_G, s);
      fixup_q_kernel<<<static_cast<unsigned>(fp.Nc), 256, 0, s>>>(G, fp.ldv, Vl, r0, Nc, yc,
                                                                  static_cast<int32_t>(p->vocab_start), lsec,
                                                                  row_grad ? gsc : nullptr, hdr, pm, fp.Nc, zt,
                                                                  scaled ? redo_rows : nullptr);
      LCE_TRY(last_error());
    }
    LCE_TRY(chunk_grads(fp, comm, dev.sms, s, hdr, t_g_k, t_w_mn, t_g_mn, scaled ? t_hs_mn : t_h_mn, r0, slab, vdh,
                        idx, dhidden, dweight, q > 0 || accumulate_dweight, scaled ? coef : nullptr, nvls_mc));
  }
  {
    LaunchScope sc(LCE_K_COMBINE, s);
    loss_reduce_kernel<<<1, 1024, 0, s>>>(ltok, hdr, loss, n_valid, p->reduction);
    LCE_TRY(last_error());
  }
  return tp_loss(tp, loss, s);
}

size_t lce_kd_workspace_bytes(const lce_problem_t* p, int64_t teacher_dim) {
  KdPlan kp;
  if (!p || !make_kd_plan(p, teacher_dim, &kp)) return 0;
  return kp.total;
}

lce_status_t lce_kd_forward_backward(const lce_problem_t* p, lce_comm_t comm_in, int64_t teacher_dim,
                                     const uint16_t* hidden_s, const uint16_t* weight_s, const uint16_t* hidden_t,
                                     const uint16_t* weight_t, const int32_t* labels, const float* grad_loss,
                                     float* loss, float* token_loss, int32_t* n_valid, uint16_t* dhidden_s,
                                     float* dweight_s, int dweight_flags, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  NvtxCall nvtx_call("lce_kd_forward_backward");
  if (!p) return LCE_ERR_NULL;
  if (dweight_flags & ~LCE_DW_ACCUMULATE) return LCE_ERR_ARG;  // fp32 only: dW is summed over row chunks
  const bool accumulate_dweight = dweight_flags != 0;
  if (p->reduction != LCE_MEAN && p->reduction != LCE_SUM && p->reduction != LCE_NONE) return LCE_ERR_REDUCTION;
  KdPlan kp;
  if (!make_kd_plan(p, teacher_dim, &kp)) return LCE_ERR_SHAPE;
  lce_comm_t comm = vocab_comm(comm_in), tp = token_comm(comm_in);
  if (!comm && (p->vocab_start != 0 || p->vocab_local != p->vocab_total)) return LCE_ERR_COMM;
  const FusedPlan& fp = kp.f;
  if (!workspace || !weight_s || !weight_t || !loss || !dweight_s) return LCE_ERR_NULL;
  if (fp.N > 0 && (!hidden_s || !hidden_t || !labels || !dhidden_s)) return LCE_ERR_NULL;
  const void* ptrs[] = {hidden_s, weight_s, hidden_t, weight_t, labels, grad_loss, loss,
                        token_loss, n_valid, dhidden_s, dweight_s, workspace};
  for (const void* q : ptrs)
    if (q && !aligned16(q)) return LCE_ERR_ALIGN;
  if (workspace_bytes < kp.total) return LCE_ERR_WORKSPACE;
  DevInfo dev;
  LCE_TRY(device_info(&dev));
  fit_plan_to_device(&kp.f, dev.sms);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  Header* hdr = reinterpret_cast<Header*>(ws + fp.hdr);
  if (fp.N == 0) {
    if (!accumulate_dweight) LCE_CUDA(cudaMemsetAsync(dweight_s, 0, fp.Vl * fp.D * sizeof(float), s));
    if (tp) return tp_empty_rank(tp, p, hdr, grad_loss, loss, n_valid, s);
    LCE_CUDA(cudaMemsetAsync(loss, 0, sizeof(float), s));
    if (n_valid) LCE_CUDA(cudaMemsetAsync(n_valid, 0, sizeof(int32_t), s));
    return LCE_OK;
  }
  const int N = static_cast<int>(fp.N);
  int32_t* idx = reinterpret_cast<int32_t*>(ws + fp.idx);
  int32_t* yc = reinterpret_cast<int32_t*>(ws + fp.yc);
  float* zt = reinterpret_cast<float*>(ws + fp.zt);
  float* lse_s = reinterpret_cast<float*>(ws + fp.lsec);
  float* lse_t = reinterpret_cast<float*>(ws + kp.lset);
  float* vmloc = reinterpret_cast<float*>(ws + fp.vmloc);
  float* vmglob = reinterpret_cast<float*>(ws + fp.vmglob);
  float* vsz = reinterpret_cast<float*>(ws + fp.vsz);
  float* vdh = reinterpret_cast<float*>(ws + fp.vdh);
  float* gsc = reinterpret_cast<float*>(ws + fp.gsc);
  float* ltok = reinterpret_cast<float*>(ws + fp.ltok);
  uint16_t* hcs = reinterpret_cast<uint16_t*>(ws + fp.hc);
  uint16_t* hct = reinterpret_cast<uint16_t*>(ws + kp.hct);
  float* pms = reinterpret_cast<float*>(ws + fp.pm);
  float* pss = reinterpret_cast<float*>(ws + fp.ps);
  float* pmt = reinterpret_cast<float*>(ws + kp.pmt);
  float* pst = reinterpret_cast<float*>(ws + kp.pst);
  float* Zs = reinterpret_cast<float*>(ws + fp.z);
  float* Zt = reinterpret_cast<float*>(ws + kp.zt2);
  uint16_t* G = reinterpret_cast<uint16_t*>(ws + fp.g);
  const float* row_grad = p->reduction == LCE_NONE ? grad_loss : nullptr;
  // KD uses the labels only as the ignore mask (R23): no upper range check
  const int64_t no_range = (1ll << 62);
  {
    LaunchScope sc(LCE_K_PREP, s);
    prep_kernel<<<1, 1024, 0, s>>>(labels, N, p->ignore_index, no_range, idx, yc, zt, nullptr, token_loss, hdr,
                                   grad_loss, p->reduction);
    LCE_TRY(last_error());
  }
  LCE_TRY(tp_sync(tp, hdr, grad_loss, p->reduction, s));
  {
    LaunchScope sc(LCE_K_GATHER, s);
    gather_kernel<<<static_cast<unsigned>(fp.cap), 128, 0, s>>>(hidden_s, fp.D, N, idx, hdr, hcs, nullptr, nullptr,
                                                               row_grad, gsc, labels, p->ignore_index, no_range,
                                                               dhidden_s);
    gather_kernel<<<static_cast<unsigned>(fp.cap), 128, 0, s>>>(hidden_t, kp.Dt, N, idx, hdr, hct, nullptr, nullptr,
                                                               nullptr, nullptr, labels, p->ignore_index, no_range,
                                                               nullptr);
    LCE_TRY(last_error());
  }
  const int32_t Nc = static_cast<int32_t>(fp.Nc), Vl = static_cast<int32_t>(fp.Vl), D = static_cast<int32_t>(fp.D);
  const int32_t Dt = static_cast<int32_t>(kp.Dt);
  lce_status_t nst;
  float* kd_mc = nvls_buffer(comm, static_cast<size_t>(fp.Nc * fp.D * 4), s, &nst);  // LCE_NVLS=1
  LCE_TRY(nst);
  CUtensorMap t_ws_k, t_wt_k, t_ws_mn, t_g_k, t_g_mn;
  LCE_TRY(map_kmajor(&t_ws_k, weight_s, fp.Vl, fp.D, fp.D, b_box_rows()));
  LCE_TRY(map_kmajor(&t_wt_k, weight_t, fp.Vl, kp.Dt, kp.Dt, b_box_rows()));
  LCE_TRY(map_mnmajor(&t_ws_mn, weight_s, fp.Vl, fp.D, fp.D));
  LCE_TRY(map_kmajor(&t_g_k, G, fp.Nc, fp.ldv, fp.ldv, BM));
  LCE_TRY(map_mnmajor(&t_g_mn, G, fp.Nc, fp.ldv, fp.ldv));
  for (int64_t q = 0; q < fp.n_chunks; ++q) {
    const int32_t r0 = static_cast<int32_t>(q * fp.Nc);
    const uint16_t* hsq = hcs + static_cast<int64_t>(r0) * fp.D;
    const uint16_t* htq = hct + static_cast<int64_t>(r0) * kp.Dt;
    CUtensorMap t_hs_k, t_hs_mn, t_ht_k;
    LCE_TRY(map_kmajor(&t_hs_k, hsq, fp.Nc, fp.D, fp.D, BM));
    LCE_TRY(map_mnmajor(&t_hs_mn, hsq, fp.Nc, fp.D, fp.D));
    LCE_TRY(map_kmajor(&t_ht_k, htq, fp.Nc, kp.Dt, kp.Dt, BM));
    {  // student and teacher logit chunks (kept in fp32) + their LSE partials
      GemmDims ds{&hdr->n_valid, 0, nullptr, D, Vl, r0, Nc, 0, 0};
      const int32_t voff = static_cast<int32_t>(p->vocab_start);
      EpiLse::Params es{yc, voff, Vl, pms, pss, fp.Nc, zt, r0, Zs, fp.ldv};
      es.use_zmap = z_tma();
      if (es.use_zmap) LCE_TRY(map_f32_store(&es.zmap, Zs, fp.ldv, fp.Nc, fp.ldv));
      LCE_TRY((launch_gemm<false, false, EpiLse>(LCE_K_FWD, t_hs_k, t_ws_k, ds, es, dev.sms, s)));
      GemmDims dt{&hdr->n_valid, 0, nullptr, Dt, Vl, r0, Nc, 0, 0};
      EpiLse::Params et{yc, voff, Vl, pmt, pst, fp.Nc, zt, r0, Zt, fp.ldv};
      et.use_zmap = z_tma();
      if (et.use_zmap) LCE_TRY(map_f32_store(&et.zmap, Zt, fp.ldv, fp.Nc, fp.ldv));
      LCE_TRY((launch_gemm<false, false, EpiLse>(LCE_K_FWD, t_ht_k, t_wt_k, dt, et, dev.sms, s)));
    }
    const unsigned cb = static_cast<unsigned>(fp.Nc / kRowsPerCta);
    const int nt = static_cast<int>(fp.n_tiles);
    if (!comm) {  // lse_S and lse_T of the chunk rows
      LaunchScope sc(LCE_K_COMBINE, s);
      combine_rows_kernel<<<cb, 256, 0, s>>>(pms, pss, nt, fp.Nc, r0, Nc, zt, idx, hdr, nullptr, nullptr, lse_s,
                                            nullptr);
      combine_rows_kernel<<<cb, 256, 0, s>>>(pmt, pst, nt, fp.Nc, r0, Nc, zt, idx, hdr, nullptr, nullptr, lse_t,
                                            nullptr);
      LCE_TRY(last_error());
    } else {  // vocab-parallel: global lse_S, then lse_T (MAX / rescale / SUM each)
      const float* pmx[2] = {pms, pmt};
      const float* psx[2] = {pss, pst};
      float* lsex[2] = {lse_s, lse_t};
      for (int h = 0; h < 2; ++h) {
        for (int mode = 1; mode <= 3; ++mode) {
          {
            LaunchScope sc(LCE_K_COMBINE, s);
            combine_chunk_vp_kernel<<<cb, 256, 0, s>>>(mode, pmx[h], psx[h], nt, fp.Nc, r0, Nc, zt, vmloc, vmglob,
                                                       vsz, idx, hdr, nullptr, nullptr, lsex[h], nullptr);
            LCE_TRY(last_error());
          }
          if (mode == 1) LCE_TRY(allreduce(comm, vmglob, static_cast<size_t>(fp.Nc), ncclMax, s));
          if (mode == 2) LCE_TRY(allreduce(comm, vsz, static_cast<size_t>(2 * fp.Nc), ncclSum, s));
        }
      }
    }
    {  // G = s_i (p_S - p_T), l_i = lse_S - E_{p_T}[z_S] (vocab-parallel: E summed over ranks first)
      LaunchScope sc(LCE_K_BWD_G, s);
      kd_fixup_kernel<<<static_cast<unsigned>(fp.Nc), 256, 0, s>>>(Zs, Zt, fp.ldv, Vl, r0, Nc, lse_s, lse_t,
                                                                   row_grad ? gsc : nullptr, hdr, G, ltok,
                                                                   token_loss, idx, comm ? vsz : nullptr);
      LCE_TRY(last_error());
    }
    if (comm) {
      LCE_TRY(allreduce(comm, vsz, static_cast<size_t>(fp.Nc), ncclSum, s));
      LaunchScope sc(LCE_K_COMBINE, s);
      kd_loss_rows_kernel<<<static_cast<unsigned>(ceil_div(fp.Nc, 256)), 256, 0, s>>>(vsz, lse_s, r0, Nc, hdr, ltok,
                                                                                     token_loss, idx);
      LCE_TRY(last_error());
    }
    // dH_S rows of the chunk and dW_S (student head only; the teacher gets no gradient)
    LCE_TRY(chunk_grads(fp, comm, dev.sms, s, hdr, t_g_k, t_ws_mn, t_g_mn, t_hs_mn, r0, Zs, vdh, idx, dhidden_s,
                        dweight_s, q > 0 || accumulate_dweight, nullptr, kd_mc));
  }
  {
    LaunchScope sc(LCE_K_COMBINE, s);
    loss_reduce_kernel<<<1, 1024, 0, s>>>(ltok, hdr, loss, n_valid, p->reduction);
    LCE_TRY(last_error());
  }
  return tp_loss(tp, loss, s);
}

lce_status_t lce_check_device_status(void* workspace, void* stream) {
  if (!workspace) return LCE_ERR_NULL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Header h;
  LCE_CUDA(cudaMemcpyAsync(&h, workspace, sizeof(Header), cudaMemcpyDeviceToHost, s));
  LCE_CUDA(cudaStreamSynchronize(s));
  if (h.status & kStatusBadLabel) return LCE_ERR_LABEL_RANGE;
  if (h.status & kStatusUpstream) return LCE_ERR_UPSTREAM;
  return LCE_OK;
}

lce_status_t lce_expect_grad(const float* grad, float expected, void* workspace, void* stream) {
  if (!grad || !workspace) return LCE_ERR_NULL;
  if (!aligned16(workspace)) return LCE_ERR_ALIGN;
  DevInfo dev;
  LCE_TRY(device_info(&dev));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LaunchScope sc(LCE_K_FINAL, s);
  expect_grad_kernel<<<1, 1, 0, s>>>(grad, expected, static_cast<Header*>(workspace));
  return last_error();
}

lce_status_t lce_comm_get_unique_id(uint8_t id[128]) {
  if (!id) return LCE_ERR_NULL;
  NcclApi* api = nccl();
  if (!api) return LCE_ERR_NCCL;
  ncclUniqueId u;
  if (api->getUniqueId(&u) != ncclSuccess) return LCE_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(id, &u, 128);
  return LCE_OK;
}

lce_status_t lce_comm_init_mode(lce_comm_t* comm, const uint8_t id[128], int nranks, int rank, int mode) {
  if (mode != LCE_PAR_VOCAB && mode != LCE_PAR_TOKEN) return LCE_ERR_COMM;
  if (!comm || !id) return LCE_ERR_NULL;
  if (nranks < 1 || rank < 0 || rank >= nranks) return LCE_ERR_SHAPE;
  NcclApi* api = nccl();
  if (!api) return LCE_ERR_NCCL;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclComm_t c;
  if (api->commInitRank(&c, nranks, u, rank) != ncclSuccess) return LCE_ERR_NCCL;
  lce_comm_s* cs = new lce_comm_s{c, nranks, rank, mode, nullptr, nullptr, nullptr, NvlsBuf{}, nullptr};
  if (cudaStreamCreateWithFlags(&cs->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&cs->dh_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&cs->dh_reduced, cudaEventDisableTiming) != cudaSuccess) {
    api->commDestroy(c);
    delete cs;
    return LCE_ERR_CUDA;
  }
  *comm = cs;
  return LCE_OK;
}

lce_status_t lce_comm_init(lce_comm_t* comm, const uint8_t id[128], int nranks, int rank) {
  return lce_comm_init_mode(comm, id, nranks, rank, LCE_PAR_VOCAB);
}

lce_status_t lce_comm_destroy(lce_comm_t comm) {
  if (!comm) return LCE_OK;
  NcclApi* api = nccl();
  lce_status_t st = LCE_OK;
  if (api && api->commDestroy(comm->comm) != ncclSuccess) st = LCE_ERR_NCCL;
  nvls_release(comm);
  if (comm->scratch) cudaFree(comm->scratch);
  if (comm->side) cudaStreamDestroy(comm->side);
  if (comm->dh_ready) cudaEventDestroy(comm->dh_ready);
  if (comm->dh_reduced) cudaEventDestroy(comm->dh_reduced);
  delete comm;
  return st;
}

int lce_comm_size(lce_comm_t comm) { return comm ? comm->nranks : 1; }
int lce_comm_rank(lce_comm_t comm) { return comm ? comm->rank : 0; }
int lce_comm_mode(lce_comm_t comm) { return comm ? comm->mode : LCE_PAR_VOCAB; }

lce_status_t lce_comm_check(lce_comm_t comm) {
  if (!comm) return LCE_OK;
  NcclApi* api = nccl();
  if (!api || !api->getAsyncError) return LCE_ERR_NCCL;
  ncclResult_t r = ncclSuccess;
  if (api->getAsyncError(comm->comm, &r) != ncclSuccess) return LCE_ERR_NCCL;
  return (r == ncclSuccess || r == ncclInProgress) ? LCE_OK : LCE_ERR_NCCL;
}

lce_status_t lce_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = on != 0;
  return LCE_OK;
}

lce_status_t lce_profile_read_clocks(double ms[LCE_K_COUNT], int64_t launches[LCE_K_COUNT],
                                     double sm_cycles[LCE_K_COUNT], double sm_ns[LCE_K_COUNT]) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  for (int i = 0; i < LCE_K_COUNT; ++i) {
    if (ms) ms[i] = 0.0;
    if (launches) launches[i] = 0;
    if (sm_cycles) sm_cycles[i] = 0.0;
    if (sm_ns) sm_ns[i] = 0.0;
  }
  lce_status_t st = LCE_OK;
  static unsigned long long host_probe[kProbeSlots][4];
  bool have_probe = false;
  for (ProfRec& r : g_prof.recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
      st = LCE_ERR_CUDA;
    if (ms) ms[r.cls] += t;
    if (launches) launches[r.cls] += 1;
    if (r.slot >= 0 && (sm_cycles || sm_ns)) {
      if (!have_probe) {
        if (cudaMemcpyFromSymbol(host_probe, g_probe, sizeof(host_probe)) != cudaSuccess) st = LCE_ERR_CUDA;
        have_probe = true;
      }
      const unsigned long long* q = host_probe[r.slot];
      if (q[2] > q[0] && q[3] > q[1]) {
        if (sm_ns) sm_ns[r.cls] += static_cast<double>(q[2] - q[0]);
        if (sm_cycles) sm_cycles[r.cls] += static_cast<double>(q[3] - q[1]);
      }
    }
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.recs.clear();
  return st;
}

lce_status_t lce_profile_read(double ms[LCE_K_COUNT], int64_t launches[LCE_K_COUNT]) {
  return lce_profile_read_clocks(ms, launches, nullptr, nullptr);
}

lce_status_t lce_debug_gemm(const uint16_t* A, const uint16_t* B, float* C, int64_t M, int64_t N, int64_t K,
                            int a_mn, int b_mn, void* stream) {
  if (!A || !B || !C) return LCE_ERR_NULL;
  if (M <= 0 || N <= 0 || K <= 0 || M >= (1 << 30) || N >= (1 << 30) || K >= (1 << 30)) return LCE_ERR_SHAPE;
  const int64_t lda = a_mn ? M : K, ldb = b_mn ? N : K;
  if (lda % 8 || ldb % 8) return LCE_ERR_SHAPE;
  if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return LCE_ERR_ALIGN;
  DevInfo dev;
  LCE_TRY(device_info(&dev));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUtensorMap ta, tb;
  if (a_mn) LCE_TRY(map_mnmajor(&ta, A, K, M, M));
  else LCE_TRY(map_kmajor(&ta, A, M, K, K, BM));
  if (b_mn) LCE_TRY(map_mnmajor(&tb, B, K, N, N));
  else LCE_TRY(map_kmajor(&tb, B, N, K, K, b_box_rows()));
  GemmDims d{nullptr, static_cast<int32_t>(M), nullptr, static_cast<int32_t>(K), static_cast<int32_t>(N)};
  if (getenv("LCE_DEBUG_GEMM_TMA") && N % 4 == 0) {
    // diagnostics (scripts/gemm_power.py): the dW epilogue's TMA-store drain
    // instead of EpiStore's scalar stores, so the GEMM runs at mainloop speed
    // (the raster / hint defaults of kernel class LCE_DEBUG_GEMM_CLS, default the forward's)
    EpiDW::Params ep{C, N, 0, nullptr, 0};
    ep.use_map = 1;
    LCE_TRY(map_f32_store(&ep.map, C, N, M, N));
    const int cls = getenv("LCE_DEBUG_GEMM_CLS") ? atoi(getenv("LCE_DEBUG_GEMM_CLS")) : LCE_K_FWD;
    if (!a_mn && !b_mn) return launch_gemm<false, false, EpiDW>(cls, ta, tb, d, ep, dev.sms, s);
    if (!a_mn && b_mn) return launch_gemm<false, true, EpiDW>(cls, ta, tb, d, ep, dev.sms, s);
    if (a_mn && !b_mn) return launch_gemm<true, false, EpiDW>(cls, ta, tb, d, ep, dev.sms, s);
    return launch_gemm<true, true, EpiDW>(cls, ta, tb, d, ep, dev.sms, s);
  }
  EpiStore::Params ep{C, N};
  if (!a_mn && !b_mn) return launch_gemm<false, false, EpiStore>(LCE_K_FWD, ta, tb, d, ep, dev.sms, s);
  if (!a_mn && b_mn) return launch_gemm<false, true, EpiStore>(LCE_K_FWD, ta, tb, d, ep, dev.sms, s);
  if (a_mn && !b_mn) return launch_gemm<true, false, EpiStore>(LCE_K_FWD, ta, tb, d, ep, dev.sms, s);
  return launch_gemm<true, true, EpiStore>(LCE_K_FWD, ta, tb, d, ep, dev.sms, s);
}

}  // extern "C"
