// kernels.cuh -- LCE-specific epilogues for the tcgen05 mainloop and the small
// HBM-bound kernels around it.
#pragma once

#include <math.h>

#include "gemm.cuh"

namespace lce {

constexpr float kLog2e = 1.4426950408889634f;
// scaled-q mode: largest log-ratio exp(z - ref) / exp(lse - ref) kept in the bf16
// chunk (e^64 ~ 6e27: the dH accumulator over V ~ 1e5 columns stays far below
// the fp32 range); rows beyond it fall back to the tile-max form
constexpr float kScaledQMax = 64.f;
constexpr uint32_t kStatusBadLabel = 1u;
constexpr uint32_t kStatusUpstream = 2u;  // lce_expect_grad saw a different upstream gradient

// Device-side header at the start of the workspace.
struct Header {
  uint32_t status;    // error bits of the most recent call (kStatusBadLabel)
  int32_t n_valid;    // N_v of the last prep
  float c;            // gradient scale: g (sum) or g / N_v (mean), 0 if N_v = 0
  uint32_t counter;   // last-block-done counter for deterministic reductions
  int32_t mean_div;   // MEAN divisor: N_v, or under token parallelism the global N_v
  int32_t tp_nv;      // token parallelism: this rank's N_v, then all-reduced (SUM)
  int32_t tp_bad;     // token parallelism: out-of-range labels anywhere (all-reduced)
};

__device__ __forceinline__ uint16_t bf16_bits(float a) {
  const __nv_bfloat16 h = __float2bfloat16_rn(a);  // RNE
  return *reinterpret_cast<const uint16_t*>(&h);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // RNE
  return *reinterpret_cast<uint32_t*>(&h);
}

// ============================================================ S1+S2 forward epilogue
// Per row of the 128x256 logit tile (still in TMEM), two passes over the fp32
// accumulator: pass 1 takes the row max m over the tile's valid columns (cols
// >= n_cols are -inf) and the target logit if the row's label falls in this
// tile; pass 2 sums e = exp(z - m) in fp32.  Writes the partials (m, s) of
// tile column n_blk; the logits never leave the SM (the dense [B,S,V]
// tensor is never materialised).  Every path uses the same passes and the
// same summation order, so lse is bitwise identical across them.
//   fused CE path (store_q): pass 2 also stores e rounded to bf16 (2 bytes
//     per logit) -- relative to a per-row reference, q = e * exp(m - ref) =
//     exp(z - ref) (scaled-q form, q_ref set, R25), or relative to
//     the tile max (q = e in [0, 1], R24, for the G fix-up).  Logits are never
//     rounded (R8): only probabilities relative to a reference are.
//   KD path (use_zmap / z): pass 1 stores the fp32 logits.
struct EpiLse : EpiBase {
  struct Params {
    const int32_t* yc;    // [N_v] compacted labels (global vocab ids)
    int32_t label_off;    // global vocab id of GEMM column 0
    int32_t n_cols;       // valid GEMM columns (V_l)
    float* part_m;        // [n_tiles][ld]
    float* part_s;        // [n_tiles][ld]
    int64_t ld;
    float* zt;            // [N_v] target logit (single writer: the owning tile)
    int32_t row_off;      // compacted row of GEMM row 0 (row chunk of the fused path)
    float* z;             // KD path: fp32 logit chunk [rows][ldz] (cols >= n_cols: -inf), or null
    int64_t ldz;
    int32_t use_zmap;     // 1: store the fp32 chunk through `zmap` (TMA, 32x32 fp32 boxes, 128B swizzle)
    int32_t store_q;      // 1 (fused CE): store q = exp(z - m_tile) in bf16 through `zmap` (64x32 boxes)
    alignas(64) CUtensorMap zmap;
    // scaled-q mode (R25): q = exp(z - q_ref[row]) with a per-row reference
    // instead of the tile max; rows whose tile max exceeds it by more than
    // kScaledQMax raise *q_flag (the chunk is then redone in the tile-max form)
    const float* q_ref;
    int32_t* q_flag;
    int32_t dbg;  // A/B diagnostics (results wrong): 1 skip the q stores, 2 skip the whole second pass
  };
  static __device__ __forceinline__ void finish(const Params& p) {
    if ((p.use_zmap || p.store_q) && (threadIdx.x & 31) == 0) tma_store_wait_all();
  }
  // Stage this warp's 32 rows x 128 bytes in the 128B-swizzled tile (16-byte
  // unit v of row l at unit v ^ (l & 7)) and let lane 0 issue the TMA store
  // at (col, row0).  Rows >= M are stored too (never read); rows past the
  // buffer are clipped.
  static __device__ __forceinline__ void tma_rows(const Params& p, TileInfo& t, int col, const uint4 (&u)[8]) {
    const int l = t.row & 31;
    uint8_t* st = stage_next(t);  // a staging tile no pending store still reads
#pragma unroll
    for (int v = 0; v < 8; ++v) *reinterpret_cast<uint4*>(st + l * 128 + ((v ^ (l & 7)) * 16)) = u[v];
    fence_async_smem();
    __syncwarp();
    if (l == 0) {
      tma_store_2d_hint(&p.zmap, st, col, t.m0 + (t.row - l), t.st_policy);
      tma_store_commit();
    }
  }
  // kFull: every column of the tile is < n_cols (no per-element bound checks;
  // same arithmetic and summation order as the checked path)
  template <bool kStoreQ, bool kFull>
  static __device__ __forceinline__ float sum_exp(const Params& p, uint32_t taddr, TileInfo& t, float ml, float qf) {
    float s = 0.f;
    if (p.dbg == 2) return 1.f;
#pragma unroll 1
    for (int c2 = 0; c2 < BN / 64; ++c2) {
      uint32_t w[32];
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float x[32];
        load_chunk(taddr, 2 * c2 + h, t.zero_acc, x);
        const int cb = t.n0 + (2 * c2 + h) * 32;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float e0 = (kFull || cb + j < p.n_cols) ? ex2_approx(fmaf(x[j], kLog2e, -ml)) : 0.f;
          const float e1 = (kFull || cb + j + 1 < p.n_cols) ? ex2_approx(fmaf(x[j + 1], kLog2e, -ml)) : 0.f;
          a0 += e0;
          a1 += e1;
          if (kStoreQ) w[h * 16 + j / 2] = pack_bf16x2(e0 * qf, e1 * qf);  // qf = 1: exact
        }
      }
      s += a0 + a1;
      if (kStoreQ && p.dbg != 1) {
        uint4 u[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) u[v] = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
        tma_rows(p, t, t.n0 + c2 * 64, u);
      }
    }
    return s;
  }
  static __device__ __forceinline__ void apply(const Params& p, uint32_t taddr, TileInfo& t) {
    const int r = t.m0 + t.row;
    const bool valid = r < t.M;
    const int yl = valid ? (p.yc[p.row_off + r] - p.label_off - t.n0) : -1;  // tile-relative target column
    float4* zrow = (p.z && valid) ? reinterpret_cast<float4*>(p.z + static_cast<int64_t>(r) * p.ldz + t.n0) : nullptr;
    float m = -INFINITY, zt = 0.f;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float x[32];
      load_chunk(taddr, c, t.zero_acc, x);
      const int cb = t.n0 + c * 32;
      if (cb + 32 > p.n_cols) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (cb + j >= p.n_cols) x[j] = -INFINITY;
      }
      if (p.use_zmap) {
        uint4 u[8];
#pragma unroll
        for (int v = 0; v < 8; ++v)
          u[v] = make_uint4(__float_as_uint(x[4 * v]), __float_as_uint(x[4 * v + 1]), __float_as_uint(x[4 * v + 2]),
                            __float_as_uint(x[4 * v + 3]));
        tma_rows(p, t, t.n0 + c * 32, u);
      } else if (zrow) {
#pragma unroll
        for (int v = 0; v < 8; ++v) zrow[c * 8 + v] = make_float4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
      }
      if ((yl >> 5) == c) {
        const int jt = yl & 31;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j == jt) zt = x[j];
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) m = fmaxf(m, x[j]);
    }
    const float ml = (m == -INFINITY) ? 0.f : m * kLog2e;
    const bool full = t.n0 + BN <= p.n_cols;
    // scaled-q mode: the stored q is e * exp(m - ref) = exp(z - ref)
    float qf = 1.f;
    if (p.store_q && p.q_ref) {
      const float dm = m - p.q_ref[p.row_off + r];
      if (valid && dm > kScaledQMax) *p.q_flag = 1;
      qf = ex2_approx(fminf(dm, kScaledQMax) * kLog2e);
    }
    const float s = p.store_q ? (full ? sum_exp<true, true>(p, taddr, t, ml, qf) : sum_exp<true, false>(p, taddr, t, ml, qf))
                              : (full ? sum_exp<false, true>(p, taddr, t, ml, qf) : sum_exp<false, false>(p, taddr, t, ml, qf));
    if (valid) {
      p.part_m[t.n_blk * p.ld + r] = m;
      p.part_s[t.n_blk * p.ld + r] = s;
      if (yl >= 0 && yl < BN && t.n0 + yl < p.n_cols) p.zt[p.row_off + r] = zt;
    }
  }
};

// ============================================================ S4 backward G epilogue
// Recomputed logit tile -> G = exp(z - lse) - [j == y] (unscaled, A9), bf16
// RNE, into the vocab chunk buffer G_c[row, col].  Rows >= N_v and columns
// >= n_cols are written as exact zeros so the next two GEMMs can run over
// whole k-blocks.
struct EpiG : EpiBase {
  struct Params {
    const int32_t* yc;
    const float* lse_c;   // [N_v] lse of compacted rows
    int32_t label_off;    // global vocab id of chunk column 0
    int32_t n_cols;       // valid columns of this chunk
    uint16_t* G;          // [rows_cap][ldg] bf16
    int64_t ldg;
    const float* row_scale;  // [N_v] per-token upstream gradient (reduction NONE) or null
    int32_t use_gmap;        // 1: store through `gmap` (TMA, 64-col x 32-row bf16 boxes, 128B swizzle)
    alignas(64) CUtensorMap gmap;
  };
  static __device__ __forceinline__ void finish(const Params& p) {
    if (p.use_gmap && (threadIdx.x & 31) == 0) tma_store_wait_all();
  }
  // G of one 32-column chunk of this thread's row, as 16 packed bf16 pairs.
  static __device__ __forceinline__ void g_chunk(const Params& p, uint32_t taddr, const TileInfo& t, int c,
                                                 bool valid, int yl, float lsel, float rs, uint32_t* w) {
    float x[32];
    load_chunk(taddr, c, t.zero_acc, x);
    const int cb = t.n0 + c * 32;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      float g0 = ex2_approx(fmaf(x[j], kLog2e, -lsel)) - (c * 32 + j == yl ? 1.f : 0.f);
      float g1 = ex2_approx(fmaf(x[j + 1], kLog2e, -lsel)) - (c * 32 + j + 1 == yl ? 1.f : 0.f);
      g0 = (!valid || cb + j >= p.n_cols) ? 0.f : g0 * rs;
      g1 = (!valid || cb + j + 1 >= p.n_cols) ? 0.f : g1 * rs;
      w[j / 2] = pack_bf16x2(g0, g1);
    }
  }
  static __device__ __forceinline__ void apply(const Params& p, uint32_t taddr, TileInfo& t) {
    const int r = t.m0 + t.row;
    const bool valid = r < t.M;
    const int yl = valid ? (p.yc[r] - p.label_off - t.n0) : -1;
    const float lsel = valid ? p.lse_c[r] * kLog2e : 0.f;
    const float rs = (valid && p.row_scale) ? p.row_scale[r] : 1.f;
    if (p.use_gmap) {
      // Two chunks (64 bf16 = 128 bytes per row) per TMA store: each lane
      // writes its row into the 128B-swizzled staging tile (16-byte unit v of
      // row l at unit v ^ (l & 7)), lane 0 issues the store.  Rows >= M are
      // stored as zeros; rows/columns past the buffer are clipped by TMA.
      const int l = t.row & 31;
#pragma unroll 1
      for (int c2 = 0; c2 < BN / 64; ++c2) {
        uint32_t w[32];
        g_chunk(p, taddr, t, 2 * c2, valid, yl, lsel, rs, w);
        g_chunk(p, taddr, t, 2 * c2 + 1, valid, yl, lsel, rs, w + 16);
        uint8_t* st = stage_next(t);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<uint4*>(st + l * 128 + ((v ^ (l & 7)) * 16)) =
              make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
        fence_async_smem();
        __syncwarp();
        if (l == 0) {
          tma_store_2d_hint(&p.gmap, st, t.n0 + c2 * 64, t.m0 + (t.row - l), t.st_policy);
          tma_store_commit();
        }
      }
      return;
    }
    uint4* dst = reinterpret_cast<uint4*>(p.G + static_cast<int64_t>(r) * p.ldg + t.n0);
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t w[16];
      g_chunk(p, taddr, t, c, valid, yl, lsel, rs, w);
#pragma unroll
      for (int v = 0; v < 4; ++v) dst[c * 4 + v] = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
    }
  }
};

// ============================================================ S6 dH epilogue
// acc = (G_c W_c)[row, cols] for vocab chunk k.  Chunks are summed unscaled
// in fp32 (acc_buf); on the last chunk (single GPU) the sum is scaled by c,
// rounded to bf16 and scattered to dhidden[idx[row]] directly.
struct EpiDH : EpiBase {
  struct Params {
    float* acc_buf;        // [rows_cap][ld] fp32 running sum over chunks
    int64_t ld;            // D
    int32_t first;         // first chunk: overwrite acc_buf
    int32_t last_direct;   // last chunk and no cross-rank reduction: write dhidden
    const Header* hdr;     // c
    uint16_t* dhidden;     // [N][D] bf16
    const int32_t* idx;    // compact row -> token row
    int32_t row_off;       // compacted row of GEMM row 0
    int32_t use_c;         // 1: scale by c on output; 0: c already folded into G
    float* part;           // split-K: fp32 partial slabs [ksplit][rows][ld] (reduced by reduce_dh_kernel)
    int64_t part_stride;   // elements per slab
    int32_t use_map;       // 1: accumulate into acc_buf through `map` with TMA stores (first chunk) /
                           //    TMA reduce-adds (the L2 adds; no read by the SM); unscaled, a
                           //    finalize pass applies c, rounds and scatters
    alignas(64) CUtensorMap map;  // acc_buf [rows, ld] fp32, 32 x 32 boxes, 128B swizzle
    const float* row_coef;  // scaled-q mode: per chunk-row factor s_i beta_i of the direct path (null: none)
    // NVLS (vocab-parallel, LCE_NVLS=1): add row r of the (row_coef-scaled)
    // accumulator into the multicast-mapped fp32 buffer [rows][ld]: the switch
    // sums every rank's (and every split-K item's) partial into every GPU's
    // copy -- the dH all-reduce fused into this epilogue
    float* mc_out;
    int32_t mc_unicast;  // LCE_NVLS=2 (one-rank emulation): plain red.global.add into a unicast buffer
  };
  // pull the running fp32 sum of this tile's row into L2 while the MMA runs
  static __device__ __forceinline__ void prefetch(const Params& p, const TileInfo& t) {
    const int r = t.m0 + t.row;
    if (p.part || p.first || p.use_map || r >= t.M) return;
    const float* row = p.acc_buf + static_cast<int64_t>(p.row_off + r) * p.ld;
    for (int c = 0; c < BN / 32 && t.n0 + 32 * c < t.N; ++c) prefetch_l2(row + t.n0 + 32 * c);
  }
  static __device__ __forceinline__ void finish(const Params& p) {
    if (p.use_map && (threadIdx.x & 31) == 0) tma_store_wait_all();
  }
  static __device__ __forceinline__ void apply(const Params& p, uint32_t taddr, TileInfo& t) {
    const int r = t.m0 + t.row;
    const bool valid = r < t.M;
    if (p.mc_out) {  // NVLS: in-switch reduction straight from registers
      const float rc = (p.row_coef && valid) ? p.row_coef[r] : 1.f;
      float* orow = p.mc_out + static_cast<int64_t>(r) * p.ld;
      uint32_t v[2][32];
      tmem_ld32(taddr, v[0]);
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        tmem_ld_wait();
        if (c + 1 < BN / 32) tmem_ld32(taddr + (c + 1) * 32, v[(c + 1) & 1]);
        const uint32_t* u = v[c & 1];
        const int cb = t.n0 + c * 32;
        if (!valid || t.zero_acc || cb >= t.N) continue;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int col = cb + 4 * q;
          if (col >= t.N) break;
          const float a = rc * __uint_as_float(u[4 * q]), b = rc * __uint_as_float(u[4 * q + 1]);
          const float c2 = rc * __uint_as_float(u[4 * q + 2]), d = rc * __uint_as_float(u[4 * q + 3]);
          if (p.mc_unicast)
            red_add_v4(orow + col, a, b, c2, d);
          else
            multimem_red_add_v4(orow + col, a, b, c2, d);
        }
      }
      return;
    }
    if (p.use_map && !p.part) {  // TMA store / reduce-add of the unscaled chunk sum
      const int l = t.row & 31;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float x[32];
        load_chunk(taddr, c, t.zero_acc, x);
        if (t.n0 + c * 32 >= t.N) continue;  // uniform across the warp
        uint8_t* st = stage_next(t);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(st + l * 128 + ((v ^ (l & 7)) * 16)) =
              make_float4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
        fence_async_smem();
        __syncwarp();
        if (l == 0) {
          if (p.first)
            tma_store_2d_hint(&p.map, st, t.n0 + c * 32, t.m0 + (t.row - l), t.st_policy);
          else
            tma_reduce_add_2d_hint(&p.map, st, t.n0 + c * 32, t.m0 + (t.row - l), t.st_policy);
          tma_store_commit();
        }
      }
      return;
    }
    if (p.part && p.use_map) {  // split-K partial through TMA stores (map over [split * rows, ld] slabs)
      const int l = t.row & 31;
      const float rc = (p.row_coef && valid) ? p.row_coef[r] : 1.f;
      const int slab_rows = static_cast<int>(p.part_stride / p.ld);
      // a warp's 32-row box past the slab's rows (a wide tile taller than the
      // chunk) would land in the next slab: skip it (uniform across the warp)
      if (t.m0 + (t.row - l) >= slab_rows) return;
      const int grow = t.split * slab_rows + t.m0 + (t.row - l);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float x[32];
        load_chunk(taddr, c, t.zero_acc, x);
        if (t.n0 + c * 32 >= t.N) continue;  // uniform across the warp
        uint8_t* st = stage_next(t);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(st + l * 128 + ((v ^ (l & 7)) * 16)) =
              make_float4(rc * x[4 * v], rc * x[4 * v + 1], rc * x[4 * v + 2], rc * x[4 * v + 3]);
        fence_async_smem();
        __syncwarp();
        if (l == 0) {
          tma_store_2d_hint(&p.map, st, t.n0 + c * 32, grow, t.st_policy);
          tma_store_commit();
        }
      }
      return;
    }
    if (p.part) {  // split-K partial: plain fp32 store, no read-modify-write
      float* prow = p.part + t.split * p.part_stride + static_cast<int64_t>(r) * p.ld;
      const float rc = (p.row_coef && valid) ? p.row_coef[r] : 1.f;  // linear: each slab scaled
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float x[32];
        load_chunk(taddr, c, t.zero_acc, x);
        const int cb = t.n0 + c * 32;
        if (!valid) continue;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int col = cb + 4 * v;
          if (col >= t.N) break;
          *reinterpret_cast<float4*>(prow + col) =
              make_float4(rc * x[4 * v], rc * x[4 * v + 1], rc * x[4 * v + 2], rc * x[4 * v + 3]);
        }
      }
      return;
    }
    const float cs = ((p.last_direct && p.use_c) ? p.hdr->c : 1.f) * ((p.row_coef && valid) ? p.row_coef[r] : 1.f);
    float* accrow = p.acc_buf + static_cast<int64_t>(p.row_off + r) * p.ld;
    uint16_t* orow = nullptr;
    if (valid && p.last_direct) orow = p.dhidden + static_cast<int64_t>(p.idx[p.row_off + r]) * p.ld;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float x[32];
      load_chunk(taddr, c, t.zero_acc, x);
      const int cb = t.n0 + c * 32;
      if (!valid) continue;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int col = cb + 4 * v;
        if (col >= t.N) break;
        float4 a = make_float4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
        if (!p.first) {
          const float4 o = *reinterpret_cast<const float4*>(accrow + col);
          a.x += o.x;
          a.y += o.y;
          a.z += o.z;
          a.w += o.w;
        }
        if (p.last_direct) {
          uint2 h = make_uint2(pack_bf16x2(cs * a.x, cs * a.y), pack_bf16x2(cs * a.z, cs * a.w));
          *reinterpret_cast<uint2*>(orow + col) = h;
        } else {
          *reinterpret_cast<float4*>(accrow + col) = a;
        }
      }
    }
  }
};

// ============================================================ S5 dW epilogue
// acc = (G_c^T H)[vocab row, cols]; dW rows of the chunk = c * acc (or +=).
struct EpiDW : EpiBase {
  struct Params {
    float* dW;            // chunk row 0 of dweight
    int64_t ld;           // D
    int32_t accumulate;
    const Header* hdr;
    int32_t use_c;        // 1: scale by c; 0: c already folded into G
    int32_t use_map;      // 1: write through `map` (fp32 32x32 boxes, 128B swizzle): TMA store,
                          //    or TMA reduce-add when accumulating (the L2 adds; no read by the SM)
    alignas(64) CUtensorMap map;  // [M rows of this GEMM, D] (rows / cols past it are clipped)
    int32_t dbg;                  // A/B diagnostics: 1 skip the writes, 2 also the TMEM reads,
                                  // 3 / 4 skip the writes of accumulating / overwriting launches only
    uint16_t* dw_bf16;            // non-null: write bf16(c * acc) rows here instead (LCE_DW_BF16,
                                  // overwrite only; the direct path)
    int32_t prefetch;             // accumulate + TMA: L2 prefetch of the old dW rows
  };
  static __device__ __forceinline__ void finish(const Params& p) {
    if (p.use_map && (threadIdx.x & 31) == 0) tma_store_wait_all();
  }
  // Accumulating (the fused path's later row chunks): the TMA reduce-add needs
  // the old dW lines in L2; pull this tile's rows in (one bulk prefetch per
  // row) while the MMA computes the tile, so the adds do not wait on HBM.
  static __device__ __forceinline__ void prefetch(const Params& p, const TileInfo& t) {
    const int r = t.m0 + t.row;
    if (!p.use_map || !p.accumulate || !p.prefetch || t.zero_acc || r >= t.M || t.n0 >= t.N) return;
    const int cols = min(BN, t.N - t.n0);
    bulk_prefetch_l2(p.dW + static_cast<int64_t>(r) * p.ld + t.n0, static_cast<uint32_t>(cols * 4));
  }
  static __device__ __forceinline__ void apply(const Params& p, uint32_t taddr, TileInfo& t) {
    if (t.zero_acc && p.accumulate) return;  // K == 0 adds nothing (uniform across the CTA)
    if (p.dbg == 1 || p.dbg == 2 || (p.dbg == 3 && p.accumulate) || (p.dbg == 4 && !p.accumulate)) {
      if (p.dbg != 2) {
        float x[32];
        for (int c = 0; c < BN / 32; ++c) load_chunk(taddr, c, false, x);
        if (x[0] == 12345.f) *p.dW = x[1];  // keep the loads
      }
      return;
    }
    const int r = t.m0 + t.row;
    const bool valid = r < t.M;
    const float cs = p.use_c ? p.hdr->c : 1.f;
    if (p.use_map) {
      const int l = t.row & 31;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float x[32];
        load_chunk(taddr, c, t.zero_acc, x);
        if (t.n0 + c * 32 >= t.N) continue;  // uniform across the warp
        uint8_t* st = stage_next(t);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(st + l * 128 + ((v ^ (l & 7)) * 16)) =
              make_float4(cs * x[4 * v], cs * x[4 * v + 1], cs * x[4 * v + 2], cs * x[4 * v + 3]);
        fence_async_smem();
        __syncwarp();
        if (l == 0) {
          if (p.accumulate)
            tma_reduce_add_2d_hint(&p.map, st, t.n0 + c * 32, t.m0 + (t.row - l), t.st_policy);
          else
            tma_store_2d_hint(&p.map, st, t.n0 + c * 32, t.m0 + (t.row - l), t.st_policy);
          tma_store_commit();
        }
      }
      return;
    }
    // Direct path: straight from registers to global memory (16-byte stores,
    // or L2 reduce-adds when accumulating; bf16 rows for LCE_DW_BF16).
    // Chunk c + 1's TMEM load is in flight while chunk c is written.
    float* row = p.dW + static_cast<int64_t>(r) * p.ld;
    uint16_t* brow = p.dw_bf16 ? p.dw_bf16 + static_cast<int64_t>(r) * p.ld : nullptr;
    uint32_t v[2][32];
    tmem_ld32(taddr, v[0]);
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      tmem_ld_wait();
      if (c + 1 < BN / 32) tmem_ld32(taddr + (c + 1) * 32, v[(c + 1) & 1]);
      const uint32_t* u = v[c & 1];
      const int cb = t.n0 + c * 32;
      if (!valid || cb >= t.N) continue;
      if (brow) {  // D % 8 == 0: a group of 8 columns is either all in range or all out
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col = cb + 8 * q;
          if (col >= t.N) break;
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            w[e] = t.zero_acc ? 0u
                              : pack_bf16x2(cs * __uint_as_float(u[8 * q + 2 * e]),
                                            cs * __uint_as_float(u[8 * q + 2 * e + 1]));
          *reinterpret_cast<uint4*>(brow + col) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        continue;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int col = cb + 4 * q;
        if (col >= t.N) break;
        float a[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) a[e] = t.zero_acc ? 0.f : cs * __uint_as_float(u[4 * q + e]);
        if (p.accumulate)
          red_add_v4(row + col, a[0], a[1], a[2], a[3]);
        else
          st_global_v4(row + col, a[0], a[1], a[2], a[3]);
      }
    }
  }
};

// ============================================================ NEXT-2: AdamW in the dW epilogue
// Optimizer-in-backward for the LM head (Sec. 4.1): a dW row block
// is final when its tile leaves TMEM (the V-chunked backward writes each dW row
// exactly once), so the epilogue applies the AdamW step there and no dW buffer
// exists.  torch.optim.AdamW order: theta *= 1 - lr wd;
// m = b1 m + (1 - b1) g; v = b2 v + (1 - b2) g^2;
// theta -= (lr / bc1) m / (sqrt(v) / sqrt(bc2) + eps); W = bf16(theta).
struct EpiAdamW : EpiBase {
  struct Params {
    float* theta;         // fp32 master weights, chunk row 0
    float* exp_avg;
    float* exp_avg_sq;
    uint16_t* w;          // bf16 weights used by the GEMMs, rewritten
    int64_t ld;           // D
    const Header* hdr;    // c
    float lr, beta1, beta2, eps, decay;  // decay = 1 - lr * weight_decay
    float step_size, sqrt_bc2;           // lr / bc1, sqrt(bc2)
  };
  // theta, m, v rows of the tile are read-modify-written: pull them into L2 early
  static __device__ __forceinline__ void prefetch(const Params& p, const TileInfo& t) {
    const int r = t.m0 + t.row;
    if (r >= t.M) return;
    const int64_t o = static_cast<int64_t>(r) * p.ld;
    for (int c = 0; c < BN / 32 && t.n0 + 32 * c < t.N; ++c) {
      prefetch_l2(p.theta + o + t.n0 + 32 * c);
      prefetch_l2(p.exp_avg + o + t.n0 + 32 * c);
      prefetch_l2(p.exp_avg_sq + o + t.n0 + 32 * c);
    }
  }
  // Each warp owns 32 accumulator rows (one per lane, its TMEM lane quarter).
  // Per 32-column chunk the lanes stage g = c * acc in shared memory (row per
  // lane), then walk the 32 rows with one COLUMN per lane, so every load and
  // store of theta / m / v / w is one coalesced 128-byte (64-byte for w) row
  // segment per warp instruction instead of 32 half-used sectors.
  static __device__ __forceinline__ void apply(const Params& p, uint32_t taddr, TileInfo& t) {
    const int l = t.row & 31;
    const int row0 = t.m0 + (t.row - l);  // first row of this warp's 32
    const float cs = p.hdr->c;
    float* st = reinterpret_cast<float*>(t.smem);  // 32 x 32 fp32 (no TMA stores in this epilogue)
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float x[32];
      load_chunk(taddr, c, t.zero_acc, x);
      const int cb = t.n0 + c * 32;
      if (cb >= t.N) break;  // uniform across the warp
      __syncwarp();          // the previous chunk's reads of st are done
#pragma unroll
      for (int v = 0; v < 8; ++v)  // row l, 16-byte unit v at unit v ^ (l & 7): conflict-free both ways
        *reinterpret_cast<float4*>(st + l * 32 + ((v ^ (l & 7)) * 4)) =
            make_float4(cs * x[4 * v], cs * x[4 * v + 1], cs * x[4 * v + 2], cs * x[4 * v + 3]);
      __syncwarp();
      const int col = cb + l;
      const int rows = (col < t.N) ? min(32, t.M - row0) : 0;
      // 16 rows at a time: their 48 state loads are in flight together
#pragma unroll 1
      for (int r0 = 0; r0 < 32; r0 += kRowsInFlight) {
        float th[kRowsInFlight], m[kRowsInFlight], v[kRowsInFlight];
#pragma unroll
        for (int i = 0; i < kRowsInFlight; ++i) {
          if (r0 + i < rows) {
            const int64_t o = static_cast<int64_t>(row0 + r0 + i) * p.ld + col;
            th[i] = p.theta[o];
            m[i] = p.exp_avg[o];
            v[i] = p.exp_avg_sq[o];
          }
        }
#pragma unroll
        for (int i = 0; i < kRowsInFlight; ++i) {
          const int r = r0 + i;
          if (r < rows) {
            const float g = st[r * 32 + ((((l >> 2) ^ (r & 7)) << 2) | (l & 3))];
            step1(p, g, th[i], m[i], v[i]);
            const int64_t o = static_cast<int64_t>(row0 + r) * p.ld + col;
            p.theta[o] = th[i];
            p.exp_avg[o] = m[i];
            p.exp_avg_sq[o] = v[i];
            p.w[o] = bf16_bits(th[i]);
          }
        }
      }
    }
  }
  static constexpr int kRowsInFlight = 32;
  // torch.optim.AdamW's single-tensor update order (R22) on one element (g = c * dW)
  static __device__ __forceinline__ void step1(const Params& p, float g, float& th, float& m, float& v) {
    th = th * p.decay;
    m = m + (1.f - p.beta1) * (g - m);  // torch: exp_avg.lerp_(grad, 1 - beta1)
    v = p.beta2 * v + (1.f - p.beta2) * g * g;
    const float denom = __fdiv_rn(__fsqrt_rn(v), p.sqrt_bc2) + p.eps;
    th = th - p.step_size * __fdiv_rn(m, denom);
  }
};

// ============================================================ diagnostics epilogue
struct EpiStore : EpiBase {
  struct Params {
    float* C;
    int64_t ldc;
  };
  static __device__ __forceinline__ void apply(const Params& p, uint32_t taddr, const TileInfo& t) {
    const int r = t.m0 + t.row;
    const bool valid = r < t.M;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float x[32];
      load_chunk(taddr, c, t.zero_acc, x);
      if (!valid) continue;
      for (int j = 0; j < 32; ++j) {
        const int col = t.n0 + c * 32 + j;
        if (col < t.N) p.C[static_cast<int64_t>(r) * p.ldc + col] = x[j];
      }
    }
  }
};

// ============================================================ S0 prep
// Label scan + stable compaction (one CTA, 1024 threads, 4 labels per thread
// per pass).  Mask-first: only rows with y != ignore_index and y in
// [0, V) enter idx[]; out-of-range labels set the status bit of this call.  Writes
// N_v and the gradient scale c into the header, zeroes lse / token_loss of
// excluded rows and zt of compacted rows.
__global__ void __launch_bounds__(1024) prep_kernel(const int32_t* __restrict__ y, int N, int32_t ignore,
                                                    int64_t vocab_total, int32_t* __restrict__ idx,
                                                    int32_t* __restrict__ yc, float* __restrict__ zt,
                                                    float* __restrict__ lse_out, float* __restrict__ tok_out,
                                                    Header* hdr, const float* __restrict__ grad_loss,
                                                    int reduction) {
  // grad_loss is a device scalar for MEAN / SUM and ignored for NONE
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  bool bad_any = false;
  for (int start = 0; start < N; start += 4096) {
    int flags[4];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = start + tid * 4 + u;
      int f = 0;
      if (i < N) {
        const int32_t l = y[i];
        if (l != ignore) {
          if (l >= 0 && static_cast<int64_t>(l) < vocab_total) {
            f = 1;
          } else {
            bad_any = true;
          }
        }
        if (!f) {
          if (lse_out) lse_out[i] = 0.f;
          if (tok_out) tok_out[i] = 0.f;
        }
      }
      flags[u] = f;
      cnt += f;
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int w = warp_tot[lane];
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += v;
      }
      warp_tot[lane] = wi - w;  // exclusive
    }
    __syncthreads();
    int pos = base_s + warp_tot[wid] + incl - cnt;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (flags[u]) {
        const int i = start + tid * 4 + u;
        idx[pos] = i;
        yc[pos] = y[i];
        zt[pos] = 0.f;
        ++pos;
      }
    }
    __syncthreads();
    if (tid == 1023) base_s = pos;
    __syncthreads();
  }
  const int any_bad = __syncthreads_or(bad_any ? 1 : 0);
  // target logits of the padding rows [N_v, ceil256(N)) are defined too (0):
  // the vocab-parallel exchange copies all of them
  if (zt)
    for (int i = base_s + tid; i < ((N + 255) & ~255); i += 1024) zt[i] = 0.f;
  if (tid == 0) {
    hdr->status = any_bad ? kStatusBadLabel : 0u;
    const int nv = base_s;
    hdr->n_valid = nv;
    const float g = (grad_loss && reduction != 2) ? *grad_loss : 1.f;
    // MEAN: g / N_v, SUM: g, NONE: 1 (per-token upstream grads are folded into G)
    hdr->c = nv == 0 ? 0.f : (reduction == 0 ? g / static_cast<float>(nv) : (reduction == 1 ? g : 1.f));
    hdr->counter = 0u;
    hdr->mean_div = nv;
    hdr->tp_nv = nv;
    hdr->tp_bad = any_bad ? 1 : 0;
  }
}

// Token parallelism (rows sharded over ranks, W replicated): after the
// all-reduce of (tp_nv, tp_bad), MEAN divides by the global N_v -- in the
// gradient scale c and in the loss -- so the per-rank losses and gradients sum
// to the full batch's.
__global__ void tp_scale_kernel(Header* hdr, const float* __restrict__ grad_loss, int reduction) {
  const int nv = hdr->tp_nv;
  // a bad label on any rank poisons the summed loss on every rank: report it on every rank too
  if (hdr->tp_bad) hdr->status |= kStatusBadLabel;
  const float g = (grad_loss && reduction != 2) ? *grad_loss : 1.f;
  hdr->mean_div = nv;
  if (hdr->n_valid > 0 && reduction == 0) hdr->c = nv == 0 ? 0.f : g / static_cast<float>(nv);
}

// NVLS barrier across the ranks of a multicast buffer: every rank release-adds
// 1 to the counter in every GPU's copy (through the switch), then waits until
// its own copy reaches `target` (= barriers so far x ranks).  The fence makes
// this stream's earlier multimem reductions visible system-wide first.
__global__ void nvls_barrier_kernel(uint32_t* mc_flag, const uint32_t* uc_flag, uint32_t target, int unicast) {
  if (threadIdx.x != 0) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (unicast)
    atomicAdd(mc_flag, 1u);
  else
    multimem_red_release_add_u32(mc_flag, 1u);
  SpinGuard g;
  while (ld_acquire_sys_u32(uc_flag) < target) g.tick("NVLS flag", target, 0);
}

// lce_expect_grad: the upstream gradient the fused call assumed vs the actual one.
__global__ void expect_grad_kernel(const float* __restrict__ grad, float expected, Header* hdr) {
  if (*grad != expected) hdr->status |= kStatusUpstream;
}

// ============================================================ S0 gather
// Block b: compact row b <- H[idx[b]] (zeros for b in [N_v, ceil256(N_v)) so
// whole 256-row pair tiles and 64-row k-blocks read finite zeros), optional lse
// gather for the backward, optional zeroing of dhidden row b if token b is
// excluded (ignored or bad label: its gradient is exactly 0).
__global__ void __launch_bounds__(128) gather_kernel(const uint16_t* __restrict__ H, int64_t D, int N,
                                                     const int32_t* __restrict__ idx, const Header* hdr,
                                                     uint16_t* __restrict__ Hc, const float* __restrict__ lse_in,
                                                     float* __restrict__ lse_c, const float* __restrict__ grad_in,
                                                     float* __restrict__ grad_c, const int32_t* __restrict__ y,
                                                     int32_t ignore, int64_t vocab_total,
                                                     uint16_t* __restrict__ dhidden) {
  const int b = blockIdx.x;
  const int nv = hdr->n_valid;
  const int nvec = static_cast<int>(D / 8);
  // Hc == null (fused path: per-chunk H_c, gather_chunk_kernel): no copy,
  // only the per-row gathers and the zero rows of dhidden
  uint4* dst = Hc ? reinterpret_cast<uint4*>(Hc + static_cast<int64_t>(b) * D) : nullptr;
  if (b < nv) {
    const int src_row = idx[b];
    const uint4* src = reinterpret_cast<const uint4*>(H + static_cast<int64_t>(src_row) * D);
    if (dst)
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = __ldg(src + v);
    if (lse_in && threadIdx.x == 0) lse_c[b] = lse_in[src_row];
    if (grad_in && threadIdx.x == 0) grad_c[b] = grad_in[src_row];
  } else if (dst && b < ((nv + 255) & ~255)) {  // up to the 256-row pair tile: no stale row enters a GEMM
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = make_uint4(0, 0, 0, 0);
  }
  if (dhidden && b < N) {
    const int32_t l = y[b];
    const bool kept = l != ignore && l >= 0 && static_cast<int64_t>(l) < vocab_total;
    if (!kept) {
      uint4* o = reinterpret_cast<uint4*>(dhidden + static_cast<int64_t>(b) * D);
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) o[v] = make_uint4(0, 0, 0, 0);
    }
  }
}

// Fused path: the compacted rows of one row chunk, [r0, r0 + cap), into a
// chunk-sized H_c (one CTA per chunk row): rows < M = clamp(N_v - r0, 0, cap)
// are hidden[idx[r0 + b]], rows [M, ceil256(M)) are zeroed (the GEMMs' last
// pair tile reads them; zero rows keep every logit finite).  The whole-batch
// H_c (2 N_v D bytes: 4.3 GB at 1M tokens of the 1B head) is never built.
__global__ void __launch_bounds__(128) gather_chunk_kernel(const uint16_t* __restrict__ H, int64_t D,
                                                           const int32_t* __restrict__ idx, const Header* hdr,
                                                           int row_off, int cap, uint16_t* __restrict__ Hc) {
  const int b = blockIdx.x;
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  const int nvec = static_cast<int>(D / 8);
  uint4* dst = reinterpret_cast<uint4*>(Hc + static_cast<int64_t>(b) * D);
  if (b < M) {
    const uint4* src = reinterpret_cast<const uint4*>(H + static_cast<int64_t>(idx[row_off + b]) * D);
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = __ldg(src + v);
  } else if (b < ((M + 255) & ~255)) {
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = make_uint4(0, 0, 0, 0);
  }
}

// ============================================================ S3 combine (+ loss)
// mode 0 (one GPU): partials -> lse, token loss, loss (fixed-order, fp64 sum).
// mode 1 (vocab-parallel, before the MAX all-reduce): partials -> local
//   (m_loc, s_loc); m_loc also copied to m_glob for the in-place all-reduce.
// mode 2 (after MAX all-reduce): s_loc *= exp(m_loc - M) for the SUM all-reduce.
// mode 3 (after SUM all-reduce of (s, zt)): lse = M + ln s, token loss, loss.
constexpr int kRowsPerCta = 8;  // combine kernels: one warp per row

// Merge of one row's per-vocab-tile partials (m_t, s_t) by a whole warp:
// M = max_t m_t, S = sum_t s_t e^{m_t - M}.  Lanes stride over the tiles and
// reduce with a fixed xor-shuffle tree, so the result is deterministic and
// identical in every lane.  (A thread per row was latency-bound: ~0.2 ms per
// 4096-row chunk at T_v = 501.)
__device__ __forceinline__ void row_merge_warp(const float* __restrict__ pm, const float* __restrict__ ps,
                                               int n_tiles, int64_t ld, int m, float& M, float& S) {
  const int lane = threadIdx.x & 31;
  float mx = -INFINITY;
  for (int t = lane; t < n_tiles; t += 32) mx = fmaxf(mx, pm[t * ld + m]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = 0.f;
  for (int t = lane; t < n_tiles; t += 32) s += ps[t * ld + m] * expf(pm[t * ld + m] - mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  M = mx;
  S = s;
}

__device__ __forceinline__ void block_loss_reduce(double li, double* block_sums, Header* hdr, float* loss,
                                                  int32_t* n_valid_out, int nv, int reduction) {
  __shared__ double red[256];
  __shared__ bool last;
  red[threadIdx.x] = li;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    block_sums[blockIdx.x] = red[0];
    __threadfence();
    const uint32_t done = atomicAdd(&hdr->counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    // fixed-order final sum: each thread a strided slice, then the same tree
    double acc = 0.0;
    for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += 256)
      acc += reinterpret_cast<volatile double*>(block_sums)[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      double L = red[0];
      const int nd = hdr->mean_div;
      if (reduction == 0) L = nd > 0 ? L / nd : 0.0;
      if (hdr->status & kStatusBadLabel) L = __longlong_as_double(0x7ff8000000000000ULL);
      *loss = static_cast<float>(L);
      if (n_valid_out) *n_valid_out = nd;
      hdr->counter = 0u;
    }
  }
}

__global__ void __launch_bounds__(256) combine_kernel(int mode, const float* __restrict__ pm,
                                                      const float* __restrict__ ps, int n_tiles, int64_t ld,
                                                      float* __restrict__ m_loc, float* __restrict__ m_glob,
                                                      float* __restrict__ s_buf, const float* __restrict__ zt,
                                                      const int32_t* __restrict__ idx, Header* hdr,
                                                      float* __restrict__ lse_out, float* __restrict__ tok_out,
                                                      double* __restrict__ block_sums, float* __restrict__ loss,
                                                      int32_t* __restrict__ n_valid_out, int reduction) {
  // one warp per compacted row (8 rows per CTA); lane 0 owns the row's outputs
  const int r = blockIdx.x * kRowsPerCta + (threadIdx.x >> 5);
  const bool lead = (threadIdx.x & 31) == 0;
  const int nv = hdr->n_valid;
  const bool valid = r < nv;
  if (mode == 0 || mode == 1) {
    float M = -INFINITY, S = 0.f;
    if (valid) row_merge_warp(pm, ps, n_tiles, ld, r, M, S);
    if (mode == 1) {
      if (valid && lead) {
        m_loc[r] = M;
        m_glob[r] = M;
        s_buf[r] = S;
      }
      return;
    }
    double li = 0.0;
    if (valid && lead) {
      const float lse = M + logf(S);
      const float l = lse - zt[r];
      const int i = idx[r];
      lse_out[i] = lse;
      if (tok_out) tok_out[i] = l;
      li = l;
    }
    block_loss_reduce(li, block_sums, hdr, loss, n_valid_out, nv, reduction);
    return;
  }
  if (mode == 2) {
    if (valid && lead) s_buf[r] *= expf(m_loc[r] - m_glob[r]);
    return;
  }
  // mode 3
  double li = 0.0;
  if (valid && lead) {
    const float lse = m_glob[r] + logf(s_buf[r]);
    const float l = lse - zt[r];
    const int i = idx[r];
    lse_out[i] = lse;
    if (tok_out) tok_out[i] = l;
    li = l;
  }
  block_loss_reduce(li, block_sums, hdr, loss, n_valid_out, nv, reduction);
}

// ============================================================ S7 finalize (multi-GPU)
// dhidden[idx[r]] = bf16(c * dH_sum[r]) after the cross-rank all-reduce.
__global__ void __launch_bounds__(256) finalize_dh_kernel(const float* __restrict__ acc, int64_t D,
                                                          const int32_t* __restrict__ idx, const Header* hdr,
                                                          uint16_t* __restrict__ dhidden) {
  const int r = blockIdx.x;
  if (r >= hdr->n_valid) return;
  const float c = hdr->c;
  const float4* src = reinterpret_cast<const float4*>(acc + static_cast<int64_t>(r) * D);
  uint2* dst = reinterpret_cast<uint2*>(dhidden + static_cast<int64_t>(idx[r]) * D);
  for (int v = threadIdx.x; v < D / 4; v += blockDim.x) {
    const float4 a = src[v];
    dst[v] = make_uint2(pack_bf16x2(c * a.x, c * a.y), pack_bf16x2(c * a.z, c * a.w));
  }
}

// ============================================================ fused fwd+bwd (row chunks)
// S3 for one row chunk: partials [n_tiles][ld] of chunk rows m < M (M =
// clamp(N_v - row_off, 0, cap)) -> lse, token loss (scattered to the token
// rows) and the compact-row copies lse_c / ltok used by the next kernels.
__global__ void __launch_bounds__(256) combine_rows_kernel(const float* __restrict__ pm, const float* __restrict__ ps,
                                                           int n_tiles, int64_t ld, int row_off, int cap,
                                                           const float* __restrict__ zt,
                                                           const int32_t* __restrict__ idx, const Header* hdr,
                                                           float* __restrict__ lse_out, float* __restrict__ tok_out,
                                                           float* __restrict__ lse_c, float* __restrict__ ltok,
                                                           const float* __restrict__ q_ref = nullptr,
                                                           int32_t* __restrict__ q_flag = nullptr) {
  const int m = blockIdx.x * kRowsPerCta + (threadIdx.x >> 5);  // one warp per row
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  if (m >= M) return;
  float Mx, S;
  row_merge_warp(pm, ps, n_tiles, ld, m, Mx, S);
  if (threadIdx.x & 31) return;
  const int r = row_off + m;
  const float lse = Mx + logf(S);
  const float l = lse - zt[r];
  const int i = idx[r];
  if (lse_out) lse_out[i] = lse;
  if (tok_out) tok_out[i] = l;
  lse_c[r] = lse;
  if (ltok) ltok[r] = l;
  if (q_ref && lse - q_ref[r] > kScaledQMax) *q_flag = 1;  // (p_y - 1) / beta would leave the range
}

// Vocab-parallel S3 of one row chunk (fused path):
//   mode 1: local partials -> m_loc, m_glob (= m_loc, MAX-reduced next), s, z_t copy
//   mode 2: after MAX all-reduce: s *= exp(m_loc - M)   (SUM-reduced next, with z_t)
//   mode 3: after SUM all-reduce: lse = M + ln s, l = lse - z_t -> outputs, lse_c, ltok
// Chunk buffers are indexed by chunk row m; [s | z_t] are adjacent (one all-reduce).
__global__ void __launch_bounds__(256) combine_chunk_vp_kernel(int mode, const float* __restrict__ pm,
                                                               const float* __restrict__ ps, int n_tiles, int64_t ld,
                                                               int row_off, int cap, const float* __restrict__ zt,
                                                               float* __restrict__ m_loc, float* __restrict__ m_glob,
                                                               float* __restrict__ sz, const int32_t* __restrict__ idx,
                                                               const Header* hdr, float* __restrict__ lse_out,
                                                               float* __restrict__ tok_out, float* __restrict__ lse_c,
                                                               float* __restrict__ ltok,
                                                               const float* __restrict__ q_ref = nullptr,
                                                               int32_t* __restrict__ q_flag = nullptr) {
  // one warp per chunk row (8 rows per CTA); lane 0 owns the row
  const int m = blockIdx.x * kRowsPerCta + (threadIdx.x >> 5);
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  if (m >= M) return;
  const int r = row_off + m;
  if (mode == 1) {
    float Mx, S;
    row_merge_warp(pm, ps, n_tiles, ld, m, Mx, S);
    if (threadIdx.x & 31) return;
    m_loc[m] = Mx;
    m_glob[m] = Mx;
    sz[m] = S;
    sz[cap + m] = zt[r];
    return;
  }
  if (threadIdx.x & 31) return;
  if (mode == 2) {
    sz[m] *= expf(m_loc[m] - m_glob[m]);
    return;
  }
  const float lse = m_glob[m] + logf(sz[m]);
  const float l = lse - sz[cap + m];
  const int i = idx[r];
  if (lse_out) lse_out[i] = lse;
  if (tok_out) tok_out[i] = l;
  lse_c[r] = lse;
  if (ltok) ltok[r] = l;
  if (q_ref && lse - q_ref[r] > kScaledQMax) *q_flag = 1;
}

// S4 of the fused CE path, in place: q = exp(z - m_t) (bf16, stored by the
// forward epilogue relative to the max m_t of its 256-column tile t) ->
// G = s_i (q exp(m_t - lse_i) - [j == y_i]) in bf16.  The target column is
// formed from the fp32 target logit instead, s_i (exp(z_y - lse_i) - 1), so
// the cancellation near p = 1 keeps its fp32 accuracy.  Rows in
// [M, ceil64(M)) and columns >= n_cols become zero.  One CTA per row.
__global__ void __launch_bounds__(256) fixup_q_kernel(uint16_t* __restrict__ Q, int64_t ldq, int n_cols, int row_off,
                                                      int cap, const int32_t* __restrict__ yc, int32_t label_off,
                                                      const float* __restrict__ lse_c,
                                                      const float* __restrict__ row_scale, const Header* hdr,
                                                      const float* __restrict__ pm, int64_t ld_pm,
                                                      const float* __restrict__ zt,
                                                      const int32_t* __restrict__ gate = nullptr) {
  if (gate && *gate == 0) return;  // scaled-q mode without fallback: nothing to fix up
  const int m = blockIdx.x;
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  if (m >= ((M + 63) & ~63)) return;
  uint4* qrow = reinterpret_cast<uint4*>(Q + static_cast<int64_t>(m) * ldq);
  const int nvec = static_cast<int>(ldq / 8);
  if (m >= M) {
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) qrow[v] = make_uint4(0, 0, 0, 0);
    return;
  }
  const int r = row_off + m;
  const float lse = lse_c[r];
  const int yl = yc[r] - label_off;
  const float sc = hdr->c * (row_scale ? row_scale[r] : 1.f);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    const int c0 = 8 * v;
    const float a = sc * ex2_approx((pm[static_cast<int64_t>(c0 / BN) * ld_pm + m] - lse) * kLog2e);
    const uint4 in = qrow[v];
    const uint32_t wi[4] = {in.x, in.y, in.z, in.w};
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 e = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wi[j]));
      const int c = c0 + 2 * j;
      const float g0 = c < n_cols ? a * e.x : 0.f;
      const float g1 = c + 1 < n_cols ? a * e.y : 0.f;
      w[j] = pack_bf16x2(g0, g1);
    }
    if (yl >= c0 && yl < c0 + 8 && yl < n_cols) {
      const float gt = sc * (ex2_approx((zt[r] - lse) * kLog2e) - 1.f);
      const int j = (yl - c0) >> 1;
      __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&w[j]);
      if ((yl - c0) & 1)
        h.y = __float2bfloat16_rn(gt);
      else
        h.x = __float2bfloat16_rn(gt);
      w[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    qrow[v] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// NEXT-4 linear KD (forward KL, reading R23) for one row chunk, from the kept
// fp32 student / teacher logits: G = s_i (p_S - p_T) in bf16 and
// l_i = lse_S - sum_j p_T z_S (fixed-order block reduction).  One CTA per row.
__global__ void __launch_bounds__(256) kd_fixup_kernel(const float* __restrict__ Zs, const float* __restrict__ Zt,
                                                       int64_t ldz, int n_cols, int row_off, int cap,
                                                       const float* __restrict__ lse_s, const float* __restrict__ lse_t,
                                                       const float* __restrict__ row_scale, const Header* hdr,
                                                       uint16_t* __restrict__ G, float* __restrict__ ltok,
                                                       float* __restrict__ tok_out, const int32_t* __restrict__ idx,
                                                       float* __restrict__ partial = nullptr) {
  // partial != null (vocab-parallel): write this shard's sum_j p_T z_S to
  // partial[m] instead of the loss (summed over ranks, then kd_loss_rows_kernel)
  __shared__ float red[256];
  const int m = blockIdx.x;
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  if (m >= ((M + 63) & ~63)) return;
  uint4* grow = reinterpret_cast<uint4*>(G + static_cast<int64_t>(m) * ldz);
  const int nvec = static_cast<int>(ldz / 8);
  if (m >= M) {
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) grow[v] = make_uint4(0, 0, 0, 0);
    return;
  }
  const int r = row_off + m;
  const float lsl = lse_s[r] * kLog2e, ltl = lse_t[r] * kLog2e;
  const float sc = hdr->c * (row_scale ? row_scale[r] : 1.f);
  const float4* zs = reinterpret_cast<const float4*>(Zs + static_cast<int64_t>(m) * ldz);
  const float4* zt = reinterpret_cast<const float4*>(Zt + static_cast<int64_t>(m) * ldz);
  float acc = 0.f;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    const float4 a0 = zs[2 * v], a1 = zs[2 * v + 1], b0 = zt[2 * v], b1 = zt[2 * v + 1];
    const float xs[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float xt[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      float g[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int col = 8 * v + j + u;
        if (col < n_cols) {
          const float ps = ex2_approx(fmaf(xs[j + u], kLog2e, -lsl));
          const float pt = ex2_approx(fmaf(xt[j + u], kLog2e, -ltl));
          acc = fmaf(pt, xs[j + u], acc);
          g[u] = sc * (ps - pt);
        } else {
          g[u] = 0.f;
        }
      }
      w[j / 2] = pack_bf16x2(g[0], g[1]);
    }
    grow[v] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (partial) {
      partial[m] = red[0];
      return;
    }
    const float l = lse_s[r] - red[0];
    ltok[r] = l;
    if (tok_out) tok_out[idx[r]] = l;
  }
}

// Vocab-parallel KD loss of the chunk rows: l_i = lse_S - (all-reduced) E_{p_T}[z_S].
__global__ void __launch_bounds__(256) kd_loss_rows_kernel(const float* __restrict__ e_sum,
                                                           const float* __restrict__ lse_s, int row_off, int cap,
                                                           const Header* hdr, float* __restrict__ ltok,
                                                           float* __restrict__ tok_out,
                                                           const int32_t* __restrict__ idx) {
  const int m = blockIdx.x * 256 + threadIdx.x;
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  if (m >= M) return;
  const int r = row_off + m;
  const float l = lse_s[r] - e_sum[m];
  ltok[r] = l;
  if (tok_out) tok_out[idx[r]] = l;
}

// Split-K dH of a row chunk: dhidden[idx[row_off + m]] = bf16(sum_s part[s][m])
// (c already folded into G), fixed split order.  One CTA per row.
// With out_f32 != null (vocab-parallel) the fp32 sum goes to out_f32[m] instead
// (all-reduced across ranks, then cast/scattered by a second ksplit = 1 call).
__global__ void __launch_bounds__(256) reduce_dh_kernel(const float* __restrict__ part, int ksplit,
                                                        int64_t part_stride, int64_t D, int row_off, int cap,
                                                        const int32_t* __restrict__ idx, const Header* hdr,
                                                        uint16_t* __restrict__ dhidden,
                                                        float* __restrict__ out_f32 = nullptr,
                                                        const float* __restrict__ row_coef = nullptr) {
  const int m = blockIdx.x;
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  if (m >= M) return;
  if (out_f32) {
    float4* o = reinterpret_cast<float4*>(out_f32 + static_cast<int64_t>(m) * D);
    for (int v = threadIdx.x; v < D / 4; v += blockDim.x) {
      float4 a = reinterpret_cast<const float4*>(part + static_cast<int64_t>(m) * D)[v];
      for (int s = 1; s < ksplit; ++s) {
        const float4 b = reinterpret_cast<const float4*>(part + s * part_stride + static_cast<int64_t>(m) * D)[v];
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
      }
      o[v] = a;
    }
    return;
  }
  uint2* dst = reinterpret_cast<uint2*>(dhidden + static_cast<int64_t>(idx[row_off + m]) * D);
  const float k = row_coef ? row_coef[m] : 1.f;
  for (int v = threadIdx.x; v < D / 4; v += blockDim.x) {
    float4 a = reinterpret_cast<const float4*>(part + static_cast<int64_t>(m) * D)[v];
    for (int s = 1; s < ksplit; ++s) {
      const float4 b = reinterpret_cast<const float4*>(part + s * part_stride + static_cast<int64_t>(m) * D)[v];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    dst[v] = make_uint2(pack_bf16x2(k * a.x, k * a.y), pack_bf16x2(k * a.z, k * a.w));
  }
}

// ============================================================ fused path, scaled-q mode (R25)
// The per-row reference of the stored probabilities: ref_i = h_i . w_{y_i} in
// fp32 (the target logit up to summation order; any value within kScaledQMax
// of the row's logits would do).  One warp per compact row; rows >= N_v get 0.
// rowmap != null: row r of the compacted rows is row rowmap[r] of hc (= the
// caller's hidden: the fused path keeps only a chunk-sized H_c).
__global__ void __launch_bounds__(256) target_dot_kernel(const uint16_t* __restrict__ hc,
                                                         const int32_t* __restrict__ rowmap,
                                                         const uint16_t* __restrict__ W, int64_t D,
                                                         const int32_t* __restrict__ yc, int32_t label_off,
                                                         int32_t n_cols, const Header* hdr, int rows,
                                                         float* __restrict__ q_ref) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int col = r < hdr->n_valid ? yc[r] - label_off : -1;
  if (col < 0 || col >= n_cols) {
    if (lane == 0) q_ref[r] = 0.f;
    return;
  }
  const uint4* a = reinterpret_cast<const uint4*>(hc + static_cast<int64_t>(rowmap ? rowmap[r] : r) * D);
  const uint4* b = reinterpret_cast<const uint4*>(W + static_cast<int64_t>(col) * D);
  float acc = 0.f;
  for (int v = lane; v < D / 8; v += 32) {
    const uint4 x = a[v], w = b[v];
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 xf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[j]));
      const float2 wf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ws[j]));
      acc = fmaf(xf.x, wf.x, acc);
      acc = fmaf(xf.y, wf.y, acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) q_ref[r] = acc;
}

// Scaled-q mode, after the chunk's lse: per chunk row i (one CTA), with
// s_i = c (or c g_i) and beta_i = exp(ref_i - lse_i):
//   coef_i = s_i beta_i                 (dH rows: coef_i (q W)_i)
//   Hs_i   = bf16(s_i beta_i h_i)        (dW = q^T Hs)
//   q[i, y_i] = bf16((p_y - 1) / beta_i), p_y = exp(z_y - lse_i) from the fp32
//   target logit, so G = s beta q holds at the target column too (R25).
// If the chunk's flag is set (some row out of range) the chunk falls back to
// the tile-max form: coef = 1, Hs = h, and the redo forward + fix-up produce G.
// Rows in [M, Nc) get zero coefficients and zero Hs rows.  Block 0 also sets
// the row extent of the conditional redo GEMM (N_v if flagged, else 0).
__global__ void __launch_bounds__(256) scaled_prep_kernel(uint16_t* __restrict__ Q, int64_t ldq, int row_off,
                                                          int cap, const uint16_t* __restrict__ hc,
                                                          const int32_t* __restrict__ rowmap, int64_t D,
                                                          const int32_t* __restrict__ yc, int32_t label_off,
                                                          int32_t n_cols, const float* __restrict__ lse_c,
                                                          const float* __restrict__ zt,
                                                          const float* __restrict__ q_ref,
                                                          const float* __restrict__ row_scale, const Header* hdr,
                                                          const int32_t* __restrict__ q_flag,
                                                          int32_t* __restrict__ redo_rows, float* __restrict__ coef,
                                                          uint16_t* __restrict__ Hs) {
  const int m = blockIdx.x;
  const int M = min(max(hdr->n_valid - row_off, 0), cap);
  const bool fallback = *q_flag != 0;
  if (m == 0 && threadIdx.x == 0) *redo_rows = fallback ? hdr->n_valid : 0;
  uint4* hs = reinterpret_cast<uint4*>(Hs + static_cast<int64_t>(m) * D);
  if (m >= M) {
    if (threadIdx.x == 0) coef[m] = 0.f;
    for (int v = threadIdx.x; v < D / 8; v += blockDim.x) hs[v] = make_uint4(0, 0, 0, 0);
    return;
  }
  const int r = row_off + m;
  const uint4* h = reinterpret_cast<const uint4*>(hc + static_cast<int64_t>(rowmap ? rowmap[r] : r) * D);
  if (fallback) {
    if (threadIdx.x == 0) coef[m] = 1.f;
    for (int v = threadIdx.x; v < D / 8; v += blockDim.x) hs[v] = h[v];
    return;
  }
  const float lse = lse_c[r];
  const float beta = ex2_approx((q_ref[r] - lse) * kLog2e);
  const float k = hdr->c * (row_scale ? row_scale[r] : 1.f) * beta;
  if (threadIdx.x == 0) {
    coef[m] = k;
    const int col = yc[r] - label_off;
    if (col >= 0 && col < n_cols) {
      const float py = ex2_approx((zt[r] - lse) * kLog2e);
      __nv_bfloat16 g = __float2bfloat16_rn((py - 1.f) / beta);
      Q[static_cast<int64_t>(m) * ldq + col] = *reinterpret_cast<uint16_t*>(&g);
    }
  }
  for (int v = threadIdx.x; v < D / 8; v += blockDim.x) {
    const uint4 x = h[v];
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[j]));
      o[j] = pack_bf16x2(k * f.x, k * f.y);
    }
    hs[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Final S3 loss of the fused path: fixed-order sum of ltok[0, N_v) in fp64.
__global__ void __launch_bounds__(1024) loss_reduce_kernel(const float* __restrict__ ltok, const Header* hdr,
                                                           float* __restrict__ loss, int32_t* __restrict__ n_valid_out,
                                                           int reduction) {
  __shared__ double red[1024];
  const int nv = hdr->n_valid;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nv; i += 1024) acc += ltok[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double L = red[0];
    const int nd = hdr->mean_div;
    if (reduction == 0) L = nd > 0 ? L / nd : 0.0;
    if (hdr->status & kStatusBadLabel) L = __longlong_as_double(0x7ff8000000000000ULL);
    *loss = static_cast<float>(L);
    if (n_valid_out) *n_valid_out = nd;
  }
}

}  // namespace lce
