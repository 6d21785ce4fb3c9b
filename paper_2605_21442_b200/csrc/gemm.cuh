// gemm.cuh -- persistent, warp-specialised tcgen05 GEMM mainloop for sm_100a.
//
//   D[m, n] = sum_k A[m, k] * B[n, k]      (bf16 x bf16 -> fp32 in TMEM)
//
// Every GEMM on the LCE hot path runs through
// this one mainloop; they differ only in operand major-ness (A_MN / B_MN) and in
// the epilogue policy `Epi`, which consumes the fp32 accumulator straight from
// TMEM, so no GEMM result (in particular no logit tile) is ever written to HBM
// unless the epilogue chooses to.
//
// CTA layout (256 threads, 1 CTA per SM, persistent over output tiles):
//   warp 0      TMA producer (one elected lane): A/B k-blocks -> smem ring
//   warp 1      MMA issuer (one lane): tcgen05.mma 128x256x16, fp32 accum in TMEM
//   warp 2      TMEM allocator (512 columns = 2 accumulator buffers of 256)
//   warp 3      (CTA-pair kernels, K-lockstep on) progress monitor, see lockstep_monitor
//   warps 4..7  epilogue: tcgen05.ld the accumulator (thread = one tile row =
//               one TMEM lane) while the MMA warp fills the other buffer.
// Pipelines: smem full/empty mbarriers (TMA <-> MMA, kStages deep) and TMEM
// full/empty mbarriers (MMA <-> epilogue, 2 deep).
// Three variants share this structure: gemm_kernel (one CTA, 128x256 tiles),
// gemm_pair_kernel (CTA pair, cta_group::2, 256x256 tiles, the default) and
// gemm_wide_kernel (CTA pair, 512x256 tiles, one accumulator per CTA half).
// Under the profiler CTA 0 records its clock64 / %globaltimer span (probe).
#pragma once

#include "sm100.cuh"

namespace lce {

constexpr int BM = 128;     // tile rows   (TMEM lanes)
constexpr int BN = 256;     // tile cols   (TMEM columns per accumulator buffer)
constexpr int BK = 64;      // k-block: 64 bf16 = one 128-byte swizzle row
constexpr int UK = 16;      // K of one tcgen05.mma.kind::f16
constexpr int kStages = 4;  // smem ring depth (4 x 48 KB)
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;
constexpr int kGroupM = 16;  // raster: 16 m-blocks share each n-block sweep (L2 reuse)

constexpr int kAStageBytes = BM * BK * 2;  // 16 KB
constexpr int kBStageBytes = BN * BK * 2;  // 32 KB
// Per epilogue warp: kEpiBufs rotating 32 x 128-byte staging tiles for TMA
// stores (4 warps), so a tile can be refilled while the previous store still
// reads its neighbour.
constexpr int kEpiWarpSmem = 4096;
constexpr int kEpiBufs = 2;
constexpr int kEpiSmemBytes = 4 * kEpiBufs * kEpiWarpSmem;
// [A stages][B stages][barriers: 1 KB][epilogue staging] after 1 KB alignment
constexpr int kSmemBytes = kStages * (kAStageBytes + kBStageBytes) + 1024 /*align slack*/ + 1024 /*barriers*/ +
                           kEpiSmemBytes;

// Problem extents.  M and K may live on the device (they depend on the number
// of non-ignored tokens, which the host never reads back).
struct GemmDims {
  const int32_t* m_dev;
  int32_t m_static;
  const int32_t* k_dev;
  int32_t k_static;
  int32_t n;
  // device extents are clamp(*dev - off, 0, cap) (cap 0 = no upper clamp): a
  // row chunk [off, off + cap) of the N_v compacted tokens
  int32_t m_off, m_cap, k_off, k_cap;
  // split-K: each output tile is computed as `ksplit` (<= 1: one) independent
  // k-ranges; the epilogue sees the split index and must reduce them itself
  int32_t ksplit;
  // raster: output tiles are walked in groups of `group_m` M-blocks, N-blocks
  // inner (0 = kGroupM); the concurrently resident tiles then share A and B
  // tiles through L2
  int32_t group_m;
  // L2 eviction priority of the A / B operand loads (0 normal, 1 evict_first,
  // 2 evict_last): operands reused by later tiles of the raster stay in L2
  int32_t a_hint, b_hint;
  // L2 eviction priority of the epilogue's TMA stores (same encoding)
  int32_t st_hint;
  // profiler (null = off): CTA 0 records {globaltimer, clock64} at start and
  // end, i.e. the SM clock the kernel actually ran at inside the step
  unsigned long long* probe;
  // K-lockstep (null = off): the leader CTA of every cluster publishes how
  // many k-block steps its producer has issued ({lock_gen, steps} in
  // lock_prog[cluster]) and its producer waits while it is more than lock_d
  // steps ahead of the slowest cluster, so clusters that share an operand
  // k-slab read it within a short window, while it is in L2.
  unsigned long long* lock_prog;
  uint32_t lock_gen;
  int32_t lock_d;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The K-lockstep is split between two warps of the leader CTA so that no
// global memory latency sits on the TMA producer's path:
//   * the producer (lockstep_gate) keeps its issued k-block count in shared
//     memory and, before each step, waits while it is more than lock_d steps
//     ahead of the slowest cluster as last seen by the monitor;
//   * the monitor (warp 3, otherwise idle; lockstep_monitor) publishes this
//     cluster's count to lock_prog[cluster] and polls every cluster's count
//     (one load per lane) about every 2 us until the producer is done (a
//     256-ns poll made the five progress lines an L2 hot spot that delayed
//     the operand loads hashed to the same slices: pair forward -26%).
// A cluster that is not running makes the gate time out, after which that
// producer stops waiting for the rest of the launch: the lockstep can delay a
// producer, never block it.  The peer CTA's producer is paced by the shared
// stage ring and needs no gate.
constexpr unsigned long long kLockTimeoutNs = 40000;
struct LockSmem {
  uint32_t steps;    // k-block steps the leader's producer has issued
  uint32_t slowest;  // min over clusters of their published steps (monitor)
  uint32_t done;     // producer finished
};
// The producer and the monitor exchange these words with shared-memory
// atomics (single writer per word, values only grow): no barrier between
// them, and no plain racing accesses.
__device__ __forceinline__ uint32_t lock_ld(uint32_t* p) { return atomicOr(p, 0u); }
__device__ __forceinline__ void lock_st(uint32_t* p, uint32_t v) { atomicExch(p, v); }

__device__ __forceinline__ void lockstep_gate(const GemmDims& d, LockSmem* ls, uint32_t steps, bool& on) {
  lock_st(&ls->steps, steps);
  if (!on || steps <= lock_ld(&ls->slowest) + static_cast<uint32_t>(d.lock_d)) return;
  const unsigned long long t0 = globaltimer_ns();
  while (steps > lock_ld(&ls->slowest) + static_cast<uint32_t>(d.lock_d)) {
    if (globaltimer_ns() - t0 > kLockTimeoutNs) {  // a cluster is not running: stop waiting
      on = false;
      return;
    }
    __nanosleep(64);
  }
}

#ifndef LCE_LOCK_MON
#define LCE_LOCK_MON 1  // A/B: 0 = no monitor loop, 2 = publish only (no polling)
#endif
#ifndef LCE_LOCK_SLEEP
#define LCE_LOCK_SLEEP 2000
#endif
__device__ __forceinline__ void lockstep_monitor(const GemmDims& d, LockSmem* ls, int cluster, int nclusters,
                                                 int lane) {
  const unsigned long long tag = static_cast<unsigned long long>(d.lock_gen) << 32;
  if (LCE_LOCK_MON == 0) return;
  for (;;) {
    uint32_t done = 0, mine = 0;
    if (lane == 0) {
      done = lock_ld(&ls->done);
      mine = done ? 0xffffffffu : lock_ld(&ls->steps);
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(d.lock_prog + cluster), "l"(tag | mine) : "memory");
    }
    if (__shfl_sync(0xffffffffu, done, 0)) return;
    if (LCE_LOCK_MON == 2) {
      __nanosleep(LCE_LOCK_SLEEP);
      continue;
    }
    uint32_t mn = 0xffffffffu;
    for (int c = lane; c < nclusters; c += 32) {
      unsigned long long v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(d.lock_prog + c));
      const uint32_t st = (v >> 32) == d.lock_gen ? static_cast<uint32_t>(v) : 0u;
      mn = st < mn ? st : mn;
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (lane == 0) lock_st(&ls->slowest, mn);
    // wait out the poll period in short naps, leaving as soon as the producer is done
    for (int i = 0; i < LCE_LOCK_SLEEP / 250; ++i) {
      if (__shfl_sync(0xffffffffu, lane == 0 ? lock_ld(&ls->done) : 0u, 0)) break;
      __nanosleep(250);
    }
  }
}

__device__ __forceinline__ void probe_mark(unsigned long long* probe, int at) {
  if (probe && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    probe[at] = t;
    probe[at + 1] = clock64();
  }
}

// Geometry handed to the epilogue for one output tile.
struct TileInfo {
  int m0, n0, n_blk;
  int M, N;
  int row;        // row of this thread inside the tile (== TMEM lane)
  bool zero_acc;  // empty k-range: the accumulator was never written, treat as 0
  int split;      // split-K index of this work item
  uint8_t* smem;  // this warp's nbufs x 4 KB epilogue staging tiles (1 KB aligned)
  uint32_t nst;   // TMA stores this warp has issued so far (selects the next staging tile)
  uint64_t st_policy;  // L2 cache policy for the epilogue's TMA stores
  int nbufs;           // staging tiles of this warp (kEpiBufs; kWideEpiBufs in the wide kernel)
};

// This warp's next staging tile: waits (lane 0) until the store that last read
// it is done reading, i.e. at most kEpiBufs - 1 newer stores may still be
// reading.  Every call must be followed by exactly one committed store group.
__device__ __forceinline__ uint8_t* stage_next(TileInfo& t) {
  if ((t.row & 31) == 0) {
    switch (t.nbufs) {  // the wait depth is an immediate
      case 1: tma_store_wait_read_n<0>(); break;
      case 2: tma_store_wait_read_n<1>(); break;
      case 3: tma_store_wait_read_n<2>(); break;
      case 4: tma_store_wait_read_n<3>(); break;
      case 5: tma_store_wait_read_n<4>(); break;
      default: tma_store_wait_read_n<5>(); break;
    }
  }
  __syncwarp();
  uint8_t* st = t.smem + (t.nst % static_cast<uint32_t>(t.nbufs)) * kEpiWarpSmem;
  ++t.nst;
  return st;
}

// Epilogue policies derive from EpiBase; `prefetch` runs before the epilogue
// waits for the tile's accumulator (i.e. while the MMA is still computing it),
// so read-modify-write epilogues can pull their old output rows into L2 early.
struct EpiBase {
  template <class P>
  static __device__ __forceinline__ void prefetch(const P&, const TileInfo&) {}
  // after the warp's last tile (e.g. drain outstanding TMA stores)
  template <class P>
  static __device__ __forceinline__ void finish(const P&) {}
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<uint64_t>(p)));
}

// One work item of the persistent schedule: output tile (mb, nb) and its k-block range.
struct WorkItem {
  int mb, nb, s, kb0, kb1;
};

__device__ __forceinline__ int extent(const int32_t* p, int32_t v, int32_t off, int32_t cap) {
  int x = p ? *p - off : v;
  x = x < 0 ? 0 : x;
  return (cap > 0 && x > cap) ? cap : x;
}

__device__ __forceinline__ void tile_of(int t, int num_m, int num_n, int GM, int& m_blk, int& n_blk) {
  const int per_group = GM * num_n;
  const int g = t / per_group;
  const int first_m = g * GM;
  const int gsz = min(num_m - first_m, GM);
  const int r = t - g * per_group;
  m_blk = first_m + r % gsz;
  n_blk = r / gsz;
}

// Split index outermost: concurrently resident work items share one k-range,
// so (with an N-fastest raster) each A k-slab is read once for all N tiles.
__device__ __forceinline__ WorkItem work_of(int t, int num_m, int num_n, int S, int num_k, int GM) {
  WorkItem w;
  const int tiles = num_m * num_n;
  w.s = t / tiles;
  const int tile = t - w.s * tiles;
  tile_of(tile, num_m, num_n, GM, w.mb, w.nb);
  w.kb0 = static_cast<int>(static_cast<long long>(num_k) * w.s / S);
  w.kb1 = static_cast<int>(static_cast<long long>(num_k) * (w.s + 1) / S);
  return w;
}

template <bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const GemmDims dims, const __grid_constant__ typename Epi::Params ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kAStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* epi_smem = reinterpret_cast<uint8_t*>(full) + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int M = extent(dims.m_dev, dims.m_static, dims.m_off, dims.m_cap);
  const int K = extent(dims.k_dev, dims.k_static, dims.k_off, dims.k_cap);
  const int N = dims.n;
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (N + BN - 1) / BN;
  const int num_k = (K + BK - 1) / BK;
  const int S = dims.ksplit > 1 ? dims.ksplit : 1;
  const int GM = dims.group_m > 0 ? dims.group_m : kGroupM;
  const int num_tiles = num_m * num_n * S;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  probe_mark(dims.probe, 0);

  if (warp == 0) {
    if (lane == 0 && num_k > 0) {
      // ---------------------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pa = l2_policy(dims.a_hint), pb = l2_policy(dims.b_hint);
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
        const int m0 = w.mb * BM, n0 = w.nb * BN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kAStageBytes + kBStageBytes);
          uint8_t* a = sA + stage * kAStageBytes;
          uint8_t* b = sB + stage * kBStageBytes;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_hint(a, &tmA, &full[stage], k0, m0, pa);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d_hint(a + j * BK * 128, &tmA, &full[stage], m0 + 64 * j, k0, pa);
          }
          if (!B_MN) {
            tma_load_2d_hint(b, &tmB, &full[stage], k0, n0, pb);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d_hint(b + j * BK * 128, &tmB, &full[stage], n0 + 64 * j, k0, pb);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * kAStageBytes);
          const uint32_t b_addr = smem_u32(sB + stage * kBStageBytes);
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = A_MN ? smem_desc_sw128(a_addr + kk * (UK * 128), BK * 128, 1024)
                                     : smem_desc_sw128(a_addr + kk * (UK * 2), 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(b_addr + kk * (UK * 128), BK * 128, 1024)
                                     : smem_desc_sw128(b_addr + kk * (UK * 2), 16, 1024);
            mma_bf16_ss(d, ad, bd, idesc, (kb != w.kb0 || kk != 0) ? 1u : 0u);
          }
          mma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (w.kb1 > w.kb0) {
          mma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        } else {
          mbar_arrive(&tfull[acc]);
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t nst = 0;
    const uint64_t stp = l2_policy(dims.st_hint);
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
      TileInfo ti{w.mb * BM, w.nb * BN, w.nb, M, N, q * 32 + lane, w.kb1 == w.kb0, w.s,
                  epi_smem + q * kEpiBufs * kEpiWarpSmem, nst, stp, kEpiBufs};
      Epi::prefetch(ep, ti);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      Epi::apply(ep, taddr, ti);
      nst = ti.nst;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    Epi::finish(ep);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  probe_mark(dims.probe, 2);
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

// =====================================================================
// CTA-pair variant: tcgen05.mma.cta_group::2, tile 256 x 256 per pair.
//
// A cluster of 2 CTAs on one TPC computes a 256-row x 256-col tile.  CTA r
// stages rows [128r, 128r+128) of the A tile and columns [128r, 128r+128) of
// the B tile (TMA .cta_group::2; both CTAs' bytes complete on the leader's
// barrier); the leader's single MMA thread issues 256x256x16 MMAs that read
// A and B from both CTAs' shared memory and write rows [128r, +128) of the
// accumulator into CTA r's TMEM.  Per SM this halves the B operand's smem and
// L2 traffic relative to the single-CTA kernel for the same MMA rate.
// Epilogues are unchanged: each CTA drains its own 128 TMEM lanes.
// =====================================================================
constexpr int kPairBM = 256;  // rows per pair tile
#ifndef LCE_PAIR_STAGES
#define LCE_PAIR_STAGES 6
#endif
constexpr int kPairStages = LCE_PAIR_STAGES;
constexpr int kPairStageBytes = 128 * BK * 2 * 2;  // A half + B half = 32 KB
constexpr int kPairSmemBytes = kPairStages * kPairStageBytes + 1024 + 1024 + kEpiSmemBytes;

template <bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmDims dims, const __grid_constant__ typename Epi::Params ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kHalf = 128 * BK * 2;  // 16 KB
  uint8_t* sA = smem;
  uint8_t* sB = smem + kPairStages * kHalf;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kPairStages * kHalf);
  uint64_t* empty = full + kPairStages;
  uint64_t* tfull = empty + kPairStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  LockSmem* lsm = reinterpret_cast<LockSmem*>(tmem_slot + 4);
  uint8_t* epi_smem = reinterpret_cast<uint8_t*>(full) + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  const int M = extent(dims.m_dev, dims.m_static, dims.m_off, dims.m_cap);
  const int K = extent(dims.k_dev, dims.k_static, dims.k_off, dims.k_cap);
  const int N = dims.n;
  const int num_m = (M + kPairBM - 1) / kPairBM;
  const int num_n = (N + BN - 1) / BN;
  const int num_k = (K + BK - 1) / BK;
  const int S = dims.ksplit > 1 ? dims.ksplit : 1;
  const int GM = dims.group_m > 0 ? dims.group_m : kGroupM;
  const int num_tiles = num_m * num_n * S;
  // K-lockstep: gate in the leader's producer, monitor in its warp 3 (nothing to pace in an empty launch)
  const bool lock = dims.lock_prog != nullptr && leader && num_k > 0 && num_tiles > 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(&full[s], 1);   // leader: its own arrive.expect_tx; bytes from both CTAs
      mbar_init(&empty[s], 1);  // one multicast commit from the leader's MMA thread
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);   // multicast commit
      mbar_init(&tempty[s], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    lsm->steps = 0;
    lsm->slowest = 0;
    lsm->done = 0;
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, kTmemCols);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  probe_mark(dims.probe, 0);

  if (warp == 0) {
    if (lane == 0 && num_k > 0) {
      // ---------------------------------------------------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pa = l2_policy(dims.a_hint), pb = l2_policy(dims.b_hint);
      uint32_t steps = 0;
      bool lock_on = lock;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
        const int ma = w.mb * kPairBM + 128 * rank;  // this CTA's A rows
        const int nbh = w.nb * BN + 128 * rank;      // this CTA's B rows (N half)
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          if (lock) lockstep_gate(dims, lsm, steps++, lock_on);
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kPairStageBytes);
          uint8_t* a = sA + stage * kHalf;
          uint8_t* b = sB + stage * kHalf;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_pair(a, &tmA, &full[stage], k0, ma, pa);
          } else {
            tma_load_2d_pair(a, &tmA, &full[stage], ma, k0, pa);
            tma_load_2d_pair(a + BK * 128, &tmA, &full[stage], ma + 64, k0, pa);
          }
          if (!B_MN) {
            tma_load_2d_pair(b, &tmB, &full[stage], k0, nbh, pb);
          } else {
            tma_load_2d_pair(b, &tmB, &full[stage], nbh, k0, pb);
            tma_load_2d_pair(b + BK * 128, &tmB, &full[stage], nbh + 64, k0, pb);
          }
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (lock) lock_st(&lsm->done, 1u);
    }
  } else if (warp == 3) {
    if (lock) lockstep_monitor(dims, lsm, cluster, nclusters, lane);
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------------------------------------------------- MMA issuer (leader only)
      constexpr uint32_t idesc = idesc_bf16_f32(kPairBM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
        mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * kHalf);
          const uint32_t b_addr = smem_u32(sB + stage * kHalf);
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = A_MN ? smem_desc_sw128(a_addr + kk * (UK * 128), BK * 128, 1024)
                                     : smem_desc_sw128(a_addr + kk * (UK * 2), 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(b_addr + kk * (UK * 128), BK * 128, 1024)
                                     : smem_desc_sw128(b_addr + kk * (UK * 2), 16, 1024);
            mma_bf16_ss_pair(d, ad, bd, idesc, (kb != w.kb0 || kk != 0) ? 1u : 0u);
          }
          mma_commit_pair(&empty[stage], 0x3);  // frees this stage in both CTAs
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (w.kb1 > w.kb0) {
          mma_commit_pair(&tfull[acc], 0x3);
        } else {
          mbar_arrive_cluster(&tfull[acc], 0);
          mbar_arrive_cluster(&tfull[acc], 1);
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t nst = 0;
    const uint64_t stp = l2_policy(dims.st_hint);
    for (int t = cluster; t < num_tiles; t += nclusters) {
      const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
      TileInfo ti{w.mb * kPairBM + 128 * static_cast<int>(rank), w.nb * BN, w.nb, M, N, q * 32 + lane,
                  w.kb1 == w.kb0, w.s, epi_smem + q * kEpiBufs * kEpiWarpSmem, nst, stp, kEpiBufs};
      Epi::prefetch(ep, ti);
      mbar_wait_cluster(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      Epi::apply(ep, taddr, ti);
      nst = ti.nst;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    Epi::finish(ep);
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  probe_mark(dims.probe, 2);
  if (warp == 2) tmem_dealloc_pair(tmem_base, kTmemCols);
}

// =====================================================================
// Wide CTA-pair variant: 512 x 256 per pair (each CTA stages 256 rows of A and
// 128 columns of B per k-block; two cta_group::2 256x256x16 MMAs per k16 step,
// one per accumulator half, share the B operand).  25% fewer operand bytes
// from L2 per flop than the 256 x 256 pair tile, which matters because these
// kernels are power-capped: fewer bytes moved per MMA, higher SM clock.
//   CTA r, accumulator half h holds pair-tile rows [256 r + 128 h, +128).
// The two 128-lane x 256-column halves fill the 512 TMEM columns, so there is
// no second buffer: half 0 gets its own full / empty barriers so the epilogue
// drains it while the MMA finishes half 1's last k-block, and the next tile's
// MMAs start on half 0 as soon as it is drained (up to kWideStages k-blocks
// ahead) and catch up on half 1 when that is drained.  (A design in which half
// 1 trails half 0 by a few k-blocks throughout, to overlap each half's drain
// with the other's MMAs, ran at 65-83% tensor utilisation: the trailing
// k-blocks hold ring stages the TMA needs for prefetch.)
// =====================================================================
constexpr int kWideBM = 512;  // rows per wide pair tile
#ifndef LCE_WIDE_STAGES
#define LCE_WIDE_STAGES 4
#endif
#ifndef LCE_WIDE_EPI_BUFS
#define LCE_WIDE_EPI_BUFS 2
#endif
constexpr int kWideStages = LCE_WIDE_STAGES;
// staging tiles per epilogue warp in the wide kernel: its unbuffered
// accumulator is drained at every tile end, as fast as the TMA stores in
// flight allow
constexpr int kWideEpiBufs = LCE_WIDE_EPI_BUFS;
constexpr int kWideAStage = 256 * BK * 2;  // 32 KB
constexpr int kWideBStage = 128 * BK * 2;  // 16 KB
constexpr int kWideSmemBytes =
    kWideStages * (kWideAStage + kWideBStage) + 1024 + 1024 + 4 * kWideEpiBufs * kEpiWarpSmem;
static_assert(kWideSmemBytes <= 232448, "wide kernel exceeds 227 KB of shared memory");

template <bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmDims dims, const __grid_constant__ typename Epi::Params ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kWideStages * kWideAStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kWideStages * kWideBStage);
  uint64_t* empty = full + kWideStages;
  uint64_t* tfull = empty + kWideStages;  // [2]: accumulator half computed
  uint64_t* tempty = tfull + 2;           // [2]: accumulator half drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  LockSmem* lsm = reinterpret_cast<LockSmem*>(tmem_slot + 4);
  uint8_t* epi_smem = reinterpret_cast<uint8_t*>(full) + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  const int M = extent(dims.m_dev, dims.m_static, dims.m_off, dims.m_cap);
  const int K = extent(dims.k_dev, dims.k_static, dims.k_off, dims.k_cap);
  const int N = dims.n;
  const int num_m = (M + kWideBM - 1) / kWideBM;
  const int num_n = (N + BN - 1) / BN;
  const int num_k = (K + BK - 1) / BK;
  const int S = dims.ksplit > 1 ? dims.ksplit : 1;
  const int GM = dims.group_m > 0 ? dims.group_m : kGroupM;
  const int num_tiles = num_m * num_n * S;
  // K-lockstep: gate in the leader's producer, monitor in its warp 3 (nothing to pace in an empty launch)
  const bool lock = dims.lock_prog != nullptr && leader && num_k > 0 && num_tiles > 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kWideStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 1);   // multicast commit
      mbar_init(&tempty[h], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    lsm->steps = 0;
    lsm->slowest = 0;
    lsm->done = 0;
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, kTmemCols);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  probe_mark(dims.probe, 0);

  if (warp == 0) {
    if (lane == 0 && num_k > 0) {
      // ---------------------------------------------------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pa = l2_policy(dims.a_hint), pb = l2_policy(dims.b_hint);
      uint32_t steps = 0;
      bool lock_on = lock;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
        const int ma = w.mb * kWideBM + 256 * rank;  // this CTA's 256 A rows
        const int nbh = w.nb * BN + 128 * rank;      // this CTA's B rows (N half)
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          if (lock) lockstep_gate(dims, lsm, steps++, lock_on);
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (kWideAStage + kWideBStage));
          uint8_t* a = sA + stage * kWideAStage;
          uint8_t* b = sB + stage * kWideBStage;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_pair(a, &tmA, &full[stage], k0, ma, pa);
            tma_load_2d_pair(a + 128 * 128, &tmA, &full[stage], k0, ma + 128, pa);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) tma_load_2d_pair(a + j * BK * 128, &tmA, &full[stage], ma + 64 * j, k0, pa);
          }
          if (!B_MN) {
            tma_load_2d_pair(b, &tmB, &full[stage], k0, nbh, pb);
          } else {
            tma_load_2d_pair(b, &tmB, &full[stage], nbh, k0, pb);
            tma_load_2d_pair(b + BK * 128, &tmB, &full[stage], nbh + 64, k0, pb);
          }
          if (++stage == kWideStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (lock) lock_st(&lsm->done, 1u);
    }
  } else if (warp == 3) {
    if (lock) lockstep_monitor(dims, lsm, cluster, nclusters, lane);
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------------------------------------------------- MMA issuer (leader only)
      constexpr uint32_t idesc = idesc_bf16_f32(kPairBM, BN, A_MN, B_MN);
      // MMAs of accumulator half h on the k-block in stage `st`
      auto issue = [&](int st, int h, bool first) {
        const uint32_t a_addr = smem_u32(sA + st * kWideAStage + h * (128 * 128));
        const uint32_t b_addr = smem_u32(sB + st * kWideBStage);
        const uint32_t d = tmem_base + h * BN;
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          const uint64_t ad = A_MN ? smem_desc_sw128(a_addr + kk * (UK * 128), BK * 128, 1024)
                                   : smem_desc_sw128(a_addr + kk * (UK * 2), 16, 1024);
          const uint64_t bd = B_MN ? smem_desc_sw128(b_addr + kk * (UK * 128), BK * 128, 1024)
                                   : smem_desc_sw128(b_addr + kk * (UK * 2), 16, 1024);
          mma_bf16_ss_pair(d, ad, bd, idesc, (first && kk == 0) ? 0u : 1u);
        }
      };
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
        const int nkb = w.kb1 - w.kb0;
        const int pre = nkb < kWideStages ? nkb : kWideStages;
        // half 0 on the first `pre` k-blocks as soon as the epilogue has drained it
        mbar_wait_cluster(&tempty[0], acc_phase ^ 1);
        tc_fence_after();
        int st = stage;
        uint32_t ph = phase;
        for (int j = 0; j < pre; ++j) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          issue(st, 0, j == 0);
          if (++st == kWideStages) {
            st = 0;
            ph ^= 1;
          }
        }
        if (pre == nkb && nkb > 0) mma_commit_pair(&tfull[0], 0x3);
        // half 1 catches up on the same k-blocks (while half 1 is drained, the
        // tensor pipe has half 0's `pre` k-blocks), then both advance together
        mbar_wait_cluster(&tempty[1], acc_phase ^ 1);
        tc_fence_after();
        for (int j = 0; j < nkb; ++j) {
          if (j >= pre) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            issue(stage, 0, false);
            // half 0 is complete: its epilogue may start while half 1 finishes
            if (j == nkb - 1) mma_commit_pair(&tfull[0], 0x3);
          }
          issue(stage, 1, j == 0);
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == kWideStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (nkb > 0) {
          mma_commit_pair(&tfull[1], 0x3);
        } else {  // empty k-range: the epilogue treats both halves as zero
          for (int h = 0; h < 2; ++h) {
            mbar_arrive_cluster(&tfull[h], 0);
            mbar_arrive_cluster(&tfull[h], 1);
          }
        }
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    uint32_t acc_phase = 0;
    uint32_t nst = 0;
    const uint64_t stp = l2_policy(dims.st_hint);
    for (int t = cluster; t < num_tiles; t += nclusters) {
      const WorkItem w = work_of(t, num_m, num_n, S, num_k, GM);
      const int m0 = w.mb * kWideBM + 256 * static_cast<int>(rank);
      TileInfo ti{m0, w.nb * BN, w.nb, M, N, q * 32 + lane, w.kb1 == w.kb0, w.s,
                  epi_smem + q * kWideEpiBufs * kEpiWarpSmem, nst, stp, kWideEpiBufs};
      Epi::prefetch(ep, ti);
      ti.m0 = m0 + 128;
      Epi::prefetch(ep, ti);
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        mbar_wait_cluster(&tfull[h], acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + h * BN + (static_cast<uint32_t>(q * 32) << 16);
        ti.m0 = m0 + 128 * h;
        Epi::apply(ep, taddr, ti);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tempty[h], 0);
      }
      nst = ti.nst;
      acc_phase ^= 1;
    }
    Epi::finish(ep);
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  probe_mark(dims.probe, 2);
  if (warp == 2) tmem_dealloc_pair(tmem_base, kTmemCols);
}

// Loads the 32-column chunk `c` of this thread's accumulator row as floats.
__device__ __forceinline__ void load_chunk(uint32_t taddr, int c, bool zero, float (&x)[32]) {
  uint32_t v[32];
  tmem_ld32(taddr + c * 32, v);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = zero ? 0.f : __uint_as_float(v[j]);
}

}  // namespace lce
