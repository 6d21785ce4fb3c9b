// Feasibility probe (not part of liblce): TMA tile::gather4 with a 128B-swizzled
// K-major bf16 map.  Loads 8 arbitrary rows (two gather4) into shared memory and
// checks they land in the same swizzled layout as an 8-row tile load would give.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/g4 scripts/probes/gather4_probe.cu -lcuda && /tmp/g4
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap m, int boxh, uint16_t* out, const int* rows) {
  __shared__ alignas(1024) uint8_t sm[2048];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * 4 * 128));
    for (int g = 0; g < 2; ++g) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + g * 512);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]),
          "r"(rows[4 * g + 3]), "r"(b)
          : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(b) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}

int main() {
  const int R = 64, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 256 + c);
  uint16_t *d, *o;
  int* dr;
  cudaMalloc(&d, R * C * 2);
  cudaMalloc(&o, 1024 * 2);
  cudaMalloc(&dr, 8 * 4);
  cudaMemcpy(d, h.data(), R * C * 2, cudaMemcpyHostToDevice);
  int rows[8] = {5, 17, 2, 40, 63, 0, 9, 33};
  cudaMemcpy(dr, rows, 32, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  for (int boxh : {1, 4}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64u, (cuuint32_t)boxh};
    cuuint32_t es[2] = {1u, 1u};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("boxh %d encode -> %d\n", boxh, (int)r);
    if (r) continue;
    cudaMemset(o, 0xff, 2048);
    probe<<<1, 128>>>(m, boxh, o, dr);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  run -> %s\n", cudaGetErrorString(e));
    if (e) return 1;
    std::vector<uint16_t> got(512);
    cudaMemcpy(got.data(), o, 1024, cudaMemcpyDeviceToHost);
    int bad_sw = 0, bad_plain = 0;
    for (int k = 0; k < 8; ++k)
      for (int c = 0; c < 64; ++c) {
        const uint16_t want = (uint16_t)(rows[k] * 256 + c);
        const int unit = c / 8, e8 = c % 8;
        if (got[k * 64 + ((unit ^ (k & 7)) * 8) + e8] != want) ++bad_sw;  // 128B swizzle: unit ^ (row % 8)
        if (got[k * 64 + c] != want) ++bad_plain;
      }
    printf("  mismatches: swizzled-layout %d, plain-layout %d (of 512)\n", bad_sw, bad_plain);
  }
  return 0;
}
