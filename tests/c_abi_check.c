/* Plain-C client of liblce.so (include/lce.h): no Python, no torch.
 *
 * Builds a problem whose answer is a closed form (SURVEY.md 8c pin P1): with
 * W = 0 every logit is 0, so lse_i = ln V exactly for every non-ignored row,
 * the MEAN loss is ln V, dH = 0 and dW_j = (1/N_v) sum_valid h_i / V -
 * (1/N_v) sum_{i: y_i = j} h_i.  Runs the split and fused paths through the
 * C ABI on the current CUDA device and prints PASS/FAIL.
 *
 *   gcc -O2 -I include tests/c_abi_check.c -L paper_2605_21442_b200 -llce \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -lm -o c_abi_check
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "lce.h"

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) {                                              \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      return 2;                                                           \
    }                                                                     \
  } while (0)
#define LK(x)                                                             \
  do {                                                                    \
    lce_status_t s_ = (x);                                                \
    if (s_ != LCE_OK) {                                                   \
      fprintf(stderr, "%s: %s\n", #x, lce_status_string(s_));             \
      return 3;                                                           \
    }                                                                     \
  } while (0)

static uint16_t f2bf(float f) { /* exact for the small dyadic values used here */
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}
static float bf2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main(void) {
  const int64_t N = 300, D = 72, V = 1000;
  uint16_t* h_hidden = malloc(N * D * 2);
  int32_t* h_labels = malloc(N * 4);
  for (int64_t i = 0; i < N * D; ++i) h_hidden[i] = f2bf((float)((i * 37 % 17) - 8) / 8.0f);
  int64_t nv = 0;
  for (int64_t i = 0; i < N; ++i) {
    h_labels[i] = (i % 7 == 3) ? -100 : (int32_t)((i * 131) % V);
    nv += h_labels[i] != -100;
  }
  lce_problem_t p = {N, D, V, 0, V, -100, LCE_MEAN, 0};
  size_t ws_bytes = lce_workspace_bytes(&p);
  size_t fws_bytes = lce_fused_workspace_bytes(&p);
  if (!ws_bytes || !fws_bytes) return 4;
  uint16_t *hidden, *weight, *dhidden;
  int32_t* labels;
  float *loss, *lse, *dweight;
  void* ws;
  CK(cudaMalloc((void**)&hidden, N * D * 2));
  CK(cudaMalloc((void**)&weight, V * D * 2));
  CK(cudaMalloc((void**)&dhidden, N * D * 2));
  CK(cudaMalloc((void**)&labels, N * 4));
  CK(cudaMalloc((void**)&loss, 16));
  CK(cudaMalloc((void**)&lse, N * 4));
  CK(cudaMalloc((void**)&dweight, V * D * 4));
  CK(cudaMalloc(&ws, ws_bytes > fws_bytes ? ws_bytes : fws_bytes));
  CK(cudaMemcpy(hidden, h_hidden, N * D * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(labels, h_labels, N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(weight, 0, V * D * 2));

  /* expected dW (closed form) */
  double* exp_dw = calloc(V * D, sizeof(double));
  for (int64_t i = 0; i < N; ++i) {
    if (h_labels[i] == -100) continue;
    for (int64_t k = 0; k < D; ++k) {
      const double h = bf2f(h_hidden[i * D + k]) / (double)nv;
      for (int64_t j = 0; j < V; ++j) exp_dw[j * D + k] += h / V;
      exp_dw[h_labels[i] * D + k] -= h;
    }
  }
  float* h_dw = malloc(V * D * 4);
  float* h_lse = malloc(N * 4);
  uint16_t* h_dh = malloc(N * D * 2);
  int fail = 0;
  for (int path = 0; path < 2; ++path) {
    float h_loss = -1.f;
    if (path == 0) {
      LK(lce_forward(&p, NULL, hidden, weight, labels, loss, lse, NULL, NULL, ws, ws_bytes, NULL));
      LK(lce_backward(&p, NULL, hidden, weight, labels, lse, NULL, dhidden, dweight, 0, ws, ws_bytes, NULL));
    } else {
      LK(lce_forward_backward(&p, NULL, hidden, weight, labels, NULL, loss, lse, NULL, NULL, dhidden, dweight, 0,
                              ws, fws_bytes, NULL));
    }
    CK(cudaDeviceSynchronize());
    LK(lce_check_device_status(ws, NULL));
    CK(cudaMemcpy(&h_loss, loss, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_lse, lse, N * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_dh, dhidden, N * D * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_dw, dweight, V * D * 4, cudaMemcpyDeviceToHost));
    const double lnV = log((double)V);
    double lse_err = 0, dh_max = 0, num = 0, den = 0;
    for (int64_t i = 0; i < N; ++i) {
      const double want = h_labels[i] == -100 ? 0.0 : lnV;
      lse_err = fmax(lse_err, fabs(h_lse[i] - want));
    }
    for (int64_t i = 0; i < N * D; ++i) dh_max = fmax(dh_max, fabs(bf2f(h_dh[i])));
    for (int64_t i = 0; i < V * D; ++i) {
      num += (h_dw[i] - exp_dw[i]) * (h_dw[i] - exp_dw[i]);
      den += exp_dw[i] * exp_dw[i];
    }
    const double loss_err = fabs(h_loss - lnV) / lnV, dw_err = sqrt(num / den);
    const int ok = loss_err < 1e-6 && lse_err < 1e-5 && dh_max == 0.0 && dw_err < 1e-2;
    printf("%s path: loss %.7f (ln V %.7f) lse err %.2e dH max %.1e dW rel err %.2e -> %s\n",
           path ? "fused" : "split", h_loss, lnV, lse_err, dh_max, dw_err, ok ? "PASS" : "FAIL");
    fail |= !ok;
  }
  printf("abi %d launches %llu\n", lce_abi_version(), (unsigned long long)lce_launch_count());
  return fail;
}
