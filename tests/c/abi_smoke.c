/* Pure-C consumer of libwhit (include/libwhit.h): no Python, no torch.
 *   ./abi_smoke host   -- host-only checks (sizes, validation) that need no GPU
 *   ./abi_smoke gpu    -- a full forward + backward on cuda:0 through the C-ABI, checked for
 *                         z == y and grad_y == g on the lambda = 0, w = 1 identity (Omega = I),
 *                         and for finiteness / no failures on a smoothing case. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "libwhit.h"

#define CHECK(c) do { if (!(c)) { fprintf(stderr, "FAIL %s:%d: %s (%s)\n", __FILE__, __LINE__, #c, whit_last_error()); return 1; } } while (0)

static int host_checks(void) {
  whit_ws* ws = NULL;
  CHECK(whit_version() == LIBWHIT_VERSION);
  CHECK(strcmp(whit_status_string(WHIT_ERR_STATE), "WHIT_ERR_STATE") == 0);
  CHECK(whit_ws_bytes(2, 3288, 262144, WHIT_F32, WHIT_LAMBDA_PER_DATE) > 0);
  CHECK(whit_ws_bytes(4, 100, 128, WHIT_F32, WHIT_LAMBDA_PER_DATE) == 0);
  CHECK(whit_ws_create(&ws, 2, 100, 130, WHIT_F32, WHIT_LAMBDA_PER_DATE, (void*)(1 << 20), 1ull << 40, NULL) == WHIT_ERR_ALIGN);
  CHECK(whit_ws_create(&ws, 2, 100, 128, WHIT_F32, WHIT_LAMBDA_PER_DATE, (void*)(1 << 20), 1ull << 40, NULL) == WHIT_OK);
  CHECK(whit_backward((void*)16, ws, NULL, (void*)16, (void*)32) == WHIT_ERR_STATE);
  whit_ws_destroy(ws);
  return 0;
}

static int gpu_run(void) {
  const int d = 2;
  const int64_t T = 365, B = 256;
  const size_t n = (size_t)T * B, nl = (size_t)(T - d) * B;
  float *hy = malloc(n * 4), *hw = malloc(n * 4), *hl = malloc(nl * 4), *hg = malloc(n * 4), *hz = malloc(n * 4),
        *hgy = malloc(n * 4);
  for (size_t i = 0; i < n; ++i) {
    hy[i] = (float)sin(0.01 * (double)i);
    hw[i] = 1.0f;
    hg[i] = (float)cos(0.003 * (double)i);
  }
  for (size_t i = 0; i < nl; ++i) hl[i] = 0.0f;
  float *y, *w, *l, *g, *z, *gy, *gl;
  void* buf;
  size_t wsb = whit_ws_bytes(d, T, B, WHIT_F32, WHIT_LAMBDA_PER_DATE);
  CHECK(cudaMalloc((void**)&y, n * 4) == cudaSuccess);
  cudaMalloc((void**)&w, n * 4); cudaMalloc((void**)&l, nl * 4); cudaMalloc((void**)&g, n * 4);
  cudaMalloc((void**)&z, n * 4); cudaMalloc((void**)&gy, n * 4); cudaMalloc((void**)&gl, nl * 4);
  CHECK(cudaMalloc(&buf, wsb) == cudaSuccess);
  cudaMemcpy(y, hy, n * 4, cudaMemcpyHostToDevice); cudaMemcpy(w, hw, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(l, hl, nl * 4, cudaMemcpyHostToDevice); cudaMemcpy(g, hg, n * 4, cudaMemcpyHostToDevice);
  whit_ws* ws = NULL;
  CHECK(whit_ws_create(&ws, d, T, B, WHIT_F32, WHIT_LAMBDA_PER_DATE, buf, wsb, NULL) == WHIT_OK);
  /* lambda = 0, w = 1: Omega = I, so z = y and grad_y = g exactly */
  CHECK(whit_forward(y, w, l, d, T, B, z, ws) == WHIT_OK);
  CHECK(whit_backward(g, ws, z, gy, gl) == WHIT_OK);
  int64_t nfail = -1;
  CHECK(whit_failures(ws, &nfail, NULL) == WHIT_OK && nfail == 0);
  cudaMemcpy(hz, z, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hgy, gy, n * 4, cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < n; ++i) CHECK(hz[i] == hy[i] && hgy[i] == hg[i]);
  /* smoothing case: lambda = 100 on every date, every 3rd date observed */
  for (size_t i = 0; i < nl; ++i) hl[i] = 100.0f;
  for (size_t i = 0; i < n; ++i) hw[i] = ((i / B) % 3 == 0) ? 1.0f : 0.0f;
  cudaMemcpy(l, hl, nl * 4, cudaMemcpyHostToDevice); cudaMemcpy(w, hw, n * 4, cudaMemcpyHostToDevice);
  CHECK(whit_forward(y, w, l, d, T, B, z, ws) == WHIT_OK);
  CHECK(whit_backward(g, ws, z, gy, gl) == WHIT_OK);
  CHECK(whit_failures(ws, &nfail, NULL) == WHIT_OK && nfail == 0);
  cudaMemcpy(hz, z, n * 4, cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < n; ++i) CHECK(isfinite(hz[i]));
  whit_ws_destroy(ws);
  printf("abi_smoke gpu ok\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_run();
  int r = host_checks();
  if (r == 0) printf("abi_smoke host ok\n");
  return r;
}
