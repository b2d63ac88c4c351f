// Latency probe: cycles per row of the factor recurrence (ldl_step, R-10) on one warp, and the
// dependent latencies of DFMA / DADD / MUFU.RCP64H+Newton that make up its chain.  Dev tool.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_00048_b200/csrc/whit_kernels.cuh"

template <int D, int NW>
__global__ void chain_kernel(double* out, long long* clk, int rows) {
  whit::FState<D> st;
  whit::state_init<D>(st);
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  long long c0 = clock64();
  for (int t = 0; t < rows; ++t) {
    const double w = ((t + lane) % 7 == 0) ? 0.0 : 1.0;
    const double lam = 1e3 + (double)((t * 13 + lane) & 63);
    double A[D], Dt, idt, vt;
    whit::ldl_step<D, NW>(st, w, lam, w * 0.5, A, Dt, idt, vt);
    acc += A[0];
  }
  long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + st.v[0];
  if ((threadIdx.x & 31) == 0) clk[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = c1 - c0;
}

// same chain, w / lambda read as fp32 from shared memory like the factor warp (K = 16 rows per
// chunk); HOIST converts a chunk's inputs to fp64 before the recurrence runs over it.
template <int D, int NW, bool HOIST>
__global__ void chain_smem_kernel(double* out, long long* clk, int rows) {
  __shared__ float sw[4][32 * 16], sl[4][32 * 16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < 16; ++k) {
    sw[warp][k * 32 + lane] = ((k + lane) % 7 == 0) ? 0.f : 1.f;
    sl[warp][k * 32 + lane] = 1e3f + (float)((k * 13 + lane) & 63);
  }
  __syncwarp();
  whit::FState<D> st;
  whit::state_init<D>(st);
  double acc = 0.0;
  long long c0 = clock64();
  for (int t0 = 0; t0 < rows; t0 += 16) {
    if (HOIST) {
      double w[16], l[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) { w[k] = (double)sw[warp][k * 32 + lane]; l[k] = (double)sl[warp][k * 32 + lane]; }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        double A[D], Dt, idt, vt;
        whit::ldl_step<D, NW>(st, w[k], l[k], 0.0, A, Dt, idt, vt);
        acc += A[0];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        double A[D], Dt, idt, vt;
        whit::ldl_step<D, NW>(st, (double)sw[warp][k * 32 + lane], (double)sl[warp][k * 32 + lane], 0.0, A, Dt, idt, vt);
        acc += A[0];
      }
    }
  }
  long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + st.v[0];
  if (lane == 0) clk[blockIdx.x * (blockDim.x / 32) + warp] = c1 - c0;
}

template <int OP>
__global__ void lat_kernel(double* out, long long* clk, int iters) {
  double a = 1.0 + 1e-9 * threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) a = fma(a, 0.999999999, 1e-10);
    if (OP == 1) a = a + 1e-12;
    if (OP == 2) a = whit::rcp64<1>(a) + 1.0;
    if (OP == 3) a = whit::rcp64<0>(a) + 1.0;
  }
  long long c1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) clk[0] = c1 - c0;
}

int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&clk, 1 << 20);
  long long h[4096];
  const int iters = 100000;
  const char* names[] = {"DFMA", "DADD", "rcp64<1>+DADD", "rcp.approx+DADD"};
#define LAT(OP) lat_kernel<OP><<<1, 32>>>(out, clk, iters); cudaMemcpy(h, clk, 8, cudaMemcpyDeviceToHost); \
  printf("dependent %-18s %.1f cycles\n", names[OP], (double)h[0] / iters);
  LAT(0) LAT(1) LAT(2) LAT(3)
  const int rows = 20000;
  for (int warps : {1, 2, 4, 8, 12, 16}) {
    chain_kernel<2, 1><<<148, 32 * warps>>>(out, clk, rows);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, clk, 8 * 148 * warps, cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148 * warps; ++i) s += h[i];
    printf("ldl_step<2,1>: %2d warps/SM: %.1f cycles per row per warp\n", warps, s / (148 * warps) / rows);
  }
  for (int warps : {1, 4}) {
    chain_kernel<2, 2><<<148, 32 * warps>>>(out, clk, rows);
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, 8 * 148 * warps, cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148 * warps; ++i) s += h[i];
    printf("ldl_step<2,2>: %2d warps/SM: %.1f cycles per row per warp\n", warps, s / (148 * warps) / rows);
  }
#define SM(H) for (int warps : {1, 4}) { \
    chain_smem_kernel<2, 1, H><<<148, 32 * warps>>>(out, clk, rows); cudaDeviceSynchronize(); \
    cudaMemcpy(h, clk, 8 * 148 * warps, cudaMemcpyDeviceToHost); \
    double s = 0; for (int i = 0; i < 148 * warps; ++i) s += h[i]; \
    printf("smem ldl_step<2,1> hoist=%d: %2d warps/SM: %.1f cycles per row per warp\n", H, warps, s / (148 * warps) / rows); }
  SM(false) SM(true)
  return 0;
}
