// Box probe: fp64 pipe rate, conversion rates, rcp rate, HBM copy.
// Not part of the hot path; measures the hardware the design depends on.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int OP>
__global__ void pipe_kernel(double* out, float* outf, int iters, long long* clk) {
  double a[8]; float f[8];
  for (int i = 0; i < 8; ++i) { a[i] = 1.0 + 1e-9 * (threadIdx.x + i); f[i] = 1.0f + 1e-6f * (threadIdx.x + i); }
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fma(a[i], 0.999999999, 1e-10);              // DFMA
      if (OP == 1) { a[i] = (double)f[i] + a[i]; f[i] = f[i] * 1.0000001f; }  // F2F.F64.F32 + DADD + FMUL
      if (OP == 2) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a[i])); a[i] = r + 1e-12; }
      if (OP == 3) { f[i] = (float)a[i] + f[i]; a[i] = a[i] * 1.0000000001; }  // F2F.F32.F64 + FADD + DMUL
      if (OP == 4) a[i] = a[i] + 1e-12;                                // DADD
    }
  }
  long long c1 = clock64();
  double s = 0; float sf = 0;
  for (int i = 0; i < 8; ++i) { s += a[i]; sf += f[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  outf[blockIdx.x * blockDim.x + threadIdx.x] = sf;
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s sms %d smem/SM %zu l2 %d MB cc %d.%d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerMultiprocessor, p.l2CacheSize >> 20, p.major, p.minor);
  int sms = p.multiProcessorCount;
  int blocks = sms * 2, threads = 512;
  double* out; float* outf; long long* clk;
  CK(cudaMalloc(&out, blocks * threads * 8)); CK(cudaMalloc(&outf, blocks * threads * 4));
  CK(cudaMalloc(&clk, blocks * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"DFMA", "F2F.F64.F32(+DADD+FMUL)", "MUFU.RCP64H(+DADD)", "F2F.F32.F64(+FADD+DMUL)", "DADD"};
  for (int op = 0; op < 5; ++op) {
    int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      switch (op) {
        case 0: pipe_kernel<0><<<blocks, threads>>>(out, outf, iters, clk); break;
        case 1: pipe_kernel<1><<<blocks, threads>>>(out, outf, iters, clk); break;
        case 2: pipe_kernel<2><<<blocks, threads>>>(out, outf, iters, clk); break;
        case 3: pipe_kernel<3><<<blocks, threads>>>(out, outf, iters, clk); break;
        case 4: pipe_kernel<4><<<blocks, threads>>>(out, outf, iters, clk); break;
      }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; CK(cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost));
    double ops = (double)blocks * threads * iters * 8;
    double ghz = (double)c / (ms * 1e6);  // approx: one block's cycles / wall time (all blocks concurrent)
    printf("%-26s %.3f ms  %.2f Gop/s  %.1f op/clk/SM (block clk %lld, ~%.2f GHz)\n", names[op], ms,
           ops / ms / 1e6, ops / ms / 1e6 / (sms * ghz), c, ghz);
  }
  size_t n = (size_t)1 << 28;  // 256 Mi float4 = 4 GiB
  float4 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 4 GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
