// HBM bandwidth by read/write mix (dev probe): copy (1R:1W), the headline kernels' mix (3R:1W),
// and read-only streams.  float4 grid-stride loops, 4 x 1 GiB buffers, best of 10 (CUDA events).
#include <cstdio>
#include <cuda_runtime.h>

template <int NR, int NW>
__global__ void mix(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                    float4* __restrict__ o, float4* __restrict__ o2, size_t n, float* sink) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = a[i];
    if (NR > 1) { const float4 u = b[i]; v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w; }
    if (NR > 2) { const float4 u = c[i]; v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w; }
    if (NW > 0) o[i] = v;
    if (NW > 1) o2[i] = v;
    if (NW == 0) acc += v.x + v.y + v.z + v.w;
  }
  if (NW == 0 && acc == 12345.f) *sink = acc;
}

template <int NR, int NW>
void run(const char* name, float4** bufs, size_t n, float* sink, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int blocksPerSm : {4, 8}) {
    for (int rep = 0; rep < 10; ++rep) {
      cudaEventRecord(e0);
      mix<NR, NW><<<sms * blocksPerSm, 512>>>(bufs[0], bufs[1], bufs[2], bufs[3], bufs[4], n, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
  }
  const double bytes = (double)n * 16 * (NR + NW);
  printf("%-28s %8.1f GB/s  (%d reads : %d writes, %.3f ms)\n", name, bytes / (best * 1e-3) / 1e9, NR, NW, best);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = (size_t(1) << 30) / 16;  // 1 GiB per buffer
  float4* bufs[5];
  for (auto& p : bufs) { if (cudaMalloc(&p, n * 16) != cudaSuccess) { printf("alloc failed\n"); return 1; } cudaMemset(p, 0, n * 16); }
  float* sink; cudaMalloc(&sink, 4);
  run<1, 1>("copy (1R:1W)", bufs, n, sink, sms);
  run<3, 1>("3R:1W (fwd/bwd-like)", bufs, n, sink, sms);
  run<3, 2>("3R:2W", bufs, n, sink, sms);
  run<3, 0>("read-only x3", bufs, n, sink, sms);
  run<1, 0>("read-only x1", bufs, n, sink, sms);
  return 0;
}
