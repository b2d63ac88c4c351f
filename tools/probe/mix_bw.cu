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

// The headline kernels' access pattern without their arithmetic: a warp owns 32 consecutive series
// (one 128-B line per [T][B] row) and walks T in 16-row chunks, reading 3 planes and writing 1.
template <int WPB>
__global__ void __launch_bounds__(32 * WPB) tb_walk(const float* __restrict__ a, const float* __restrict__ b,
                                                    const float* __restrict__ c, float* __restrict__ o, int T,
                                                    long long B) {
  const long long col = ((long long)blockIdx.x * WPB + (threadIdx.x >> 5)) * 32 + (threadIdx.x & 31);
  if (col >= B) return;
  float carry = 0.f;
  for (int t0 = 0; t0 < T; t0 += 16) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const long long i = (long long)(t0 + k) * B + col;
      v[k] = (t0 + k < T) ? a[i] + b[i] + c[i] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      carry = carry * 0.5f + v[k];
      if (t0 + k < T) o[(long long)(t0 + k) * B + col] = carry;
    }
  }
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
  {
    const int T = 3288; const long long B = 65536;  // 4 planes of 0.86 GB inside the 1 GiB buffers
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 10; ++rep) {
      cudaEventRecord(e0);
      tb_walk<4><<<(unsigned)(B / 128), 128>>>((const float*)bufs[0], (const float*)bufs[1], (const float*)bufs[2],
                                               (float*)bufs[3], T, B);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-28s %8.1f GB/s  (T=%d B=%lld, 16-row chunks per warp, %.3f ms)\n", "[T][B] warp walk 3R:1W",
           4.0 * T * B * 4 / (best * 1e-3) / 1e9, T, B, best);
  }
  return 0;
}
