// Probe: HBM bandwidth of the headline kernels' access pattern without their arithmetic.  Each
// group of G warps walks its G*32 series of a [T][B] fp32 layout in 16-row chunks through a
// 2-stage TMA ring (box {G*32 series x 16 rows} of 3 input planes), sums the planes and writes
// one output plane with TMA tensor stores.  G = 1 is the per-warp pipeline of whit_kernel;
// G = 2 / 4 share one wider box per warp pair / CTA (longer contiguous DRAM runs, group barriers).
// Dev tool: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_pattern.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);              \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int K = 16, ST = 2, WARPS = 4;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sa(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void load2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(sa(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(sa(b))
      : "memory");
}
__device__ __forceinline__ void store2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0),
               "r"(c1), "r"(sa(src))
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void gbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct Maps {
  CUtensorMap a, b, c, o;
};

template <int G>
__global__ void __launch_bounds__(32 * WARPS) walk(const __grid_constant__ Maps m, int T) {
  constexpr int W = 32 * G, ROWB = W * 4, STAGE = 3 * K * ROWB, NG = WARPS / G;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[NG][ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = warp / G, gw = warp % G;
  unsigned char* ring = smem + grp * (ST * STAGE + K * ROWB);
  float* out = reinterpret_cast<float*>(ring + ST * STAGE);
  const int c0 = (blockIdx.x * NG + grp) * W;
  const int C = (T + K - 1) / K;
  const bool leader = gw == 0 && lane == 0;
  auto issue = [&](int i) {
    unsigned char* s = ring + (i % ST) * STAGE;
    expect(&full[grp][i % ST], 3 * K * ROWB);
    load2d(s, &m.a, c0, i * K, &full[grp][i % ST]);
    load2d(s + K * ROWB, &m.b, c0, i * K, &full[grp][i % ST]);
    load2d(s + 2 * K * ROWB, &m.c, c0, i * K, &full[grp][i % ST]);
  };
  if (leader) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[grp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < ST && i < C; ++i) issue(i);
  }
  if (G > 1) gbar(1 + grp, 32 * G); else __syncwarp();
  float carry = 0.f;
  for (int c = 0; c < C; ++c) {
    const int s = c % ST;
    wait(&full[grp][s], (c / ST) & 1);
    const float* st = reinterpret_cast<const float*>(ring + s * STAGE) + gw * 32 + lane;
    if (leader) wait_read0();
    if (G > 1) gbar(1 + grp, 32 * G); else __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      carry = carry * 0.5f + st[k * W] + st[(K + k) * W] + st[(2 * K + k) * W];
      out[k * W + gw * 32 + lane] = carry;
    }
    fence_async();
    if (G > 1) gbar(1 + grp, 32 * G); else __syncwarp();
    if (leader) {
      store2d(&m.o, out, c0, c * K);
      commit();
      if (c + ST < C) issue(c + ST);
    }
  }
  if (leader) wait_all0();
}

int main() {
  const int T = 3288;
  const long long B = 262144;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  float* buf[4];
  for (auto& p : buf) {
    CK(cudaMalloc(&p, size_t(T) * B * 4));
    CK(cudaMemset(p, 0, size_t(T) * B * 4));
  }
  for (int G : {1, 2, 4}) {
    Maps m;
    CUtensorMap* maps[4] = {&m.a, &m.b, &m.c, &m.o};
    for (int i = 0; i < 4; ++i) {
      cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)T};
      cuuint64_t strides[1] = {(cuuint64_t)B * 4};
      cuuint32_t box[2] = {(cuuint32_t)(32 * G), (cuuint32_t)K};
      cuuint32_t es[2] = {1, 1};
      if (enc(maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf[i], dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
      }
    }
    const int smem = (WARPS / G) * (ST * 3 * K * 32 * G * 4 + K * 32 * G * 4);
    auto kern = G == 1 ? walk<1> : G == 2 ? walk<2> : walk<4>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const unsigned grid = (unsigned)(B / (32 * WARPS));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      kern<<<grid, 32 * WARPS, smem>>>(m, T);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    printf("G=%d (box %3d series x %d rows, smem %6d B/CTA): %.3f ms  %.1f GB/s (3 reads : 1 write)\n", G, 32 * G, K,
           smem, best, 4.0 * T * B * 4 / (best * 1e-3) / 1e9);
  }
  return 0;
}
