// Kernel launchers of libwhit (internal, not part of the ABI).
//
// The launch templates are DECLARED here for every translation unit and DEFINED only where
// WHIT_LAUNCH_DEFS is set: the inst_*.cu units define it and explicitly instantiate one slice of
// the kernel families each, so the sm_100a kernels compile in parallel (make -j) while whit_api.cu
// (dispatch, validation) only references them.
#pragma once
#include <cuda_runtime.h>

#include <atomic>

#include "libwhit.h"
#include "whit_internal.h"
#include "whit_kernels.cuh"
#include "whit_mb2.cuh"
#include "whit_twist.cuh"

namespace whit_detail {

// Dynamic smem budget of one CTA (227 KB opt-in minus the kernels' static barriers).
constexpr int kSmemBudget = 232448 - 2048;

// Single-series daily-grid kernel (forward / backward / fused-loss forward / bit-packed W;
// WD: the forward detects binary W and writes its bit plane, the backward reads it).
template <int D, typename IO, bool PD, bool BWD, bool LOSS = false, bool WB = false>
whit_status launch(const whit::Params& p, cudaStream_t s);
// Multi-band shared-factor kernel (NEXT-1; IRR: on uneven dates, NEXT-2).
template <int D, typename IO, bool PD, bool BWD, bool IRR = false>
whit_status launch_mb2(const whit::Params& p, cudaStream_t s);
// Posterior variance diag(Omega^-1) (NEXT-4).
template <int D, typename IO, bool PD>
whit_status launch_var(const whit::Params& p, cudaStream_t s);
// Single-series irregular-grid kernel (NEXT-2).
template <int D, typename IO, bool PD, bool BWD>
whit_status launch_irr(const whit::Params& p, cudaStream_t s);
// Twisted (two-ended) single-series kernel for small batches (whit_twist.cuh); HIREG: the 255-register build.
template <int D, typename IO, bool PD, bool BWD, bool HIREG = false>
whit_status launch_tw(const whit::Params& p, cudaStream_t s);

#ifdef WHIT_LAUNCH_DEFS
constexpr int kMaxDevices = 64;

// Opt a kernel into its dynamic shared memory once PER DEVICE (the attribute belongs to the
// device context; a workspace on a second GPU must set it again).  A failed attempt is not
// cached, so a later call retries.
template <auto KERNEL>
cudaError_t ensure_smem_attr(int bytes) {
  static std::atomic<int> done[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const bool cacheable = dev >= 0 && dev < kMaxDevices;
  if (cacheable && done[dev].load(std::memory_order_acquire) == bytes) return cudaSuccess;
  cudaFuncSetAttribute(KERNEL, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  const cudaError_t e = cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && cacheable) done[dev].store(bytes, std::memory_order_release);
  return e;
}

inline whit_status launch_error(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return WHIT_OK;
}

template <int D, typename IO, bool PD, bool BWD, bool LOSS, bool WB>
whit_status launch(const whit::Params& p, cudaStream_t s) {
  using L = whit::Layout<D, IO, PD, BWD, LOSS, WB>;
  constexpr int SMEM = whit::WarpAlloc<D, IO, PD, BWD, LOSS, WB>::smem;
  static_assert(SMEM <= kSmemBudget, "CTA shared memory over budget");
  constexpr auto K = whit::whit_kernel<D, IO, PD, BWD, LOSS, WB>;
  const cudaError_t ae = ensure_smem_attr<K>(SMEM);
  if (ae != cudaSuccess) return fail(WHIT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ae));
  // one series per thread, one TMA pipeline per warp (hybrid: only the CTAs of groups [0, g_hi))
  const int threads = 32 * L::WARPS;
  const long long nser = p.g_hi > 0 && 32LL * p.g_hi < p.B ? 32LL * p.g_hi : p.B;
  const long long grid = (nser + threads - 1) / threads;
  K<<<dim3((unsigned)grid), dim3(threads), SMEM, s>>>(p);
  return launch_error("kernel launch");
}

template <int D, typename IO, bool PD, bool BWD, bool IRR>
whit_status launch_mb2(const whit::Params& p, cudaStream_t s) {
  using L = whit::MB2Layout<D, IO, PD, BWD, IRR>;
  constexpr int max_smem = L::smem(whit::kMaxBands);
  constexpr auto K = whit::whit_mb2_kernel<D, IO, PD, BWD, IRR>;
  const cudaError_t ae = ensure_smem_attr<K>(max_smem < kSmemBudget ? max_smem : kSmemBudget);
  if (ae != cudaSuccess) return fail(WHIT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ae));
  const int smem = L::smem(p.nb);
  if (smem > kSmemBudget) return fail(WHIT_ERR_SHAPE, "%d bands need %d B of shared memory", p.nb, smem);
  const long long grid = (p.B + 31) / 32;
  const int threads = 32 * (L::nwarps(p.nb) + 1);
  K<<<dim3((unsigned)grid), dim3(threads), smem, s>>>(p);
  return launch_error("kernel launch");
}

template <int D, typename IO, bool PD>
whit_status launch_var(const whit::Params& p, cudaStream_t s) {
  using V = whit::VarLayout<D, IO, PD>;
  constexpr auto K = whit::whit_var_kernel<D, IO, PD>;
  const cudaError_t ae = ensure_smem_attr<K>(V::SMEM);
  if (ae != cudaSuccess) return fail(WHIT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ae));
  const long long per_cta = 32 * V::WARPS;
  const long long grid = (p.B + per_cta - 1) / per_cta;
  K<<<dim3((unsigned)grid), dim3((unsigned)per_cta), V::SMEM, s>>>(p);
  return launch_error("kernel launch");
}

template <int D, typename IO, bool PD, bool BWD>
whit_status launch_irr(const whit::Params& p, cudaStream_t s) {
  using L = whit::IrrLayout<D, IO, PD, BWD>;
  constexpr auto K = whit::whit_irr_kernel<D, IO, PD, BWD>;
  const cudaError_t ae = ensure_smem_attr<K>(L::SMEM);
  if (ae != cudaSuccess) return fail(WHIT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ae));
  const long long per_cta = 32 * L::WARPS;
  const long long grid = (p.B + per_cta - 1) / per_cta;
  K<<<dim3((unsigned)grid), dim3((unsigned)per_cta), L::SMEM, s>>>(p);
  return launch_error("kernel launch");
}
template <int D, typename IO, bool PD, bool BWD, bool HIREG>
whit_status launch_tw(const whit::Params& p, cudaStream_t s) {
  using L = whit::TwLayout<D, IO, PD, BWD>;
  static_assert(L::SMEM <= kSmemBudget, "CTA shared memory over budget");
  constexpr auto K = whit::whit_tw_kernel<D, IO, PD, BWD, HIREG>;
  const cudaError_t ae = ensure_smem_attr<K>(L::SMEM);
  if (ae != cudaSuccess) return fail(WHIT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ae));
  const long long per_cta = 32 * L::PAIRS;  // series per CTA (two warps per 32 series)
  const long long grid = (p.B + per_cta - 1) / per_cta - p.tw_cta0;  // (hybrid: from CTA tw_cta0 on)
  K<<<dim3((unsigned)grid), dim3(64 * L::PAIRS), L::SMEM, s>>>(p);
  return launch_error("kernel launch");
}
#endif  // WHIT_LAUNCH_DEFS

}  // namespace whit_detail
