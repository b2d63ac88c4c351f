// libwhit device code: fused assemble + banded LDL^T + substitutions for
// (W + D^T diag(lambda) D) z = W y   (Eq. (3); Omega)
// and its adjoint (Eq. (4)-(5)), one series per thread, fp64 math.
//
// Design:
//  * layout [T][B]: one time row of a warp's 32 series is 32 contiguous
//    elements; each warp runs its own TMA pipeline: lane 0 stages 2-D boxes
//    {32 series x K steps} of every input plane into a private shared-memory
//    ring (mbarrier complete_tx), so warps never wait on each other;
//  * the band row of Omega is never materialised: it is assembled in
//    registers from w_t, lambda_{t-d..t} and the constant stencil;
//  * banded LDL^T in "deviation form" (R-10): L = M + A,
//    D_t = lambda_t + Delta_t, where (M, Lambda) is the exact LDL^T of the
//    pure penalty D^T Lambda D; every term is data-scale, no lambda-scale
//    cancellation (the textbook form loses 60-100x accuracy);
//  * "R-mode": the up sweep (factor + forward substitution) writes a
//    fp64 checkpoint of the recurrence state every K steps; the down sweep
//    walks chunks in reverse, recomputes the chunk's factor from its
//    checkpoint (bitwise identical: same instruction sequence, -fmad=false,
//    explicit fma) into registers, and back-substitutes.  No per-step
//    factor is ever written to HBM;
//  * forward emits z and D z (from fp64 registers, cached in the workspace
//    for the backward's lambda gradient); backward re-runs both sweeps on
//    g = dL/dz with the same factor and emits w*u and -(D u)(D z).
#pragma once
#include <cuda.h>
#include <cstdint>
#include <type_traits>

namespace whit {

// ------------------------------------------------------------------ constants
// Non-recursive so that, once the loops are unrolled, every use folds to a
// literal (a recursive constexpr helper is NOT evaluated at compile time in
// device code unless forced, and became a runtime CALL).
// M_j = (-1)^j C(d, j): unit lower-banded column of D^T (M_0 = 1).
__host__ __device__ __forceinline__ constexpr double Mj(int d, int j) {
  return d == 1 ? (j == 0 ? 1.0 : j == 1 ? -1.0 : 0.0)
       : d == 2 ? (j == 0 ? 1.0 : j == 1 ? -2.0 : j == 2 ? 1.0 : 0.0)
                : (j == 0 ? 1.0 : j == 1 ? -3.0 : j == 2 ? 3.0 : j == 3 ? -1.0 : 0.0);
}
// c_j = (-1)^(d-j) C(d, j): a row of D on the daily grid (R-3).
__host__ __device__ __forceinline__ constexpr double Cj(int d, int j) {
  return ((d & 1) ? -1.0 : 1.0) * Mj(d, j);
}

// ------------------------------------------------------------------ kernel parameters
// B = number of pixels; nb = bands per pixel sharing w, lambda and therefore
// Omega (NEXT-1; nb = 1: independent series).  Band planes are
// [nb][rows][B] and use 3-D maps {B, rows, nb}; w and lambda are 2-D [rows][B].
struct Params {
  CUtensorMap tm_rhs;     // y (forward) or grad_z (backward): [nb][T][B], box {32, K, 1}
  CUtensorMap tm_w;       // w: [T][B], box {32, K}
  CUtensorMap tm_lam_up;  // per-date lambda [T-d][B], box {32, K}
  CUtensorMap tm_lam_dn;  // per-date lambda [T-d][B], box {32, K+d} (rows t0-d..t0+K-1)
  CUtensorMap tm_dz;      // D z cache [nb][T-d][B], box {32, K, 1} (backward only)
  CUtensorMap tm_out0;    // z (forward) / grad_y (backward): [nb][T][B], box {32, K, 1}  (TMA store)
  CUtensorMap tm_out1;    // forward: D z cache [nb][T-d][B] (3-D); backward: per-date grad_lambda [T-d][B] (2-D)
  const void* lam_scalar; // [B] (scalar lambda mode)
  const void* lam_plane;  // [T-d][B] (per-date mode; read directly only by the cold failure path)
  void* out0;             // multi-band kernel (direct stores): z (forward) / grad_y (backward) [nb][T][B]
  const void* dz_cache;   // multi-band backward: the forward's D z cache [nb][T-d][B]
  void* out1;             // multi-band forward: D z cache; backward: grad_lambda [T-d][B] per date or [B] scalar
  CUtensorMap tm_lw;      // LOSS: loss weights [T][B], box {32, K}; irregular grid: the dates [T][B], box {32, K+2d}
  CUtensorMap tm_out2;    // LOSS: grad_z = dL/dz [1][T][B], box {32, K, 1} (TMA store)
  void* loss;             // LOSS: per-series loss [B]
  void* out2;             // LOSS: grad_z = dL/dz [T][B] (direct coalesced stores)
  const uint32_t* wbits;  // WB: bit-packed 0/1 weights [ceil(T/32)][B], bit t%32 of word t/32 (caller's, or
                          // the plane the plain forward wrote: binary-W detection, WD below)
  uint32_t* wbits_out;    // WD forward: the bit plane of W [ceil(T/32)][B] it writes (workspace)
  int32_t* wflag;         // WD: per-warp flag [ceil(B/32)]: 1 if all 32 series' w are exactly 0 / 1
                          // (forward writes it, backward reads it; NULL: detection off)
  double* ck_fac;         // factor checkpoints [C][NFAC][B] (forward up sweep; read by every later sweep)
  double* ck_rhs_f;       // forward rhs checkpoints [C][nb][d][B]
  double* ck_rhs_b;       // backward rhs checkpoints [C][nb][d][B]
  int32_t* info;          // [B]
  // twisted factorisation (whit_twist.cuh): maps of the bottom half (planes based at row tw_m), the split row,
  // the chunk counts of the two halves, per-warp-group decision flags (1: solved twisted; 0: by whit_kernel)
  CUtensorMap tmb_rhs, tmb_w, tmb_lam, tmb_dz, tmb_out0, tmb_out1;
  int32_t* twflag;
  int tw_m, tw_C1, tw_C2;
  int tw_filter;          // whit_kernel as the twisted path's fallback: skip warp groups with twflag = 1
  int g_hi;               // hybrid launch (> 0): whit_kernel solves only warp groups [0, g_hi)
  int tw_cta0;            // hybrid launch: the twisted kernel's first CTA (its groups start at 2 * tw_cta0)
  int bwd_fac_from;       // hybrid backward (> 0): groups >= this write the factor checkpoints in the up sweep
                          // (their forward ran twisted, with its own checkpoint layout)
  long long B;
  int T;
  int C;                  // number of K-step chunks = ceil(T / K)
  int nb;                 // bands per pixel
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint (ns): the warp sleeps until the phase completes (or the hint
// expires) instead of spinning, so waiting warps leave the issue slots to the working ones.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (a CUDA error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait_sleep(bar, parity)) {
    if (clock64() - t0 > 20000000000LL) __trap();  // ~10 s at 2 GHz
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a tensor box (no shared memory, no completion): the next tile's bytes start moving from
// HBM one tile earlier than its shared-memory load, which then hits L2.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until the TMA engine has finished READING the smem of all committed stores.
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// Wait until all committed stores are complete (globally visible).
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Named barrier over a subset of the CTA's warps (nthreads a multiple of 32).
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Order this warp's earlier generic-proxy reads of a stage before the TMA
// (async proxy) write that refills it.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// fp64 reciprocal: MUFU.RCP64H seed (~2^-22) + NEWTON Newton steps.  Two steps
// give ~1 ulp (fp64 I/O: the 1e-10 target); one step gives ~2^-44 relative,
// ~1e4x below what the fp32-I/O tolerances can see, and shortens the
// per-row dependency chain by two DFMAs.  Every sweep uses the identical
// sequence, so recomputed factors are bitwise identical.
template <int NEWTON>
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
  for (int i = 0; i < NEWTON; ++i) {
    const double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
  }
  return r;
}
// fp32 I/O at d <= 2: one step (~2^-44, four orders below what fp32 outputs can show).  d = 3 takes two
// steps in fp32 I/O too: its Omega is ill-conditioned enough (long gaps) that a 1e-13 pivot error
// reaches the 3rd differences D z (and so dL/dlambda) at the 1e-2 level on small-|D z| series.
template <typename IO, int D> struct Newton { static constexpr int N = (sizeof(IO) == 4 && D <= 2) ? 1 : 2; };

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000LL); }

// Pivot test of row t (status, R-8): D_t must be a positive NORMAL double below 2^1022, i.e. finite,
// > 0, and with a normal reciprocal.  Biased exponent 1..2044 with the sign bit clear; integer ALU
// work only (no fp64-pipe compare).  A positive subnormal pivot (or one >= 2^1022) has no normal
// reciprocal -- the MUFU seed flushes it -- so it is reported as a failure instead of producing
// silent Inf/NaN with info = 0.  (Exact arithmetic on real data never comes near either bound.)
__device__ __forceinline__ bool pivot_ok(double Dt) {
  return ((static_cast<unsigned>(__double2hiint(Dt)) >> 20) - 1u) < 2044u;
}

// LAPACK-style status from the up sweep: bad = 1-based first failing pivot row (0: none);
// nobs < d days observed means Omega is singular (for lambda > 0) with the zero pivot at row T-d,
// so T-d+1 -- unless a pivot had already failed before that row.
__device__ __forceinline__ int status_info(int bad, int nobs, int d, int T) {
  if (nobs >= d) return bad;
  return (bad != 0 && bad <= T - d) ? bad : T - d + 1;
}

template <typename IO> __device__ __forceinline__ double to_f64(IO v) { return static_cast<double>(v); }
template <typename IO> __device__ __forceinline__ IO from_f64(double v) { return static_cast<IO>(v); }

// Right-hand side of the row: forward b_t = (W y)_t with (W y)_t := 0 where
// w_t = 0 (R-4: values at masked slots, NaN included, never enter), selected
// on the raw I/O value before widening; backward b_t = g_t.
template <typename IO, bool BWD>
__device__ __forceinline__ double rhs_times_w(IO rhs, IO wio, double w) {
  if (BWD) return to_f64<IO>(rhs);
  return w * to_f64<IO>(wio != IO(0) ? rhs : IO(0));
}

// ------------------------------------------------------------------ recurrence state
// State entering row t: values of rows t-1..t-D (index i <-> row t-1-i).
template <int D> struct FState {
  double dl[D];      // Delta[t-1-i]
  double id[D];      // 1 / D[t-1-i]
  double lm[D];      // lambda~[t-1-i]
  double ap[D][D];   // ap[m][k] = A[t-1-m][k+1]   (used: k+1 <= D-1-m)
  double v[D];       // v[t-1-i]  (forward-substituted rhs)
};

// Virtual rows t < 0: Delta = 0, D = 1, lambda~ = 0, A = 0, v = 0 (DESIGN §3 R-10)
template <int D> __device__ __forceinline__ void state_init(FState<D>& s) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    s.dl[i] = 0.0; s.id[i] = 1.0; s.lm[i] = 0.0; s.v[i] = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s.ap[i][k] = 0.0;
  }
}

// One row t of the deviation-form banded LDL^T fused with forward
// substitution.  Recurrences (DESIGN.md §3 R-10, derived there):
//   E_D  = 0
//   E_m  = -sum_{j=m+1..D} ( M_j lam~[t-j] A[t-m][j-m] + E_j (M_{j-m} + A[t-m][j-m]) ),  m = D-1..1
//   A_m  = ( E_m - M_m Delta[t-m] ) / D[t-m]                 (L[t][t-m] = M_m + A_m)
//   Delta_t = w_t - sum_j ( M_j E_j + A_j (M_j lam~[t-j] + E_j) )
//   D_t  = lam~_t + Delta_t                                   (SPD <=> D_t > 0 for all t)
//   v_t  = b_t - sum_j M_j v[t-j] - sum_j A_j v[t-j]
// Outputs A[0..D-1] (= A_{t,1..D}), D_t, 1/D_t, v_t; advances the state.
// Terms with E_D = 0 are dropped at compile time (an fma with a zero operand
// is not foldable under IEEE rules, so it must not be written).
//
// Accumulation order is chosen for latency: terms are added from j = D down to
// j = 1 so that A_1 (the last-computed, on the loop-carried chain
// Delta_{t-1} -> 1/D_{t-1} -> A_{t,1} -> Delta_t) enters last.
template <int D, int NEWTON>
__device__ __forceinline__ void ldl_step(FState<D>& s, double w, double lam_t, double b, double (&A)[D],
                                         double& Dt, double& idt, double& vt) {
  // A[t][j] = c_j / D_{t-j} with c_j the deviation-form numerator; the j = 1 term of the new pivot is
  // summed as (c_1 * inner_1) / D_{t-1} (fma with the reciprocal last), so the loop-carried chain from the
  // previous row's reciprocal to this row's pivot is one fma instead of a multiply and an fma
  double E[D + 1], c[D];
  E[D] = 0.0;
  c[D - 1] = -Mj(D, D) * s.dl[D - 1];
  A[D - 1] = c[D - 1] * s.id[D - 1];
#pragma unroll
  for (int m = D - 1; m >= 1; --m) {
    // j = D term (E_D = 0): - M_D lam~[t-D] A[t-m][D-m]
    double e = (-(Mj(D, D) * s.lm[D - 1])) * s.ap[m - 1][D - m - 1];
#pragma unroll
    for (int j = D - 1; j >= m + 1; --j) {
      const double a = s.ap[m - 1][j - m - 1];
      e = fma(-(Mj(D, j) * s.lm[j - 1]), a, e);
      e = fma(-E[j], a, e);
      e = fma(-Mj(D, j - m), E[j], e);
    }
    E[m] = e;
    c[m - 1] = fma(-Mj(D, m), s.dl[m - 1], e);
    A[m - 1] = c[m - 1] * s.id[m - 1];
  }
  double dl = w;
#pragma unroll
  for (int j = D - 1; j >= 1; --j) dl = fma(-Mj(D, j), E[j], dl);
#pragma unroll
  for (int j = D; j >= 1; --j) {
    const double inner = (j < D) ? fma(Mj(D, j), s.lm[j - 1], E[j]) : Mj(D, j) * s.lm[j - 1];
    dl = (j > 1) ? fma(-A[j - 1], inner, dl) : fma(-s.id[0], c[0] * inner, dl);
  }
  Dt = lam_t + dl;
  idt = rcp64<NEWTON>(Dt);
  double v = b;  // forward substitution; the j = 1 term with L = M + A summed first (as the back substitution)
#pragma unroll
  for (int j = D; j >= 1; --j) {
    if (j > 1) {
      v = fma(-Mj(D, j), s.v[j - 1], v);
      v = fma(-A[j - 1], s.v[j - 1], v);
    } else {
      v = fma(-(Mj(D, 1) + A[0]), s.v[0], v);
    }
  }
  vt = v;
  // advance
#pragma unroll
  for (int i = D - 1; i >= 1; --i) {
    s.dl[i] = s.dl[i - 1]; s.id[i] = s.id[i - 1]; s.lm[i] = s.lm[i - 1]; s.v[i] = s.v[i - 1];
#pragma unroll
    for (int k = 0; k < D; ++k) s.ap[i][k] = s.ap[i - 1][k];
  }
  s.dl[0] = dl; s.id[0] = idt; s.lm[0] = lam_t; s.v[0] = v;
#pragma unroll
  for (int k = 0; k < D; ++k) s.ap[0][k] = A[k];
}

// 4-B global load under a predicate, into a register that keeps its value (0 here) when the predicate is off.
__device__ __forceinline__ uint32_t ld_pred_u32(const uint32_t* a, bool ok) {
  uint32_t v = 0u;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.u32 %0, [%1];\n\t}"
               : "+r"(v) : "l"(a), "r"((uint32_t)ok) : "memory");
  return v;
}

// 8-B global load under a predicate, likewise (checkpoints loaded a chunk ahead: `valid ? load : 0.0`
// compiled to a move of the loaded value into the loop-carried register right after the load, i.e. a wait
// on DRAM latency per chunk).
__device__ __forceinline__ double ld_pred_f64(const double* a, bool ok) {
  double v = 0.0;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.f64 %0, [%1];\n\t}"
               : "+d"(v) : "l"(a), "r"((uint32_t)ok) : "memory");
  return v;
}

// Checkpoint field counts: factor part = D (Delta) + D(D-1)/2 (A), rhs part = D (v).
template <int D> struct Ck {
  static constexpr int NFAC = D + D * (D - 1) / 2;
  static constexpr int NF = NFAC + D;  // forward checkpoint fields
};

// ------------------------------------------------------------------ tiling config
// One warp = 32 series = one TMA pipeline.  K time steps per chunk/tile, ST
// ring stages per warp, WARPS warps per CTA.  K = 16 for d <= 2; d = 3 keeps
// 4 fp64 values per chunk row in registers, so its chunk is 12 steps (WHIT_TILE_K3).
// Registers are granted per SMSP file (16K regs each; cudaFuncGetAttributes:
// maxThreadsPerBlock = 256 at 192 regs, 384 at 168), so 12 warps/SM need <= 168
// regs.  Forward: 4-warp CTAs, 3 per SM (16.8 KB smem per warp).  Backward (one
// more staged plane, 21 KB per warp): 2-warp CTAs at <= 200 regs (8 warps/SM);
// ncu shows both DRAM-bound (~6.0 TB/s), and staging the backward's outputs in
// place to reach 12 warps measured no faster (slower on small batches).
#ifndef WHIT_TILE_K2
#define WHIT_TILE_K2 16
#endif
#ifndef WHIT_FWD_MAXREG
#define WHIT_FWD_MAXREG 168
#endif
#ifndef WHIT_BWD_MAXREG
#define WHIT_BWD_MAXREG 200
#endif
#ifndef WHIT_BWD_WARPS
#define WHIT_BWD_WARPS 2
#endif
#ifndef WHIT_IRR_UP_UNROLL
#define WHIT_IRR_UP_UNROLL 8
#endif
#ifndef WHIT_L2_PREFETCH
#define WHIT_L2_PREFETCH 0
#endif
#ifndef WHIT_BWD_DIRECT  // backward outputs by direct stores: measured slower once W is read as bits (binary-W
#define WHIT_BWD_DIRECT 0  // detection: 5.87 vs 5.41 ms hetero) and equal on soft W (5.58 vs 5.64): TMA stores
#endif
#ifndef WHIT_FWD_DIRECT  // plain forward by direct stores: measured neutral (hetero fwd 5.52-5.56 ms vs 5.51-5.55
#define WHIT_FWD_DIRECT 0  // staged; the forward is register-limited to 12 warps/SM either way), so TMA stores stay
#endif
#ifndef WHIT_TILE_ST
#define WHIT_TILE_ST 2
#endif
#ifndef WHIT_BWD_WB_ST
#define WHIT_BWD_WB_ST 2
#endif
#ifndef WHIT_BWD_WB_DIRECT
#define WHIT_BWD_WB_DIRECT 0
#endif
#ifndef WHIT_FWD_WARPS
#define WHIT_FWD_WARPS 4
#endif
#ifndef WHIT_TILE_K3
#define WHIT_TILE_K3 12
#endif
template <typename IO, int D, bool BWD> struct Tile {
  static constexpr int K = D <= 2 ? WHIT_TILE_K2 : WHIT_TILE_K3;
  static constexpr int ST = WHIT_TILE_ST;
  static constexpr int WARPS = BWD ? WHIT_BWD_WARPS : WHIT_FWD_WARPS;
  static constexpr int MAXREG = BWD ? WHIT_BWD_MAXREG : WHIT_FWD_MAXREG;  // SMSP register files (16K): 3 warps/SMSP need <= 168
};
constexpr int kMaxBands = 10;

template <int D, typename IO, bool PD, bool BWD, bool LOSS = false, bool WB = false> struct Layout {
  // LOSS: 2-warp CTAs (its stage carries the loss weights too: 10 warps/SM fit at <= 200 registers)
  // the bit-packed backward body (WB) may run a deeper ring (WHIT_BWD_WB_ST): without the w rows its stages are
  // smaller, and it runs inside the float layout's per-warp allocation when it serves the plain backward
  static constexpr int K = Tile<IO, D, BWD>::K, ST = (BWD && WB) ? WHIT_BWD_WB_ST : Tile<IO, D, BWD>::ST,
                       WARPS = LOSS ? 2 : Tile<IO, D, BWD>::WARPS;
  static constexpr int ROW = 32 * (int)sizeof(IO);  // bytes of one staged time row (one warp)
  static constexpr int OFF_RHS = 0;
  static constexpr int OFF_W = K * ROW;                        // (absent with WB: w comes as bits)
  static constexpr int OFF_LAM = (WB ? 1 : 2) * K * ROW;
  static constexpr int OFF_DZ = OFF_LAM + (PD ? (K + D) * ROW : 0);
  static constexpr int OFF_LW = OFF_DZ + (BWD ? K * ROW : 0);  // LOSS (forward): loss-weight tile
  static constexpr int STAGE = (OFF_LW + (LOSS ? K * ROW : 0) + 127) / 128 * 128;
  static constexpr int OUT = K * ROW;                        // one staged output plane (TMA store)
  // outputs are staged per chunk and written by TMA tensor stores (staging in the consumed input slots,
  // and direct 128-B warp stores, were measured no faster: DESIGN.md §5)
  // backward outputs by direct coalesced stores (WHIT_BWD_DIRECT): no staging planes, 10 warps/SM
  // (measured +2% backward on homo/hetero; the bit-W backward stays staged: direct was 8% slower there)
  static constexpr bool BDIRECT = BWD && (WB ? WHIT_BWD_WB_DIRECT : WHIT_BWD_DIRECT);
  // plain forward: z and D z by direct coalesced stores too (WHIT_FWD_DIRECT)
  static constexpr bool FDIRECT = !BWD && !WB && !LOSS && WHIT_FWD_DIRECT;
  static constexpr bool DIRECT = BDIRECT || FDIRECT;
  static constexpr int WARP_SMEM = ST * STAGE + (DIRECT ? 0 : 2 * OUT);  // (LOSS: grad_z goes out directly)
  static constexpr int SMEM = WARPS * WARP_SMEM;
  static constexpr uint32_t BYTES_UP = ((WB ? 1 : 2) * K + (PD ? K : 0)) * ROW;
  static constexpr uint32_t BYTES_DN = ((WB ? 1 : 2) * K + (PD ? K + D : 0) + (BWD ? K : 0) + (LOSS ? K : 0)) * ROW;
};

// Shared memory per warp of a whit_kernel instantiation: the plain backward also hosts the bit-packed body
// (warps whose forward found W binary), whose ring may be deeper (WHIT_BWD_WB_ST) -- the larger of the two.
template <int D, typename IO, bool PD, bool BWD, bool LOSS, bool WB> struct WarpAlloc {
  static constexpr int a = Layout<D, IO, PD, BWD, LOSS, WB>::WARP_SMEM;
  static constexpr int b = (BWD && !WB && !LOSS) ? Layout<D, IO, PD, BWD, LOSS, true>::WARP_SMEM : 0;
  static constexpr int value = a > b ? a : b;
  static constexpr int smem = Layout<D, IO, PD, BWD, LOSS, WB>::WARPS * value;
};

// Issue tile i (up sweep tiles 0..C-1, then down sweep C-1..0) of one warp.
// skip_w (binary W detected, WD): the tile's w rows are not loaded -- the consumer reads the bit plane.
template <int D, typename IO, bool PD, bool BWD, bool LOSS = false, bool WB = false>
__device__ __forceinline__ void issue_tile(const Params& p, unsigned char* stage, uint64_t* bar, int i, int C,
                                           int c0, int band, bool skip_w = false) {
  using L = Layout<D, IO, PD, BWD, LOSS, WB>;
  const bool up = i < C;
  const int c = up ? i : 2 * C - 1 - i;
  const int t0 = c * L::K;
  const bool load_w = !WB && !skip_w;
  mbar_arrive_expect_tx(bar, (up ? L::BYTES_UP : L::BYTES_DN) - (load_w || WB ? 0u : uint32_t(L::K * L::ROW)));
  tma_load_3d(stage + L::OFF_RHS, &p.tm_rhs, c0, t0, band, bar);
  if (load_w) tma_load_2d(stage + L::OFF_W, &p.tm_w, c0, t0, bar);
  if (PD) {
    if (up) tma_load_2d(stage + L::OFF_LAM, &p.tm_lam_up, c0, t0, bar);
    else tma_load_2d(stage + L::OFF_LAM, &p.tm_lam_dn, c0, t0 - D, bar);
  }
  if (BWD && !up) tma_load_3d(stage + L::OFF_DZ, &p.tm_dz, c0, t0, band, bar);
  if (LOSS && !up) tma_load_2d(stage + L::OFF_LW, &p.tm_lw, c0, t0, bar);
#if WHIT_L2_PREFETCH
  // the tile after this one (one more tile of HBM traffic in flight per warp, held in L2)
  if (i + 1 < 2 * C) {
    const bool up1 = i + 1 < C;
    const int c1 = up1 ? i + 1 : 2 * C - 2 - i;
    const int t1 = c1 * L::K;
    tma_prefetch_3d(&p.tm_rhs, c0, t1, band);
    if (!WB) tma_prefetch_2d(&p.tm_w, c0, t1);
    if (PD) {
      if (up1) tma_prefetch_2d(&p.tm_lam_up, c0, t1);
      else tma_prefetch_2d(&p.tm_lam_dn, c0, t1 - D);
    }
    if (BWD && !up1) tma_prefetch_3d(&p.tm_dz, c0, t1, band);
  }
#endif
}

// ------------------------------------------------------------------ per-thread sweep bodies
// Weight of row k of a chunk: from the staged w tile, or (ub: bit-packed W -- the caller's (WB) or the
// plane the forward wrote after detecting a binary W) bit k of the chunk's mask.  A bit reconstructs
// w_t = 1 / 0 exactly, so every downstream value is bitwise the float-plane one.
template <typename IO>
__device__ __forceinline__ void row_w(const IO* t_w, uint32_t wm, int k, IO& wio, double& w, bool ub) {
  if (ub) {
    const bool on = (wm >> k) & 1u;
    wio = on ? IO(1) : IO(0);
    w = on ? 1.0 : 0.0;
  } else {
    wio = t_w[k * 32];
    w = to_f64<IO>(wio);
  }
}

// Binary-W detection (WD): is this weight exactly +0 or 1 (bit patterns; -0, soft weights, NaN: no)?
template <typename IO> __device__ __forceinline__ bool w_is_binary(IO v);
template <> __device__ __forceinline__ bool w_is_binary<float>(float v) {
  const unsigned u = __float_as_uint(v);
  return (u == 0u) | (u == 0x3f800000u);
}
template <> __device__ __forceinline__ bool w_is_binary<double>(double v) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
  return (u == 0ull) | (u == 0x3ff0000000000000ull);
}

template <int D, typename IO, bool PD, bool BWD, bool LOSS = false, bool WB = false>
struct Sweep {
  using L = Layout<D, IO, PD, BWD, LOSS, WB>;
  static constexpr int K = L::K;

  // ---- up sweep over one chunk (rows t0..t0+K-1); RAGGED: the chunk reaches row T-D or beyond
  // WD (plain forward): also gathers the chunk's mask bits (cb) and whether every w is exactly 0 / 1.
  static constexpr bool WD = !BWD && !WB;
  template <bool RAGGED>
  static __device__ __forceinline__ void up_chunk(FState<D>& st, const unsigned char* stg, int lane, int t0, int T,
                                                  double lam_s, int& nobs, bool& pos, uint32_t wm, bool ub,
                                                  uint32_t& cb, bool& isbin) {
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + lane;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;
    const int TmD = T - D;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int t = t0 + k;
      if (RAGGED && t >= T) break;  // rows past the end: nothing uses the state after row T-1
      IO wio;
      double w;
      row_w<IO>(t_w, wm, k, wio, w, ub);
      if (WD) {
        cb |= uint32_t(wio != IO(0)) << k;
        isbin = isbin && w_is_binary<IO>(wio);
      }
      double lt = PD ? to_f64<IO>(t_lam[k * 32]) : lam_s;
      if (!PD && RAGGED) lt = (t < TmD) ? lt : 0.0;
      const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, w);
      double A[D], Dt, idt, vt;
      ldl_step<D, Newton<IO, D>::N>(st, w, lt, bb, A, Dt, idt, vt);
      if (!BWD) {
        if (!WB) nobs += (wio > IO(0));  // (WB: counted per chunk with popc)
        pos = pos && pivot_ok(Dt);  // all pivots valid (false on NaN); exact index found in a cold path
      }
    }
  }

  // ---- cold path (failing series only): 1-based row of the first pivot
  // D_t <= 0 / non-finite in the chunk starting at t0, by replaying the chunk
  // from the checkpoint the up sweep stored for it, with exactly the state
  // restore of the down sweep and the same ldl_step (bitwise-identical).
  static __device__ __noinline__ int first_bad_row(const Params& p, int c, long long b, const unsigned char* stg,
                                                   int lane, int t0, int T, double lam_s, uint32_t wm = 0) {
    constexpr int NFAC = Ck<D>::NFAC;
    const long long B = p.B;
    const double* ck = p.ck_fac + (long long)c * NFAC * B + b;
    const IO* lam_plane = reinterpret_cast<const IO*>(p.lam_plane);
    FState<D> st;
    state_init<D>(st);  // v = 0: the pivots do not depend on the right-hand side
    int f = 0;
    for (int i = 0; i < D; ++i) st.dl[i] = ck[(long long)(f++) * B];
    for (int m = 0; m < D - 1; ++m)
      for (int k = 0; k < D - 1 - m; ++k) st.ap[m][k] = ck[(long long)(f++) * B];
    for (int i = 0; i < D; ++i) {
      const int tj = t0 - 1 - i;
      const bool in = tj >= 0 && tj < T - D;
      const double l = !in ? 0.0 : PD ? to_f64<IO>(lam_plane[(long long)tj * B + b]) : lam_s;
      st.lm[i] = l;
      st.id[i] = (tj < 0) ? 1.0 : rcp64<Newton<IO, D>::N>(l + st.dl[i]);
    }
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + lane;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;
    for (int k = 0; k < K && t0 + k < T; ++k) {
      const int t = t0 + k;
      IO wio;
      double w;
      row_w<IO>(t_w, wm, k, wio, w, WB);
      const double lt = PD ? to_f64<IO>(t_lam[k * 32]) : (t < T - D ? lam_s : 0.0);
      const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, w);
      double A[D], Dt, idt, vt;
      ldl_step<D, Newton<IO, D>::N>(st, w, lt, bb, A, Dt, idt, vt);
      if (!pivot_ok(Dt)) return t + 1;
    }
    return 0;
  }

  // ---- one row of the down-sweep recompute: the factor row k (t = t0 + k) of a chunk from the running
  // state, into (Arow, qk = v_t / D_t).  RAGGED: rows past T give q = 0, A = 0 (z = 0 exactly there).
  template <bool RAGGED, bool UB>
  static __device__ __forceinline__ void rec_row(FState<D>& st, const unsigned char* stg, int lane, int k, int t0,
                                                 int T, double lam_s, uint32_t wm, bool ub_rt, double (&Arow)[D],
                                                 double& qk) {
    const bool ub = UB || ub_rt;
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + lane;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;  // row k <-> t0 - D + k
    const int t = t0 + k;
    IO wio;
    double w;
    row_w<IO>(t_w, wm, k, wio, w, ub);
    double lt = PD ? to_f64<IO>(t_lam[(k + D) * 32]) : lam_s;
    if (!PD && RAGGED) lt = (t < T - D) ? lt : 0.0;
    const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, w);
    double Dt, idt, vt;
    ldl_step<D, Newton<IO, D>::N>(st, w, lt, bb, Arow, Dt, idt, vt);
    qk = vt * idt;
    if (RAGGED && t >= T) {
      qk = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) Arow[j] = 0.0;
    }
  }

  // ---- one row of the back substitution: z_t = q_t - sum_j (M_j + A[t+j][j]) z[t+j] with win[i] = the A row of
  // t+1+i, then the row's outputs: z and D z (forward; fused loss), or w u and -(D u)(D z) (backward).
  // Outputs of row t0+k go to the warp's staging tiles so0/so1 (row k, this lane's column; the caller writes
  // them out with TMA stores, which clip rows past T / T-d and columns past B) or, DIRECT, straight to HBM.
  template <bool RAGGED, bool UB>
  static __device__ __forceinline__ void back_row(int k, double qk, const double (&win)[D][D], double (&zw)[D],
                                                  double& lam_acc, const unsigned char* stg, int lane, int t0, int T,
                                                  IO* so0, IO* so1, double two_over_T, uint32_t wm, IO* gz0,
                                                  long long Bst, bool valid, IO* gl0, bool ub_rt) {
    const bool ub = UB || ub_rt;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_dz = reinterpret_cast<const IO*>(stg + L::OFF_DZ) + lane;
    const int TmD = T - D;
    const int t = t0 + k;
    double z = qk;
#pragma unroll
    for (int j = D; j >= 1; --j) {  // z[t+1] (just computed) enters last, with L = M + A summed first:
      if (j > 1) {                   // one fma on the loop-carried chain (every kernel family alike)
        z = fma(-Mj(D, j), zw[j - 1], z);
        z = fma(-win[j - 1][j - 1], zw[j - 1], z);
      } else {
        z = fma(-(Mj(D, 1) + win[0][0]), zw[0], z);
      }
    }
    // (D z)_t = sum_j c_j z[t+j]  (rows t <= T-d-1)
    double dz = Cj(D, 0) * z;
#pragma unroll
    for (int j = 1; j <= D; ++j) dz = fma(Cj(D, j), zw[j - 1], dz);
#pragma unroll
    for (int i = D - 1; i >= 1; --i) zw[i] = zw[i - 1];
    zw[0] = z;
    if (!BWD) {
      if (L::FDIRECT) {  // gz0: z rows, gl0: D z rows of this chunk
        if (valid && (!RAGGED || t < T)) gz0[(long long)k * Bst] = from_f64<IO>(z);
        if (valid && (!RAGGED || t < T - D)) gl0[(long long)k * Bst] = from_f64<IO>(dz);
      } else {
        so0[k * 32] = from_f64<IO>(z);
        so1[k * 32] = from_f64<IO>(dz);
      }
      if (LOSS) {  // masked MSE: L += lw (z - y)^2 / T, g = 2 lw (z - y) / T
        const IO lw = reinterpret_cast<const IO*>(stg + L::OFF_LW)[lane + k * 32];
        const IO yr = reinterpret_cast<const IO*>(stg + L::OFF_RHS)[lane + k * 32];
        const double e = (lw != IO(0)) ? z - to_f64<IO>(yr) : 0.0;  // unscored dates: exactly 0 (y may be NaN)
        const double lwe = to_f64<IO>(lw) * e;
        if (valid && (!RAGGED || t < T)) gz0[(long long)k * Bst] = from_f64<IO>(two_over_T * lwe);
        if (!RAGGED || t < T) lam_acc = fma(lwe, e, lam_acc);  // (forward: lam_acc holds the loss sum)
      }
    } else {
      IO gy, gl = IO(0);
      IO wk;
      double wkd;
      row_w<IO>(t_w, wm, k, wk, wkd, ub);  // (bits: the exact 1 / 0 the float plane holds)
      if (sizeof(IO) == 4 && PD) {
        // fp32 I/O: w*u and -(Du)(Dz) formed from u, Du rounded once to fp32 (<= 1.5 ulp fp32)
        gy = wk * from_f64<IO>(z);
        gl = -(from_f64<IO>(dz) * t_dz[k * 32]);  // D z tile is 0 past row T-d-1
      } else {
        gy = from_f64<IO>(wkd * z);
        const double g = -dz * to_f64<IO>(t_dz[k * 32]);  // D z tile is 0 past row T-d-1
        if (PD) gl = from_f64<IO>(g);
        else if (!RAGGED || t < TmD) lam_acc += g;
      }
      if (L::BDIRECT) {  // gz0: grad_y rows, gl0: grad_lambda rows of this chunk
        if (valid && (!RAGGED || t < T)) gz0[(long long)k * Bst] = gy;
        if (PD && valid && (!RAGGED || t < TmD)) gl0[(long long)k * Bst] = gl;
      } else {
        so0[k * 32] = gy;
        if (PD) so1[k * 32] = gl;
      }
    }
  }

  // ---- down sweep over one chunk: recompute the factor from the restored state, then back-substitute rows
  // t0+K-1..t0 and emit outputs.  cA: the A rows t0+K.. of the chunk processed before (later in time).
  // UB: W read as bits in this chunk (compile-time: the forward picks the instantiation after its warp vote)
  template <bool RAGGED, bool UB = WB>
  static __device__ __forceinline__ void down_chunk(FState<D>& st, double (&cA)[D][D], double (&zw)[D],
                                                    double& lam_acc, const unsigned char* stg, int lane, int t0,
                                                    int T, double lam_s, IO* so0, IO* so1, IO* so2 = nullptr,
                                                    double two_over_T = 0.0, uint32_t wm = 0, IO* gz0 = nullptr,
                                                    long long Bst = 0, bool valid = false, IO* gl0 = nullptr,
                                                    bool ub_rt = WB) {
    double q[K];
    double Ak[K][D];
#pragma unroll
    for (int k = 0; k < K; ++k) rec_row<RAGGED, UB>(st, stg, lane, k, t0, T, lam_s, wm, ub_rt, Ak[k], q[k]);
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      double win[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) win[i][j] = (k + 1 + i < K) ? Ak[k + 1 + i][j] : cA[k + 1 + i - K][j];
      back_row<RAGGED, UB>(k, q[k], win, zw, lam_acc, stg, lane, t0, T, so0, so1, two_over_T, wm, gz0, Bst, valid,
                           gl0, ub_rt);
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) cA[i][j] = Ak[i][j];
  }

};

// ------------------------------------------------------------------ the kernel
// The kernel body of one warp (32 series).  ring / bars: this warp's smem ring (sized by the launching
// layout) and mbarriers; ub: W is read as bits (WB, or the binary-W flag of the plain backward).
template <int D, typename IO, bool PD, bool BWD, bool LOSS, bool WB>
__device__ __forceinline__ void whit_body(const Params& p, unsigned char* ring, uint64_t* bars, int lane,
                                          long long bw, bool ub) {
  using L = Layout<D, IO, PD, BWD, LOSS, WB>;
  using S = Sweep<D, IO, PD, BWD, LOSS, WB>;
  constexpr int K = L::K, ST = L::ST;
  constexpr int NFAC = Ck<D>::NFAC;
  const int T = p.T, C = p.C, nb = 1;
  const long long B = p.B;
  const int band = 0;
  const long long b = bw + lane;
  const bool valid = b < B;
  IO* so0 = reinterpret_cast<IO*>(ring + ST * L::STAGE);             // output staging
  IO* so1 = reinterpret_cast<IO*>(ring + ST * L::STAGE + L::OUT);
  const int ntiles = 2 * C;

  // Binary-W detection (WD): the plain forward gathers the mask bits of its series in the up
  // sweep, writes them to the workspace's bit plane and, if all 32 series of the warp have w in {0, 1},
  // a per-warp flag; from then on its down sweep reads the bits instead of the float w rows (their TMA loads
  // are skipped), and the backward of a flagged warp runs this body with WB = true.
  constexpr bool WD = S::WD;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < ST && i < ntiles; ++i)
      issue_tile<D, IO, PD, BWD, LOSS, WB>(p, ring + i * L::STAGE, &bars[i], i, C, (int)bw, band, ub);
  }
  __syncwarp();

  const double lam_s = (!PD && valid) ? to_f64<IO>(reinterpret_cast<const IO*>(p.lam_scalar)[b]) : 0.0;
  const int cr = (T - D) / K;  // first chunk that reaches row T-D (ragged handling from there on)
  double* const ck_rhs = (BWD ? p.ck_rhs_b : p.ck_rhs_f) + (long long)band * D * B + b;  // + c * nb * D * B
  const long long ck_rhs_stride = (long long)nb * D * B;

  FState<D> st;
  state_init<D>(st);
  int nobs = 0, bad = 0;
  bool allpos = true;
  int it = 0;
  // bits of W (WB, or WD once detected): the chunk's mask bits.  wload() issues the plain coalesced 4-B
  // load(s) of the word(s) holding chunk cc's bits one chunk ahead; wbits_of() extracts them when the chunk
  // starts -- only then, so the in-order warp does not wait on the load right after issuing it (it did:
  // the shift next to the load was the backward's top stall in ncu's source view)
  // (each word comes from a predicated load straight into the register that carries it to the next chunk:
  // a plain `ok ? load : 0` compiled to a move right after the load, which waited on it.  K = 12 (d = 3): a
  // chunk may straddle two words)
  struct WRaw { uint32_t lo, hi; };
  auto wload = [&](int cc) -> WRaw {
    const bool ok = ub && valid && cc >= 0 && cc < C;
    const int bit0 = cc * K, r = bit0 >> 5, sh = bit0 & 31;
    const uint32_t* a = p.wbits + (long long)r * B + b;
    WRaw v;
    v.lo = ld_pred_u32(a, ok);
    v.hi = (32 % K == 0) ? 0u : ld_pred_u32(a + B, ok && sh + K > 32 && (r + 1) * 32 < T);
    return v;
  };
  auto wbits_of = [&](WRaw v, int cc) -> uint32_t {
    const uint64_t two = (uint64_t)v.lo | ((uint64_t)v.hi << 32);
    return (uint32_t)(two >> ((cc * K) & 31)) & (K >= 32 ? 0xffffffffu : ((1u << K) - 1u));
  };
  WRaw wm_next = wload(0);
  uint64_t wacc = 0;   // WD: mask bits of rows wbase*32.. not yet stored
  int wbase = 0;
  bool isbin = true;   // WD: every w of this series so far is exactly 0 or 1

  // ================================================================ up sweep
  for (int c = 0; c < C; ++c, ++it) {
    const int s = it % ST;
    const uint32_t wm = wbits_of(wm_next, c);
    wm_next = wload(c + 1);
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * L::STAGE;
    const int t0 = c * K;
    if (valid) {  // checkpoint: state entering row t0
      if (!BWD || (p.bwd_fac_from > 0 && (bw >> 5) >= p.bwd_fac_from)) {
        double* ck = p.ck_fac + (long long)c * NFAC * B + b;
        int f = 0;
#pragma unroll
        for (int i = 0; i < D; ++i) ck[(long long)(f++) * B] = st.dl[i];
#pragma unroll
        for (int m = 0; m < D - 1; ++m)
#pragma unroll
          for (int k = 0; k < D - 1 - m; ++k) ck[(long long)(f++) * B] = st.ap[m][k];
      }
      double* ck = ck_rhs + (long long)c * ck_rhs_stride;
#pragma unroll
      for (int i = 0; i < D; ++i) ck[(long long)i * B] = st.v[i];
    }
    bool pos = true;
    uint32_t cb = 0;
    if (c < cr) S::template up_chunk<false>(st, stg, lane, t0, T, lam_s, nobs, pos, wm, ub, cb, isbin);
    else S::template up_chunk<true>(st, stg, lane, t0, T, lam_s, nobs, pos, wm, ub, cb, isbin);
    if (WB && !BWD) nobs += __popc(wm);  // bits past T are 0 (packing)
    if (WD && p.wflag != nullptr) {  // append the chunk's K bits; store each completed 32-row word
      wacc |= uint64_t(cb) << (t0 - wbase * 32);
      if (t0 + K >= (wbase + 1) * 32) {
        if (valid) p.wbits_out[(long long)wbase * B + b] = uint32_t(wacc);
        wacc >>= 32;
        ++wbase;
      }
    }
    allpos = allpos && pos;
    // exact failing row (cold path): replayed from the factor checkpoint this warp wrote
    if (!BWD && !pos && bad == 0 && valid) bad = S::first_bad_row(p, c, b, stg, lane, t0, T, lam_s, wm);
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue_tile<D, IO, PD, BWD, LOSS, WB>(p, ring + s * L::STAGE, &bars[s], it + ST, C, (int)bw, band, ub);
    }
  }
  if (WD && p.wflag != nullptr) {  // last partial word, the warp's vote, and bits from here on
    if (valid && wbase * 32 < T) p.wbits_out[(long long)wbase * B + b] = uint32_t(wacc);
    const bool all_bin = __all_sync(0xffffffffu, isbin || !valid);
    if (lane == 0) p.wflag[bw >> 5] = all_bin ? 1 : 0;
    ub = all_bin;  // (this lane's own stores above are what wload() reads back)
  }

  // Status (LAPACK xPBTRF style): fewer than d observed days -> T-d+1 (exactly
  // singular for lambda > 0); else first non-positive pivot row.  A failed
  // series is poisoned with NaN in the restored rhs state, so every output
  // derived from it (z, D z, w*u, -(D u)(D z)) is NaN without per-store checks.
  bool failed;
  if (!BWD) {
    const int info = status_info(bad, nobs, D, T);
    if (valid) p.info[b] = info;
    failed = info != 0 || !allpos;
  } else {
    failed = valid ? (p.info[b] != 0) : true;
  }
  const double poison = failed ? qnan() : 0.0;

  // ================================================================ down sweep
  double cA[D][D];  // A[t0+K+i][j+1] of the chunk processed before (later in time)
  double zw[D];     // z[t+1..t+D] window (u in the backward)
#pragma unroll
  for (int i = 0; i < D; ++i) {
    zw[i] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) cA[i][j] = 0.0;
  }
  double lam_acc = 0.0;  // scalar-lambda gradient accumulator

  // checkpoint prefetch registers (next chunk to process)
  double pdl[D], pap[NFAC - D > 0 ? NFAC - D : 1], pv[D];
#define WHIT_LOAD_CK(cc)                                                                          \
  do {                                                                                            \
    if (valid) {                                                                                  \
      const double* ckf = p.ck_fac + (long long)(cc) * NFAC * B + b;                              \
      _Pragma("unroll") for (int i = 0; i < D; ++i) pdl[i] = ckf[(long long)i * B];               \
      _Pragma("unroll") for (int f = 0; f < NFAC - D; ++f) pap[f] = ckf[(long long)(D + f) * B];  \
      const double* ckr = ck_rhs + (long long)(cc) * ck_rhs_stride;                               \
      _Pragma("unroll") for (int i = 0; i < D; ++i) pv[i] = ckr[(long long)i * B];                \
    }                                                                                             \
  } while (0)
  WHIT_LOAD_CK(C - 1);
  wm_next = wload(C - 1);

  for (int c = C - 1; c >= 0; --c, ++it) {
    const int s = it % ST;
    const uint32_t wm = wbits_of(wm_next, c);
    wm_next = wload(c - 1);
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * L::STAGE;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;  // row k <-> t0 - D + k
    const int t0 = c * K;

    // restore the state entering row t0 from the checkpoint
    {
      int f = 0;
#pragma unroll
      for (int m = 0; m < D - 1; ++m)
#pragma unroll
        for (int k = 0; k < D - 1 - m; ++k) st.ap[m][k] = pap[f++];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const int tj = t0 - 1 - i;
        st.dl[i] = pdl[i];
        st.v[i] = pv[i] + poison;
        const double l = PD ? to_f64<IO>(t_lam[(D - 1 - i) * 32]) : ((tj >= 0 && tj < T - D) ? lam_s : 0.0);
        st.lm[i] = l;
        st.id[i] = (tj < 0) ? 1.0 : rcp64<Newton<IO, D>::N>(l + pdl[i]);
      }
    }
    if (c > 0) WHIT_LOAD_CK(c - 1);

    // the staging tiles must have been read by the previous chunk's TMA stores
    if (!L::DIRECT) {
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
    }
    const double two_over_T = 2.0 / (double)T;
    IO* const gz0 = LOSS ? reinterpret_cast<IO*>(p.out2) + (long long)t0 * B + b
                  : L::DIRECT ? reinterpret_cast<IO*>(p.out0) + (long long)t0 * B + b : nullptr;
    IO* const gl0 = ((L::BDIRECT && PD) || L::FDIRECT) ? reinterpret_cast<IO*>(p.out1) + (long long)t0 * B + b
                                                       : nullptr;
    // W as bits in the down sweep: WB bodies always; the plain forward once its warp vote found W binary
    // (a warp-uniform branch between two compile-time instantiations, no per-row bit / float select:
    // hetero forward 5.00 vs 5.12 ms).  Per-date lambda only: with scalar lambda the second instantiation
    // spills at 168 registers (homo forward 1.77 vs 1.65 ms), so there the runtime select stays.
    if (WD && PD && ub) {
      if (c < cr)
        S::template down_chunk<false, true>(st, cA, zw, lam_acc, stg, lane, t0, T, lam_s, so0 + lane, so1 + lane,
                                            nullptr, two_over_T, wm, gz0, B, valid, gl0);
      else
        S::template down_chunk<true, true>(st, cA, zw, lam_acc, stg, lane, t0, T, lam_s, so0 + lane, so1 + lane,
                                           nullptr, two_over_T, wm, gz0, B, valid, gl0);
    } else if (c < cr) {
      S::template down_chunk<false>(st, cA, zw, lam_acc, stg, lane, t0, T, lam_s, so0 + lane, so1 + lane,
                                    nullptr, two_over_T, wm, gz0, B, valid, gl0, ub);
    } else {
      S::template down_chunk<true>(st, cA, zw, lam_acc, stg, lane, t0, T, lam_s, so0 + lane, so1 + lane,
                                   nullptr, two_over_T, wm, gz0, B, valid, gl0, ub);
    }
    fence_proxy_async_smem();  // make this lane's staged outputs visible to the TMA engine
    __syncwarp();
    if (lane == 0 && !L::DIRECT) {
      tma_store_3d(&p.tm_out0, so0, (int)bw, t0, band);
      if (!BWD) tma_store_3d(&p.tm_out1, so1, (int)bw, t0, band);
      if (BWD && PD) tma_store_2d(&p.tm_out1, so1, (int)bw, t0);
      bulk_commit();
    }
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue_tile<D, IO, PD, BWD, LOSS, WB>(p, ring + s * L::STAGE, &bars[s], it + ST, C, (int)bw, band, ub);
    }
  }
#undef WHIT_LOAD_CK
  if (lane == 0) bulk_wait0();  // stores complete before the CTA exits (smem stays valid)
  if (LOSS && valid) reinterpret_cast<IO*>(p.loss)[b] = from_f64<IO>(lam_acc / (double)T);
  if (BWD && !PD && valid) reinterpret_cast<IO*>(p.out1)[b] = from_f64<IO>(lam_acc);
}

// One launch = one full forward (BWD=false) or backward (BWD=true) of independent series.  Each
// warp owns 32 consecutive series (one per lane) and its own TMA ring: up sweep over C chunks,
// then down sweep over C chunks in reverse; WARPS independent warps per CTA.  (Multi-band
// pixels sharing a factor use whit_mb2_kernel, whit_mb2.cuh.)  The plain backward runs a warp whose
// forward found W binary with the compile-time bit-packed body (no per-row bit / float select).
template <int D, typename IO, bool PD, bool BWD, bool LOSS = false, bool WB = false>
__global__ void __maxnreg__((LOSS ? 200 : Tile<IO, D, BWD>::MAXREG)) whit_kernel(const __grid_constant__ Params p) {
  static_assert(!LOSS || !BWD, "the fused loss is a forward variant");
  static_assert(!WB || !LOSS, "bit-packed W is a fwd/bwd variant");
  using L = Layout<D, IO, PD, BWD, LOSS, WB>;
  extern __shared__ __align__(1024) unsigned char smem[];
  // mbarriers: enough for the bit-packed backward body's ring too (WHIT_BWD_WB_ST)
  constexpr int NBAR = Layout<D, IO, PD, BWD, LOSS, true>::ST > L::ST ? Layout<D, IO, PD, BWD, LOSS, true>::ST : L::ST;
  __shared__ __align__(8) uint64_t full_bar[L::WARPS][NBAR];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long bw = ((long long)blockIdx.x * L::WARPS + warp) * 32;
  if (bw >= p.B) return;  // past the end; no barrier follows for these warps
  if (p.g_hi > 0 && (bw >> 5) >= p.g_hi) return;       // hybrid: the twisted kernel's groups
  if (p.tw_filter && p.twflag[bw >> 5] != 0) return;  // solved by the twisted kernel
  unsigned char* ring = smem + warp * WarpAlloc<D, IO, PD, BWD, LOSS, WB>::value;
  if constexpr (BWD && !WB && !LOSS) {
    if (p.wflag != nullptr && p.wflag[bw >> 5] != 0) {
      whit_body<D, IO, PD, BWD, LOSS, true>(p, ring, full_bar[warp], lane, bw, true);
      return;
    }
  }
  whit_body<D, IO, PD, BWD, LOSS, WB>(p, ring, full_bar[warp], lane, bw, WB);
}

// ------------------------------------------------------------------ irregular grid (NEXT-2)
// The paper's operator on uneven acquisition dates t_0 < ... < t_{T-1} (dspline
// divided differences): row r of D has coefficients
//   c_{r,j} = (d-1)! (t_{r+d} - t_r) / prod_{i != j} (t_{r+j} - t_{r+i}),   j = 0..d.
// Deviation form with a column-dependent unit factor (R-18): column k of M~ is d_k / c_{k,0}
// (normalised stencil mu_k[j] = c_{k,j} / c_{k,0}, mu_k[0] = 1) and Lambda~_k = lambda_k c_{k,0}^2,
// so D^T Lambda D = M~ Lambda~ M~^T again and the recurrences of R-10 hold with M_j replaced by
// M~[t][t-j] = mu_{t-j}[j] and M_{j-m} by M~[t-m][t-j] = mu_{t-j}[j-m].  Columns k < 0 and
// k >= T-d (no difference row) use the binomial M (their Lambda~ is 0, any unit column works).
template <int D> struct IState {
  FState<D> f;
  double mu[D][D];  // mu[i][j] = mu_{t-1-i}[j+1]
};

// Normalised stencil of column k (times tk[0..D] = t_k..t_{k+D}) and its c_{k,0}.
template <int D, int NEWTON>
__device__ __forceinline__ void col_stencil(const double (&tk)[D + 1], double (&mu)[D], double& c0) {
  if (D == 1) {
    mu[0] = -1.0;
    c0 = -1.0;
  } else if (D == 2) {
    const double h1 = tk[1] - tk[0], h2 = tk[2] - tk[1];
    const double r2 = rcp64<NEWTON>(h2);
    mu[1] = h1 * r2;
    mu[0] = -1.0 - mu[1];
    c0 = rcp64<NEWTON>(h1);
  } else {
    double P[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) {
      double p = 1.0;
#pragma unroll
      for (int i = 0; i <= D; ++i)
        if (i != j) p *= (tk[j] - tk[i]);
      P[j] = p;
    }
    const double rp0 = rcp64<NEWTON>(P[0]);
#pragma unroll
    for (int j = 1; j <= D; ++j) mu[j - 1] = P[0] * rcp64<NEWTON>(P[j]);
    double fact = 1.0;
#pragma unroll
    for (int i = 2; i < D; ++i) fact *= i;
    c0 = fact * (tk[D] - tk[0]) * rp0;
  }
}

template <int D>
__device__ __forceinline__ void binomial_col(double (&mu)[D]) {
#pragma unroll
  for (int j = 1; j <= D; ++j) mu[j - 1] = Mj(D, j);
}

template <int D, int NEWTON>
__device__ __forceinline__ void ldl_step_irr(IState<D>& S, const double (&mu_t)[D], double w, double lam_t,
                                             double b, double (&A)[D], double& Dt, double& idt, double& vt) {
  FState<D>& s = S.f;
  // Mt[j] = M~[t][t-j] = mu_{t-j}[j] = S.mu[j-1][j-1];  Mm(m, j) = M~[t-m][t-j] = S.mu[j-1][j-m-1]
  double E[D + 1], c[D];  // (the j = 1 term with the reciprocal last, as ldl_step)
  E[D] = 0.0;
  c[D - 1] = -S.mu[D - 1][D - 1] * s.dl[D - 1];
  A[D - 1] = c[D - 1] * s.id[D - 1];
#pragma unroll
  for (int m = D - 1; m >= 1; --m) {
    double e = (-(S.mu[D - 1][D - 1] * s.lm[D - 1])) * s.ap[m - 1][D - m - 1];
#pragma unroll
    for (int j = D - 1; j >= m + 1; --j) {
      const double a = s.ap[m - 1][j - m - 1];
      e = fma(-(S.mu[j - 1][j - 1] * s.lm[j - 1]), a, e);
      e = fma(-E[j], a, e);
      e = fma(-S.mu[j - 1][j - m - 1], E[j], e);
    }
    E[m] = e;
    c[m - 1] = fma(-S.mu[m - 1][m - 1], s.dl[m - 1], e);
    A[m - 1] = c[m - 1] * s.id[m - 1];
  }
  double dl = w;
#pragma unroll
  for (int j = D - 1; j >= 1; --j) dl = fma(-S.mu[j - 1][j - 1], E[j], dl);
#pragma unroll
  for (int j = D; j >= 1; --j) {
    const double inner = (j < D) ? fma(S.mu[j - 1][j - 1], s.lm[j - 1], E[j]) : S.mu[j - 1][j - 1] * s.lm[j - 1];
    dl = (j > 1) ? fma(-A[j - 1], inner, dl) : fma(-s.id[0], c[0] * inner, dl);
  }
  Dt = lam_t + dl;
  idt = rcp64<NEWTON>(Dt);
  double v = b;  // (the j = 1 term with L = M~ + A summed first, as ldl_step)
#pragma unroll
  for (int j = D; j >= 1; --j) {
    if (j > 1) {
      v = fma(-S.mu[j - 1][j - 1], s.v[j - 1], v);
      v = fma(-A[j - 1], s.v[j - 1], v);
    } else {
      v = fma(-(S.mu[0][0] + A[0]), s.v[0], v);
    }
  }
  vt = v;
#pragma unroll
  for (int i = D - 1; i >= 1; --i) {
    s.dl[i] = s.dl[i - 1]; s.id[i] = s.id[i - 1]; s.lm[i] = s.lm[i - 1]; s.v[i] = s.v[i - 1];
#pragma unroll
    for (int k = 0; k < D; ++k) { s.ap[i][k] = s.ap[i - 1][k]; S.mu[i][k] = S.mu[i - 1][k]; }
  }
  s.dl[0] = dl; s.id[0] = idt; s.lm[0] = lam_t; s.v[0] = v;
#pragma unroll
  for (int k = 0; k < D; ++k) { s.ap[0][k] = A[k]; S.mu[0][k] = mu_t[k]; }
}

// Stage: rhs K rows, w K rows, times K+2D rows (t0-D .. t0+K+D-1), lambda (K / K+D rows), D z K rows.
template <int D, typename IO, bool PD, bool BWD>
struct IrrLayout {
  // d = 3 holds a 3 x 3 stencil window per row: more registers, so 2-warp CTAs at <= 224 registers
  static constexpr int K = 8, ST = 2, WARPS = D == 3 ? 2 : 4;  // (the kernel caps d = 3 at 224 registers)
  static constexpr int ROW = 32 * (int)sizeof(IO);
  static constexpr int OFF_RHS = 0;
  static constexpr int OFF_W = K * ROW;
  static constexpr int OFF_TT = 2 * K * ROW;
  static constexpr int OFF_LAM = OFF_TT + (K + 2 * D) * ROW;
  static constexpr int OFF_DZ = OFF_LAM + (PD ? (K + D) * ROW : 0);
  static constexpr int STAGE = (OFF_DZ + (BWD ? K * ROW : 0) + 127) / 128 * 128;
  static constexpr int OUT = K * ROW;
  static constexpr int WARP_SMEM = ST * STAGE + 2 * OUT;
  static constexpr int SMEM = WARPS * WARP_SMEM;
  static constexpr uint32_t BYTES_UP = (2 * K + (K + 2 * D) + (PD ? K : 0)) * ROW;
  static constexpr uint32_t BYTES_DN = (2 * K + (K + 2 * D) + (PD ? K + D : 0) + (BWD ? K : 0)) * ROW;
};

template <int D, typename IO, bool PD, bool BWD>
__device__ __forceinline__ void issue_tile_irr(const Params& p, unsigned char* stage, uint64_t* bar, int i, int C,
                                               int c0) {
  using L = IrrLayout<D, IO, PD, BWD>;
  const bool up = i < C;
  const int c = up ? i : 2 * C - 1 - i;
  const int t0 = c * L::K;
  mbar_arrive_expect_tx(bar, up ? L::BYTES_UP : L::BYTES_DN);
  tma_load_3d(stage + L::OFF_RHS, &p.tm_rhs, c0, t0, 0, bar);
  tma_load_2d(stage + L::OFF_W, &p.tm_w, c0, t0, bar);
  tma_load_2d(stage + L::OFF_TT, &p.tm_lw, c0, t0 - D, bar);  // times (tm_lw reused: box K+2D)
  if (PD) {
    if (up) tma_load_2d(stage + L::OFF_LAM, &p.tm_lam_up, c0, t0, bar);
    else tma_load_2d(stage + L::OFF_LAM, &p.tm_lam_dn, c0, t0 - D, bar);
  }
  if (BWD && !up) tma_load_3d(stage + L::OFF_DZ, &p.tm_dz, c0, t0, 0, bar);
}

// mu and c0 of column k = t0 + kk (kk may be in [-D, K)), times tile row index kk + D.
template <int D, typename IO, int NEWTON>
__device__ __forceinline__ void tile_col(const IO* tt, int kk, int k, int T, double (&mu)[D], double& c0,
                                         bool check = true) {
  if (check && (k < 0 || k >= T - D)) {
    binomial_col<D>(mu);
    c0 = 0.0;
    return;
  }
  double tk[D + 1];
#pragma unroll
  for (int j = 0; j <= D; ++j) tk[j] = to_f64<IO>(tt[(kk + D + j) * 32]);
  col_stencil<D, NEWTON>(tk, mu, c0);
}

template <int D, typename IO, bool PD, bool BWD>
__global__ void __maxnreg__((D == 3 ? 224 : 168)) whit_irr_kernel(const __grid_constant__ Params p) {
  using L = IrrLayout<D, IO, PD, BWD>;
  constexpr int K = L::K, ST = L::ST, WARPS = L::WARPS;
  constexpr int UP_UNROLL = WHIT_IRR_UP_UNROLL;
  constexpr int NFAC = Ck<D>::NFAC;
  constexpr int NW = Newton<IO, D>::N;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[WARPS][ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = p.T, C = p.C, TmD = T - D;
  const long long B = p.B;
  const long long bw = ((long long)blockIdx.x * WARPS + warp) * 32;
  if (bw >= B) return;
  const long long b = bw + lane;
  const bool valid = b < B;
  unsigned char* ring = smem + warp * L::WARP_SMEM;
  IO* so0 = reinterpret_cast<IO*>(ring + ST * L::STAGE);
  IO* so1 = reinterpret_cast<IO*>(ring + ST * L::STAGE + L::OUT);
  uint64_t* bars = full_bar[warp];
  const int ntiles = 2 * C;
  if (lane == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < ST && i < ntiles; ++i)
      issue_tile_irr<D, IO, PD, BWD>(p, ring + i * L::STAGE, &bars[i], i, C, (int)bw);
  }
  __syncwarp();
  const double lam_s = (!PD && valid) ? to_f64<IO>(reinterpret_cast<const IO*>(p.lam_scalar)[b]) : 0.0;
  double* const ck_rhs = (BWD ? p.ck_rhs_b : p.ck_rhs_f) + b;

  IState<D> S;
  state_init<D>(S.f);
#pragma unroll
  for (int i = 0; i < D; ++i) binomial_col<D>(S.mu[i]);
  int nobs = 0, bad = 0;  // bad: 1-based first failing pivot row
  int it = 0;
  // ================================================================ up sweep
  for (int c = 0; c < C; ++c, ++it) {
    const int s = it % ST;
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * L::STAGE;
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + lane;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_tt = reinterpret_cast<const IO*>(stg + L::OFF_TT) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;
    const int t0 = c * K;
    if (valid) {
      if (!BWD) {
        double* ck = p.ck_fac + (long long)c * NFAC * B + b;
        int f = 0;
#pragma unroll
        for (int i = 0; i < D; ++i) ck[(long long)(f++) * B] = S.f.dl[i];
#pragma unroll
        for (int m = 0; m < D - 1; ++m)
#pragma unroll
          for (int k = 0; k < D - 1 - m; ++k) ck[(long long)(f++) * B] = S.f.ap[m][k];
      }
      double* ck = ck_rhs + (long long)c * D * B;
#pragma unroll
      for (int i = 0; i < D; ++i) ck[(long long)i * B] = S.f.v[i];
    }
    // EDGE: the chunk touches rows >= T - D (no difference row / past the end): per-row checks; interior
    // chunks (the steady state) run without them
    auto up_rows = [&](auto edge_tag) {
      constexpr bool EDGE = decltype(edge_tag)::value;
#pragma unroll UP_UNROLL
      for (int k = 0; k < K; ++k) {
        const int t = t0 + k;
        if (EDGE && t >= T) break;
        const IO wio = t_w[k * 32];
        const double w = to_f64<IO>(wio);
        double mu_t[D], c0;
        tile_col<D, IO, NW>(t_tt, k, t, T, mu_t, c0, EDGE);
        const double lraw = PD ? to_f64<IO>(t_lam[k * 32]) : lam_s;
        const double lt = (!EDGE || t < TmD) ? lraw * c0 * c0 : 0.0;  // Lambda~_t = lambda_t c_{t,0}^2
        const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, w);
        double A[D], Dt, idt, vt;
        ldl_step_irr<D, NW>(S, mu_t, w, lt, bb, A, Dt, idt, vt);
        if (!BWD) {
          nobs += (wio > IO(0));
          if (bad == 0 && !pivot_ok(Dt)) bad = t + 1;
        }
      }
    };
    if (t0 + K > TmD) up_rows(std::true_type{});
    else up_rows(std::false_type{});
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue_tile_irr<D, IO, PD, BWD>(p, ring + s * L::STAGE, &bars[s], it + ST, C, (int)bw);
    }
  }
  bool failed;
  if (!BWD) {
    const int info = status_info(bad, nobs, D, T);
    if (valid) p.info[b] = info;
    failed = info != 0;
  } else {
    failed = valid ? (p.info[b] != 0) : true;
  }
  const double poison = failed ? qnan() : 0.0;

  // ================================================================ down sweep
  double cA[D][D], cM[D][D];  // A[t0+K+i][j+1] and mu_{t0+K+i}[j+1] of the later chunk
  double zw[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    zw[i] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) { cA[i][j] = 0.0; cM[i][j] = Mj(D, j + 1); }
  }
  double lam_acc = 0.0;
  // checkpoints of the next chunk, loaded one chunk ahead (their latency leaves the chunk's start)
  double pck[NFAC], pv[D];
  auto load_ck = [&](int cc) {
    const double* ckf = p.ck_fac + (long long)cc * NFAC * B + b;
    const double* ckr = ck_rhs + (long long)cc * D * B;
#pragma unroll
    for (int f = 0; f < NFAC; ++f) pck[f] = ld_pred_f64(ckf + (long long)f * B, valid);
#pragma unroll
    for (int i = 0; i < D; ++i) pv[i] = ld_pred_f64(ckr + (long long)i * B, valid);
  };
  load_ck(C - 1);
  for (int c = C - 1; c >= 0; --c, ++it) {
    const int s = it % ST;
    // restore the state entering row t0
    {
      int f = 0;
#pragma unroll
      for (int i = 0; i < D; ++i) S.f.dl[i] = pck[f++];
#pragma unroll
      for (int m = 0; m < D - 1; ++m)
#pragma unroll
        for (int k = 0; k < D - 1 - m; ++k) S.f.ap[m][k] = pck[f++];
#pragma unroll
      for (int i = 0; i < D; ++i) S.f.v[i] = pv[i] + poison;
    }
    if (c > 0) load_ck(c - 1);
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * L::STAGE;
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + lane;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_tt = reinterpret_cast<const IO*>(stg + L::OFF_TT) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;  // row k <-> t0 - D + k
    const IO* t_dz = reinterpret_cast<const IO*>(stg + L::OFF_DZ) + lane;
    const int t0 = c * K;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int tj = t0 - 1 - i;
      double c0;
      tile_col<D, IO, NW>(t_tt, -1 - i, tj, T, S.mu[i], c0);
      const double lraw = PD ? to_f64<IO>(t_lam[(D - 1 - i) * 32]) : lam_s;
      const double l = (tj >= 0 && tj < TmD) ? lraw * c0 * c0 : 0.0;
      S.f.lm[i] = l;
      S.f.id[i] = (tj < 0) ? 1.0 : rcp64<NW>(l + S.f.dl[i]);
    }
    auto down_rows = [&](auto edge_tag) {
      constexpr bool EDGE = decltype(edge_tag)::value;  // the chunk touches rows >= T - D
      double q[K], Ak[K][D], Mk[K][D], c0k[K];
  #pragma unroll
      for (int k = 0; k < K; ++k) {
        const int t = t0 + k;
        const IO wio = t_w[k * 32];
        const double w = to_f64<IO>(wio);
        double c0;
        tile_col<D, IO, NW>(t_tt, k, t, T, Mk[k], c0, EDGE);
        c0k[k] = c0;
        const double lraw = PD ? to_f64<IO>(t_lam[(k + D) * 32]) : lam_s;
        const double lt = (!EDGE || t < TmD) ? lraw * c0 * c0 : 0.0;
        const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, w);
        double Dt, idt, vt;
        ldl_step_irr<D, NW>(S, Mk[k], w, lt, bb, Ak[k], Dt, idt, vt);
        q[k] = vt * idt;
        if (EDGE && t >= T) {
          q[k] = 0.0;
  #pragma unroll
          for (int j = 0; j < D; ++j) Ak[k][j] = 0.0;
        }
      }
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
  #pragma unroll
      for (int k = K - 1; k >= 0; --k) {
        const int t = t0 + k;
        double z = q[k];
        // z_t = q_t - sum_j (M~[t+j][t] + A[t+j][j]) z_{t+j},  M~[t+j][t] = mu_t[j]
  #pragma unroll
        for (int j = D; j >= 1; --j) {
          const double a = (k + j < K) ? Ak[k + j][j - 1] : cA[k + j - K][j - 1];
          if (j > 1) {
            z = fma(-Mk[k][j - 1], zw[j - 1], z);
            z = fma(-a, zw[j - 1], z);
          } else {
            z = fma(-(Mk[k][0] + a), zw[0], z);  // (L = M~ + A first, as Sweep::back_row)
          }
        }
        // (D z)_t = c_{t,0} (z_t + sum_j mu_t[j] z_{t+j})
        double u = z;
  #pragma unroll
        for (int j = 1; j <= D; ++j) u = fma(Mk[k][j - 1], zw[j - 1], u);
        const double dz = c0k[k] * u;
  #pragma unroll
        for (int i = D - 1; i >= 1; --i) zw[i] = zw[i - 1];
        zw[0] = z;
        if (!BWD) {
          so0[k * 32 + lane] = from_f64<IO>(z);
          so1[k * 32 + lane] = from_f64<IO>(dz);
        } else {
          const double w = to_f64<IO>(t_w[k * 32]);
          so0[k * 32 + lane] = from_f64<IO>(w * z);
          const double g = -dz * to_f64<IO>(t_dz[k * 32]);
          if (PD) so1[k * 32 + lane] = from_f64<IO>(g);
          else if (!EDGE || t < TmD) lam_acc += g;
        }
      }
  #pragma unroll
      for (int i = 0; i < D; ++i)
  #pragma unroll
        for (int j = 0; j < D; ++j) { cA[i][j] = Ak[i][j]; cM[i][j] = Mk[i][j]; }
    };
    if (t0 + K > TmD) down_rows(std::true_type{});
    else down_rows(std::false_type{});
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&p.tm_out0, so0, (int)bw, t0, 0);
      if (!BWD) tma_store_3d(&p.tm_out1, so1, (int)bw, t0, 0);
      if (BWD && PD) tma_store_2d(&p.tm_out1, so1, (int)bw, t0);
      bulk_commit();
      if (it + ST < ntiles) {
        fence_proxy_async_smem();
        issue_tile_irr<D, IO, PD, BWD>(p, ring + s * L::STAGE, &bars[s], it + ST, C, (int)bw);
      }
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait0();
  if (BWD && !PD && valid) reinterpret_cast<IO*>(p.out1)[b] = from_f64<IO>(lam_acc);
}

// ------------------------------------------------------------------ posterior variance (NEXT-4)
// diag(Omega^{-1}) by Takahashi's selected inversion on the same deviation-form
// factor (R-15).  With Sigma = Omega^{-1} = L^{-T} D^{-1} L^{-1}, rows descending:
//   Sigma[t][t+l] = -sum_{k=1..d} L[t+k][t] Sigma[t+k][t+l]        (l = 1..d)
//   Sigma[t][t]   = 1/D_t - sum_{k=1..d} L[t+k][t] Sigma[t][t+k]
// needs only the d x d window of Sigma below-right of row t; L[t+k][t] = M_k + A[t+k][k].
// Up sweep: factor + checkpoints (no right-hand side); down sweep: recompute the
// chunk's factor, run the recurrence, stage Sigma[t][t] and TMA-store it.
template <int D, typename IO, bool PD>
struct VarLayout {
  using L = Layout<D, IO, PD, false>;
  static constexpr int K = L::K, ST = L::ST, ROW = L::ROW;
  static constexpr int OFF_W = 0;
  static constexpr int OFF_LAM = K * ROW;
  static constexpr int STAGE = (OFF_LAM + (PD ? (K + D) * ROW : 0) + 127) / 128 * 128;
  static constexpr int OUT = K * ROW;
  static constexpr int WARP_SMEM = ST * STAGE + OUT;
  static constexpr int WARPS = 4;
  static constexpr int SMEM = WARPS * WARP_SMEM;
  static constexpr uint32_t BYTES_UP = (K + (PD ? K : 0)) * ROW;
  static constexpr uint32_t BYTES_DN = (K + (PD ? K + D : 0)) * ROW;
};

template <int D, typename IO, bool PD>
__device__ __forceinline__ void issue_tile_var(const Params& p, unsigned char* stage, uint64_t* bar, int i, int C,
                                               int c0) {
  using V = VarLayout<D, IO, PD>;
  const bool up = i < C;
  const int c = up ? i : 2 * C - 1 - i;
  const int t0 = c * V::K;
  mbar_arrive_expect_tx(bar, up ? V::BYTES_UP : V::BYTES_DN);
  tma_load_2d(stage + V::OFF_W, &p.tm_w, c0, t0, bar);
  if (PD) {
    if (up) tma_load_2d(stage + V::OFF_LAM, &p.tm_lam_up, c0, t0, bar);
    else tma_load_2d(stage + V::OFF_LAM, &p.tm_lam_dn, c0, t0 - D, bar);
  }
}

template <int D, typename IO, bool PD>
__global__ void __maxnreg__(168) whit_var_kernel(const __grid_constant__ Params p) {
  using V = VarLayout<D, IO, PD>;
  constexpr int K = V::K, ST = V::ST, WARPS = V::WARPS;
  constexpr int NFAC = Ck<D>::NFAC;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[WARPS][ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = p.T, C = p.C, TmD = T - D;
  const long long B = p.B;
  const long long bw = ((long long)blockIdx.x * WARPS + warp) * 32;
  if (bw >= B) return;
  const long long b = bw + lane;
  const bool valid = b < B;
  unsigned char* ring = smem + warp * V::WARP_SMEM;
  IO* so = reinterpret_cast<IO*>(ring + ST * V::STAGE);
  uint64_t* bars = full_bar[warp];
  const int ntiles = 2 * C;
  if (lane == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < ST && i < ntiles; ++i) issue_tile_var<D, IO, PD>(p, ring + i * V::STAGE, &bars[i], i, C, (int)bw);
  }
  __syncwarp();
  const double lam_s = (!PD && valid) ? to_f64<IO>(reinterpret_cast<const IO*>(p.lam_scalar)[b]) : 0.0;

  FState<D> st;
  state_init<D>(st);
  int nobs = 0, bad = 0;  // bad: 1-based first failing pivot row
  int it = 0;
  // ---------------------------------------------------------------- up sweep: factor only
  for (int c = 0; c < C; ++c, ++it) {
    const int s = it % ST;
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * V::STAGE;
    const IO* t_w = reinterpret_cast<const IO*>(stg + V::OFF_W) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + V::OFF_LAM) + lane;
    const int t0 = c * K;
    if (valid) {
      double* ck = p.ck_fac + (long long)c * NFAC * B + b;
      int f = 0;
#pragma unroll
      for (int i = 0; i < D; ++i) ck[(long long)(f++) * B] = st.dl[i];
#pragma unroll
      for (int m = 0; m < D - 1; ++m)
#pragma unroll
        for (int k = 0; k < D - 1 - m; ++k) ck[(long long)(f++) * B] = st.ap[m][k];
    }
    auto up_rows = [&](auto edge_tag) {  // EDGE: the chunk touches rows >= T - d
      constexpr bool EDGE = decltype(edge_tag)::value;
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        const int t = t0 + k;
        if (EDGE && t >= T) break;
        const IO wio = t_w[k * 32];
        const double w = to_f64<IO>(wio);
        const double lt = PD ? to_f64<IO>(t_lam[k * 32]) : ((!EDGE || t < TmD) ? lam_s : 0.0);
        double A[D], Dt, idt, vt;
        ldl_step<D, Newton<IO, D>::N>(st, w, lt, 0.0, A, Dt, idt, vt);
        nobs += (wio > IO(0));
        if (bad == 0 && !pivot_ok(Dt)) bad = t + 1;
      }
    };
    if (t0 + K > TmD) up_rows(std::true_type{});
    else up_rows(std::false_type{});
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue_tile_var<D, IO, PD>(p, ring + s * V::STAGE, &bars[s], it + ST, C, (int)bw);
    }
  }
  const int info = status_info(bad, nobs, D, T);
  if (valid) p.info[b] = info;
  const bool failed = info != 0;
  const double poison = failed ? qnan() : 0.0;

  // ---------------------------------------------------------------- down sweep: Takahashi
  double cA[D][D];
  double S[D][D];  // S[k][l] = Sigma[t+1+k][t+1+l], rows t+1..t+D
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) { cA[i][j] = 0.0; S[i][j] = poison; }
  double pck[NFAC];  // the next chunk's factor checkpoint, loaded one chunk ahead
  auto load_ck = [&](int cc) {
    const double* ckf = p.ck_fac + (long long)cc * NFAC * B + b;
#pragma unroll
    for (int f = 0; f < NFAC; ++f) pck[f] = ld_pred_f64(ckf + (long long)f * B, valid);
  };
  load_ck(C - 1);
  for (int c = C - 1; c >= 0; --c, ++it) {
    const int s = it % ST;
    {
      int f = 0;
#pragma unroll
      for (int i = 0; i < D; ++i) st.dl[i] = pck[f++];
#pragma unroll
      for (int m = 0; m < D - 1; ++m)
#pragma unroll
        for (int k = 0; k < D - 1 - m; ++k) st.ap[m][k] = pck[f++];
    }
    if (c > 0) load_ck(c - 1);
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * V::STAGE;
    const IO* t_w = reinterpret_cast<const IO*>(stg + V::OFF_W) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + V::OFF_LAM) + lane;  // row k <-> t0 - D + k
    const int t0 = c * K;
    const bool ragged = (t0 + K > T), edge = (t0 + K > TmD);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int tj = t0 - 1 - i;
      st.v[i] = 0.0;
      const double l = PD ? to_f64<IO>(t_lam[(D - 1 - i) * 32]) : ((tj >= 0 && tj < TmD) ? lam_s : 0.0);
      st.lm[i] = l;
      st.id[i] = (tj < 0) ? 1.0 : rcp64<Newton<IO, D>::N>(l + st.dl[i]);
    }
    double idk[K];
    double Ak[K][D];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int t = t0 + k;
      const double w = to_f64<IO>(t_w[k * 32]);
      double lt = PD ? to_f64<IO>(t_lam[(k + D) * 32]) : lam_s;
      if (!PD) lt = (!edge || t < TmD) ? lt : 0.0;
      double Dt, vt;
      ldl_step<D, Newton<IO, D>::N>(st, w, lt, 0.0, Ak[k], Dt, idk[k], vt);
      if (ragged && t >= T) {  // rows past the end: Sigma = 0 there, no coupling
        idk[k] = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) Ak[k][j] = 0.0;
      }
    }
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      double Lc[D];  // L[t+j][t] - M_j = A[t+j][j]
#pragma unroll
      for (int j = 1; j <= D; ++j) Lc[j - 1] = (k + j < K) ? Ak[k + j][j - 1] : cA[k + j - K][j - 1];
      double up[D];  // Sigma[t][t+l], l = 1..D
#pragma unroll
      for (int l = 1; l <= D; ++l) {
        double acc = 0.0;
#pragma unroll
        for (int j = D; j >= 1; --j) {
          const double sjl = (j <= l) ? S[j - 1][l - 1] : S[l - 1][j - 1];
          acc = fma(-Mj(D, j), sjl, acc);
          acc = fma(-Lc[j - 1], sjl, acc);
        }
        up[l - 1] = acc;
      }
      double dg = idk[k];
#pragma unroll
      for (int j = D; j >= 1; --j) {
        dg = fma(-Mj(D, j), up[j - 1], dg);
        dg = fma(-Lc[j - 1], up[j - 1], dg);
      }
      // shift the window: new row t becomes index 0
#pragma unroll
      for (int i = D - 1; i >= 1; --i)
#pragma unroll
        for (int j = D - 1; j >= i; --j) S[i][j] = S[i - 1][j - 1];
      S[0][0] = dg;
#pragma unroll
      for (int l = 1; l < D; ++l) S[0][l] = up[l - 1];
      so[k * 32 + lane] = from_f64<IO>(dg);
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) cA[i][j] = Ak[i][j];
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&p.tm_out0, so, (int)bw, t0, 0);
      bulk_commit();
      if (it + ST < ntiles) {
        fence_proxy_async_smem();
        issue_tile_var<D, IO, PD>(p, ring + s * V::STAGE, &bars[s], it + ST, C, (int)bw);
      }
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait0();
}

// Bit-pack a 0/1 weight plane: word r of series b holds w[32r + j][b] != 0 in bit j (0 past T).
template <typename IO>
__global__ void pack_mask(const IO* __restrict__ w, long long T, long long B, uint32_t* __restrict__ bits) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long r = blockIdx.y;
  if (b >= B) return;
  uint32_t word = 0;
  const long long t0 = r * 32;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) {
    const long long t = t0 + j;
    if (t < T && w[t * B + b] != IO(0)) word |= 1u << j;
  }
  bits[r * B + b] = word;
}

// dL/dw (NEXT-3 option): gw[t][b] = sum_c u_{c,t} (y_{c,t} - z_{c,t}) with u = grad_y / w (grad_y = W u,
// Eq. (5)), 0 where w_t = 0 (reading R-19), NaN for a failed series.  Differences and products in
// fp64; the band sum in band order.  One thread per (t, b); a block covers 256 series of rows
// blockIdx.y, blockIdx.y + gridDim.y, ...
template <typename IO>
__global__ void grad_w_kernel(const IO* __restrict__ w, const IO* __restrict__ y, const IO* __restrict__ z,
                              const IO* __restrict__ gy, const int32_t* __restrict__ info, IO* __restrict__ gw,
                              long long T, long long B, int nb) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= B) return;
  const bool failed = info[b] != 0;
  const long long plane = T * B;
  for (long long t = blockIdx.y; t < T; t += gridDim.y) {
    const long long i = t * B + b;
    const IO wt = w[i];
    double acc = 0.0;
    if (wt != IO(0)) {
      const double wd = to_f64<IO>(wt);
      for (int c = 0; c < nb; ++c) {
        const long long j = c * plane + i;
        acc = fma(to_f64<IO>(gy[j]) / wd, to_f64<IO>(y[j]) - to_f64<IO>(z[j]), acc);
      }
    }
    gw[i] = from_f64<IO>(failed ? qnan() : acc);
  }
}

// Count of failed series (info != 0) for whit_failures.
static __global__ void count_failures(const int32_t* __restrict__ info, long long B, unsigned long long* out) {
  unsigned long long n = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < B; i += (long long)gridDim.x * blockDim.x)
    n += (info[i] != 0);
  for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(out, n);
}

}  // namespace whit
