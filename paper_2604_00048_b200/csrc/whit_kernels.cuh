// libwhit device code: fused assemble + banded LDL^T + substitutions for
// (W + D^T diag(lambda) D) z = W y   (Eq. (3); Omega)
// and its adjoint (Eq. (4)-(5)), one series per thread, fp64 math.
//
// Design:
//  * layout [T][B]: one time row of a CTA's NT series is NT contiguous
//    elements; a TMA 2-D box {NT series x K steps} stages a time tile of each
//    input plane into a shared-memory ring fed by one producer warp;
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
struct Params {
  CUtensorMap tm_rhs;     // y (forward) or grad_z (backward): [T][B], box {NT, K}
  CUtensorMap tm_w;       // w: [T][B], box {NT, K}
  CUtensorMap tm_lam_up;  // per-date lambda [T-d][B], box {NT, K}
  CUtensorMap tm_lam_dn;  // per-date lambda [T-d][B], box {NT, K+d} (rows t0-d..t0+K-1)
  CUtensorMap tm_dz;      // D z cache [T-d][B], box {NT, K} (backward only)
  const void* lam_scalar; // [B] (scalar lambda mode)
  void* out0;             // forward: z [T][B]; backward: grad_y [T][B]
  void* out1;             // forward: D z [T-d][B] (ws); backward: grad_lambda
  double* ck_f;           // forward checkpoints [C][NF][B]  (factor + rhs state)
  double* ck_b;           // backward checkpoints [C][d][B]  (rhs state)
  int32_t* info;          // [B]
  long long B;
  int T;
  int C;                  // number of K-step chunks = ceil(T / K)
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
// Bounded wait: a pipeline bug traps (a CUDA error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > 20000000000LL) __trap();  // ~10 s at 2 GHz
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// fp64 reciprocal: MUFU.RCP64H seed + 2 Newton steps (error ~1 ulp).  Used
// identically by every sweep so recomputed factors are bitwise identical.
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  return r;
}

template <typename IO> __device__ __forceinline__ double to_f64(IO v) { return static_cast<double>(v); }
template <typename IO> __device__ __forceinline__ IO from_f64(double v) { return static_cast<IO>(v); }

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
//   E_m  = -sum_{j=m+1..D} ( M_j lam~[t-j] A[t-m][j-m] + E_j (M_{j-m} + A[t-m][j-m]) ),  m = D..1
//   A_m  = ( E_m - M_m Delta[t-m] ) / D[t-m]                 (L[t][t-m] = M_m + A_m)
//   Delta_t = w_t - sum_j ( M_j E_j + A_j (M_j lam~[t-j] + E_j) )
//   D_t  = lam~_t + Delta_t                                   (SPD <=> D_t > 0 for all t)
//   v_t  = b_t - sum_j M_j v[t-j] - sum_j A_j v[t-j]
// Outputs A[0..D-1] (= A_{t,1..D}), D_t, 1/D_t, v_t; advances the state.
template <int D>
__device__ __forceinline__ void ldl_step(FState<D>& s, double w, double lam_t, double b, double (&A)[D],
                                         double& Dt, double& idt, double& vt) {
  double E[D + 1];
#pragma unroll
  for (int m = D; m >= 1; --m) {
    double e = 0.0;
#pragma unroll
    for (int j = m + 1; j <= D; ++j) {
      const double a = s.ap[m - 1][j - m - 1];
      e = fma(-(Mj(D, j) * s.lm[j - 1]), a, e);
      e = fma(-E[j], a, e);
      e = fma(-Mj(D, j - m), E[j], e);
    }
    E[m] = e;
    const double num = (m == D) ? (-Mj(D, m) * s.dl[m - 1]) : fma(-Mj(D, m), s.dl[m - 1], e);
    A[m - 1] = num * s.id[m - 1];
  }
  double dl = w;
#pragma unroll
  for (int j = 1; j <= D; ++j) {
    if (j < D) dl = fma(-Mj(D, j), E[j], dl);
    const double inner = (j < D) ? fma(Mj(D, j), s.lm[j - 1], E[j]) : Mj(D, j) * s.lm[j - 1];
    dl = fma(-A[j - 1], inner, dl);
  }
  Dt = lam_t + dl;
  idt = rcp64(Dt);
  double v = b;
#pragma unroll
  for (int j = 1; j <= D; ++j) {
    v = fma(-Mj(D, j), s.v[j - 1], v);
    v = fma(-A[j - 1], s.v[j - 1], v);
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

// Checkpoint field counts: factor part = D (Delta) + D(D-1)/2 (A), rhs part = D (v).
template <int D> struct Ck {
  static constexpr int NFAC = D + D * (D - 1) / 2;
  static constexpr int NF = NFAC + D;  // forward checkpoint fields
};

// ------------------------------------------------------------------ tiling config
// NT series per CTA (one per consumer thread), K time steps per chunk/tile,
// ST ring stages.  K = 16 for d <= 2; d = 3 keeps 4 fp64 values per chunk row
// in registers, so its chunk is 8 steps.  MAXREG keeps 2 CTAs (10 warps)/SM.
template <typename IO, int D> struct Tile {
  static constexpr int NT = sizeof(IO) == 4 ? 128 : 64;
  static constexpr int K = D <= 2 ? 16 : 8;
  static constexpr int ST = 3;
  static constexpr int MAXREG = sizeof(IO) == 4 ? 200 : 255;
};

template <int D, typename IO, bool PD, bool BWD> struct Layout {
  static constexpr int NT = Tile<IO, D>::NT, K = Tile<IO, D>::K, ST = Tile<IO, D>::ST;
  static constexpr int ROW = NT * (int)sizeof(IO);  // bytes of one staged time row
  static constexpr int OFF_RHS = 0;
  static constexpr int OFF_W = K * ROW;
  static constexpr int OFF_LAM = 2 * K * ROW;
  static constexpr int OFF_DZ = OFF_LAM + (PD ? (K + D) * ROW : 0);
  static constexpr int STAGE = OFF_DZ + (BWD ? K * ROW : 0);
  static constexpr int SMEM = ST * STAGE;
  static constexpr uint32_t BYTES_UP = (2 * K + (PD ? K : 0)) * ROW;
  static constexpr uint32_t BYTES_DN = (2 * K + (PD ? K + D : 0) + (BWD ? K : 0)) * ROW;
};

// ------------------------------------------------------------------ the kernel
// One launch = one full forward (BWD=false) or backward (BWD=true) for NT
// series per CTA: up sweep over C chunks, then down sweep over C chunks.
template <int D, typename IO, bool PD, bool BWD>
__global__ void __maxnreg__((Tile<IO, D>::MAXREG)) whit_kernel(const __grid_constant__ Params p) {
  using L = Layout<D, IO, PD, BWD>;
  constexpr int NT = L::NT, K = L::K, ST = L::ST;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[ST];
  __shared__ __align__(8) uint64_t empty_bar[ST];

  const int tid = threadIdx.x;
  const int T = p.T, C = p.C;
  const long long B = p.B;
  const long long b0 = (long long)blockIdx.x * NT;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer warp
  if (tid >= NT) {
    if (tid == NT) {
      prefetch_map(&p.tm_rhs);
      prefetch_map(&p.tm_w);
      if (PD) { prefetch_map(&p.tm_lam_up); prefetch_map(&p.tm_lam_dn); }
      if (BWD) prefetch_map(&p.tm_dz);
      for (int i = 0; i < 2 * C; ++i) {
        const int s = i % ST;
        const uint32_t ph = (uint32_t)((i / ST) & 1);
        mbar_wait(&empty_bar[s], ph ^ 1u);
        const bool up = i < C;
        const int c = up ? i : 2 * C - 1 - i;
        const int t0 = c * K;
        unsigned char* st = smem + s * L::STAGE;
        mbar_arrive_expect_tx(&full_bar[s], up ? L::BYTES_UP : L::BYTES_DN);
        tma_load_2d(st + L::OFF_RHS, &p.tm_rhs, (int)b0, t0, &full_bar[s]);
        tma_load_2d(st + L::OFF_W, &p.tm_w, (int)b0, t0, &full_bar[s]);
        if (PD) {
          if (up) tma_load_2d(st + L::OFF_LAM, &p.tm_lam_up, (int)b0, t0, &full_bar[s]);
          else tma_load_2d(st + L::OFF_LAM, &p.tm_lam_dn, (int)b0, t0 - D, &full_bar[s]);
        }
        if (BWD && !up) tma_load_2d(st + L::OFF_DZ, &p.tm_dz, (int)b0, t0, &full_bar[s]);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers: one series each
  const long long b = b0 + tid;
  const bool valid = b < B;
  const int lane_leader = (tid & 31) == 0;
  const double lam_s = (!PD && valid) ? to_f64<IO>(reinterpret_cast<const IO*>(p.lam_scalar)[b]) : 0.0;
  const int TmD = T - D;
  constexpr int NF = Ck<D>::NF, NFAC = Ck<D>::NFAC;

  FState<D> st;
  state_init<D>(st);
  int nobs = 0, bad = 0;
  int it = 0;  // tile sequence index (ring position)

  // ================================================================ up sweep
  for (int c = 0; c < C; ++c, ++it) {
    const int s = it % ST;
    mbar_wait(&full_bar[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = smem + s * L::STAGE;
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + tid;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + tid;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + tid;
    const int t0 = c * K;
    // checkpoint: state entering row t0
    if (valid) {
      if (!BWD) {
        double* ck = p.ck_f + (long long)c * NF * B + b;
        int f = 0;
#pragma unroll
        for (int i = 0; i < D; ++i) ck[(long long)(f++) * B] = st.dl[i];
#pragma unroll
        for (int m = 0; m < D - 1; ++m)
#pragma unroll
          for (int k = 0; k < D - 1 - m; ++k) ck[(long long)(f++) * B] = st.ap[m][k];
#pragma unroll
        for (int i = 0; i < D; ++i) ck[(long long)(f++) * B] = st.v[i];
      } else {
        double* ck = p.ck_b + (long long)c * D * B + b;
#pragma unroll
        for (int i = 0; i < D; ++i) ck[(long long)i * B] = st.v[i];
      }
    }
    const int n = min(K, T - t0);
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
      const int t = t0 + k;
      const double rhs = to_f64<IO>(t_rhs[k * NT]);
      const double w = to_f64<IO>(t_w[k * NT]);
      const double lt = PD ? to_f64<IO>(t_lam[k * NT]) : (t < TmD ? lam_s : 0.0);
      const double bb = BWD ? rhs : (w != 0.0 ? w * rhs : 0.0);
      double A[D], Dt, idt, vt;
      ldl_step<D>(st, w, lt, bb, A, Dt, idt, vt);
      if (!BWD) {
        nobs += (w > 0.0);
        if (bad == 0 && !(Dt > 0.0)) bad = t + 1;  // also catches NaN
      }
    }
    __syncwarp();
    if (lane_leader) mbar_arrive(&empty_bar[s]);
  }

  bool failed;
  if (!BWD) {
    const int info = (nobs < D) ? (T - D + 1) : bad;
    if (valid) p.info[b] = info;
    failed = info != 0;
  } else {
    failed = valid ? (p.info[b] != 0) : true;
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);

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

  // checkpoint prefetch registers
  double pdl[D], pap[NFAC - D > 0 ? NFAC - D : 1], pv[D];
  auto load_ck = [&](int c) {
    if (!valid) return;
    const double* ckf = p.ck_f + (long long)c * NF * B + b;
#pragma unroll
    for (int i = 0; i < D; ++i) pdl[i] = ckf[(long long)i * B];
#pragma unroll
    for (int f = 0; f < NFAC - D; ++f) pap[f] = ckf[(long long)(D + f) * B];
    if (!BWD) {
#pragma unroll
      for (int i = 0; i < D; ++i) pv[i] = ckf[(long long)(NFAC + i) * B];
    } else {
      const double* ckb = p.ck_b + (long long)c * D * B + b;
#pragma unroll
      for (int i = 0; i < D; ++i) pv[i] = ckb[(long long)i * B];
    }
  };
  load_ck(C - 1);

  IO* out0 = reinterpret_cast<IO*>(p.out0);
  IO* out1 = reinterpret_cast<IO*>(p.out1);

  for (int c = C - 1; c >= 0; --c, ++it) {
    const int s = it % ST;
    mbar_wait(&full_bar[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = smem + s * L::STAGE;
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + tid;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + tid;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + tid;  // row k <-> t0 - D + k
    const IO* t_dz = reinterpret_cast<const IO*>(stg + L::OFF_DZ) + tid;
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
        st.v[i] = pv[i];
        const double l = PD ? to_f64<IO>(t_lam[(D - 1 - i) * NT]) : ((tj >= 0 && tj < TmD) ? lam_s : 0.0);
        st.lm[i] = l;
        st.id[i] = (tj < 0) ? 1.0 : rcp64(l + pdl[i]);
      }
    }
    if (c > 0) load_ck(c - 1);

    // recompute the chunk's factor into registers
    double q[K];
    double Ak[K][D];
    const bool ragged = (t0 + K > T);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int t = t0 + k;
      if (ragged && t >= T) {
        q[k] = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) Ak[k][j] = 0.0;
        continue;
      }
      const double rhs = to_f64<IO>(t_rhs[k * NT]);
      const double w = to_f64<IO>(t_w[k * NT]);
      const double lt = PD ? to_f64<IO>(t_lam[(k + D) * NT]) : (t < TmD ? lam_s : 0.0);
      const double bb = BWD ? rhs : (w != 0.0 ? w * rhs : 0.0);
      double Dt, idt, vt;
      ldl_step<D>(st, w, lt, bb, Ak[k], Dt, idt, vt);
      q[k] = vt * idt;
    }

    // back substitution over the chunk, descending
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      const int t = t0 + k;
      if (ragged && t >= T) continue;
      double z = q[k];
#pragma unroll
      for (int j = 1; j <= D; ++j) {
        const double a = (k + j < K) ? Ak[k + j][j - 1] : cA[k + j - K][j - 1];
        z = fma(-Mj(D, j), zw[j - 1], z);
        z = fma(-a, zw[j - 1], z);
      }
      // (D z)_t = sum_j c_j z[t+j]  (rows t <= T-d-1)
      double dz = Cj(D, 0) * z;
#pragma unroll
      for (int j = 1; j <= D; ++j) dz = fma(Cj(D, j), zw[j - 1], dz);
#pragma unroll
      for (int i = D - 1; i >= 1; --i) zw[i] = zw[i - 1];
      zw[0] = z;
      if (valid) {
        const long long idx = (long long)t * B + b;
        if (!BWD) {
          out0[idx] = from_f64<IO>(failed ? qnan : z);
          if (t < TmD) out1[idx] = from_f64<IO>(failed ? qnan : dz);
        } else {
          const double w = to_f64<IO>(t_w[k * NT]);
          out0[idx] = from_f64<IO>(failed ? qnan : w * z);
          if (t < TmD) {
            const double g = -dz * to_f64<IO>(t_dz[k * NT]);
            if (PD) out1[idx] = from_f64<IO>(failed ? qnan : g);
            else lam_acc += g;
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) cA[i][j] = Ak[i][j];

    __syncwarp();
    if (lane_leader) mbar_arrive(&empty_bar[s]);
  }
  if (BWD && !PD && valid) out1[b] = from_f64<IO>(failed ? qnan : lam_acc);
}

// Count of failed series (info != 0) for whit_failures.
__global__ void count_failures(const int32_t* __restrict__ info, long long B, unsigned long long* out) {
  unsigned long long n = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < B; i += (long long)gridDim.x * blockDim.x)
    n += (info[i] != 0);
  for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(out, n);
}

}  // namespace whit
