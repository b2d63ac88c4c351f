// libwhit multi-band kernel with a shared factor warp (NEXT-1, P:28 / P:147: the C bands of a
// pixel share W and Lambda, hence Omega and its factor).
//
// CTA = ceil(C/2) band warps (two bands each) + 1 factor warp over 32 pixels, K = 8-row chunks:
//  * the factor warp streams w and lambda (and, IRR, the acquisition dates) through its own TMA ring
//    (4 slots in the forward, 2 in the backward), runs the deviation-form LDL^T (ldl_step, R-10; IRR:
//    ldl_step_irr on the per-row dspline stencils, R-18) once per pixel and publishes, per chunk, the
//    rows (A_{t,1..d}, 1/D_t, w_t; IRR also mu and c_{t,0}) into a ring of 3 shared-memory factor buffers
//    (mbarriers fac_full / fac_empty); it writes the factor checkpoints and, in the down sweep,
//    recomputes each chunk's factor from them (loaded a chunk ahead);
//  * each band warp streams its two bands' right-hand sides (TMA) and runs the forward-substitution
//    recurrences and the back substitutions with the published rows (two independent chains per lane =
//    ILP), storing z / D z / grad_y straight to HBM with coalesced 128-B warp stores (no staging),
//    reading D z in the backward with plain loads issued a chunk ahead of use; per-date dL/dlambda
//    partials are summed across the band warps through shared memory (one barrier per chunk).
//  * interior chunks run without per-row range checks (compile-time interior / edge split).
// Shared memory per CTA (~54-67 KB at C = 10, fp32) and <= 168 registers give two CTAs -- two
// independent pixel groups and factor chains -- per SM at C = 10, four at C <= 4.
// The band warps execute exactly the fp64 operation sequence of the single-band kernels, so every
// band's z and grad_y equal the independent-series results bit for bit; grad_lambda is the band sum
// in fp64 (fixed order).
#pragma once
#include <type_traits>
#include "whit_kernels.cuh"

namespace whit {

template <int D, typename IO, bool PD, bool BWD, bool IRR = false>
struct MB2Layout {
#ifndef WHIT_MB2_K
#define WHIT_MB2_K 8
#endif
#ifndef WHIT_MB2_ST
#define WHIT_MB2_ST 2
#endif
  // rows per chunk; TMA ring slots (ST - 1 chunks of loads in flight per warp); bands per band warp
#ifndef WHIT_MB2_BPW
#define WHIT_MB2_BPW 2
#endif
  static constexpr int K = WHIT_MB2_K, ST = WHIT_MB2_ST, BPW = WHIT_MB2_BPW;
  // factor-warp ring slots: the factor warp's per-chunk work is short (K rows of the recurrence), so
  // in the forward its w / lambda (/ dates) loads are issued 3 chunks ahead to cover the HBM latency
  // (measured: forward faster, backward not -- its smem goes to the reduction rows)
  static constexpr int FST = BWD ? 2 : 4;
  static constexpr int ROW = 32 * (int)sizeof(IO);
  // factor warp ring: w K rows | lambda K (+d) rows | IRR: acquisition dates K+2d rows (t0-d .. t0+K+d-1)
  static constexpr int F_OFF_W = 0, F_OFF_LAM = K * ROW;
  static constexpr int F_OFF_TT = F_OFF_LAM + (PD ? (K + D) * ROW : 0);
  static constexpr int F_STAGE = (F_OFF_TT + (IRR ? (K + 2 * D) * ROW : 0) + 127) / 128 * 128;
  // band warp ring stage: rhs K rows for each of its bands
  static constexpr int B_STAGE = BPW * K * ROW;
  static constexpr int B_WARP = ST * B_STAGE;
  // factor buffer, lane-contiguous fp64 rows: A[k][0..d-1], 1/D[k]; IRR also the normalised stencils
  // mu of rows t0-d .. t0+K-1 ([K+d][d], R-18) and c_{t,0} [K]; then w[k] (IO)
  static constexpr int FB_A = 0, FB_ID = D * K * 32 * 8;
  static constexpr int FB_MU = FB_ID + K * 32 * 8;
  static constexpr int FB_C0 = FB_MU + (IRR ? (K + D) * D * 32 * 8 : 0);
  static constexpr int FB_W = FB_C0 + (IRR ? K * 32 * 8 : 0);
  static constexpr int FBUF = (FB_W + K * 32 * (int)sizeof(IO) + 127) / 128 * 128;
  static constexpr uint32_t F_BYTES_UP = (K + (PD ? K : 0) + (IRR ? K + 2 * D : 0)) * ROW;
  static constexpr uint32_t F_BYTES_DN = (K + (PD ? K + D : 0) + (IRR ? K + 2 * D : 0)) * ROW;
  // smem: factor ring | factor buffers | band warps | per-warp reduction rows (fp64) + scalars
  static constexpr int OFF_FB = FST * F_STAGE;
  // factor buffers in flight: enough that the factor warp runs ahead of the band warps' jitter
  static constexpr int NFB = (BWD && !PD) ? 4 : 3;
  static constexpr int OFF_BAND = OFF_FB + NFB * FBUF;
  __host__ __device__ static constexpr int nwarps(int nb) { return (nb + BPW - 1) / BPW; }
#ifndef WHIT_MB2_RED2
#define WHIT_MB2_RED2 1
#endif
  // per-date dL/dlambda partials: slots of [nw][K][32] fp64; RED2: four slots, one barrier per two chunks
  static constexpr int RSLOTS = WHIT_MB2_RED2 ? 4 : 2;
  static constexpr int smem(int nb) {
    return OFF_BAND + nwarps(nb) * B_WARP + (BWD && PD ? RSLOTS * nwarps(nb) * K * 32 * 8 : 0) +
           (BWD && !PD ? nwarps(nb) * 32 * 8 : 0);
  }
};

#ifndef WHIT_MB2_MAXREG_D3
#define WHIT_MB2_MAXREG_D3 168
#endif
#ifndef WHIT_MB2_MAXREG
#define WHIT_MB2_MAXREG 168
#endif
template <int D, typename IO, bool PD, bool BWD, bool IRR = false>
__global__ void __maxnreg__((D == 3 ? WHIT_MB2_MAXREG_D3 : WHIT_MB2_MAXREG)) whit_mb2_kernel(const __grid_constant__ Params p) {
  using L = MB2Layout<D, IO, PD, BWD, IRR>;
#ifndef WHIT_MB2_IRR_FUNROLL
#define WHIT_MB2_IRR_FUNROLL 2
#endif
  // factor-warp row loops: the irregular grid's per-row stencil makes them long (instruction cache)
  constexpr int FROW_UNROLL = IRR ? WHIT_MB2_IRR_FUNROLL : 8;
#ifndef WHIT_MB2_IRR_BUNROLL
#define WHIT_MB2_IRR_BUNROLL 8
#endif
  constexpr int BROW_UNROLL = IRR ? WHIT_MB2_IRR_BUNROLL : 8;  // band warps' up-sweep rows
  constexpr int K = L::K, ST = L::ST, FST = L::FST, NFAC = Ck<D>::NFAC, NW = Newton<IO, D>::N, BPW = L::BPW;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t f_full[FST];
  __shared__ __align__(8) uint64_t b_full[(kMaxBands + 1) / 2][ST];
  __shared__ __align__(8) uint64_t fac_full[L::NFB], fac_empty[L::NFB];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = p.nb, nw = L::nwarps(nb), T = p.T, C = p.C, TmD = T - D;
  const long long B = p.B;
  const long long bw = (long long)blockIdx.x * 32;
  if (bw >= B) return;  // whole CTA
  const long long b = bw + lane;
  const bool valid = b < B;
  const bool fwarp = warp == nw;  // the factor warp
  const int ntiles = 2 * C;
  unsigned char* fbuf0 = smem + L::OFF_FB;

  if (threadIdx.x == 0) {
    for (int i = 0; i < L::NFB; ++i) {
      mbar_init(&fac_full[i], 1);
      mbar_init(&fac_empty[i], nw);
    }
  }
  if (lane == 0) {
    if (fwarp) {
      for (int s = 0; s < FST; ++s) mbar_init(&f_full[s], 1);
    } else {
      for (int s = 0; s < ST; ++s) mbar_init(&b_full[warp][s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ============================================================== factor warp
  if (fwarp) {
    unsigned char* ring = smem;
    auto issue = [&](int i) {
      const bool up = i < C;
      const int c = up ? i : 2 * C - 1 - i;
      const int t0 = c * K;
      unsigned char* stg = ring + (i % FST) * L::F_STAGE;
      mbar_arrive_expect_tx(&f_full[i % FST], up ? L::F_BYTES_UP : L::F_BYTES_DN);
      tma_load_2d(stg + L::F_OFF_W, &p.tm_w, (int)bw, t0, &f_full[i % FST]);
      if (PD) {
        if (up) tma_load_2d(stg + L::F_OFF_LAM, &p.tm_lam_up, (int)bw, t0, &f_full[i % FST]);
        else tma_load_2d(stg + L::F_OFF_LAM, &p.tm_lam_dn, (int)bw, t0 - D, &f_full[i % FST]);
      }
      if (IRR) tma_load_2d(stg + L::F_OFF_TT, &p.tm_lw, (int)bw, t0 - D, &f_full[i % FST]);  // dates
    };
    if (lane == 0)
      for (int i = 0; i < FST && i < ntiles; ++i) issue(i);
    __syncwarp();
    const double lam_s = (!PD && valid) ? to_f64<IO>(reinterpret_cast<const IO*>(p.lam_scalar)[b]) : 0.0;
    IState<D> S;  // factor recurrence state (S.mu: stencils of the last d columns, IRR only)
    FState<D>& st = S.f;
    state_init<D>(st);
#pragma unroll
    for (int i = 0; i < D; ++i) binomial_col<D>(S.mu[i]);
    int nobs = 0, bad = 0;  // bad: 1-based first failing pivot row
    int it = 0, fb = 0;  // fb: factor-buffer sequence number
    // one factor row: daily grid (ldl_step, binomial stencil) or uneven dates (R-18: stencil of
    // column t from the dates tile, Lambda~_t = lambda_t c_{t,0}^2, ldl_step_irr)
    // edge: the chunk touches rows >= T - d (range checks needed); interior chunks skip them
    auto factor_row = [&](const IO* t_tt, int k, int t, double w, double lraw, double (&A)[D], double& Dt,
                          double& idt, double (&mu_t)[D], double& c0, bool edge) {
      double vt;
      if constexpr (IRR) {
        tile_col<D, IO, NW>(t_tt, k, t, T, mu_t, c0, edge);
        const double lt = (!edge || t < TmD) ? lraw * c0 * c0 : 0.0;
        ldl_step_irr<D, NW>(S, mu_t, w, lt, 0.0, A, Dt, idt, vt);
      } else {
        const double lt = (!edge || t < TmD) ? lraw : 0.0;
        ldl_step<D, NW>(st, w, lt, 0.0, A, Dt, idt, vt);
      }
    };
    // IRR: stencils of the d rows before the chunk (the band warps' recurrences reach back to them)
    auto publish_pre_mu = [&](double* FMU) {
      if constexpr (IRR) {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int j = 0; j < D; ++j) FMU[((D - 1 - i) * D + j) * 32] = S.mu[i][j];
      }
    };
    // ---- up sweep
    for (int c = 0; c < C; ++c, ++it, ++fb) {
      const int s = it % FST;
      mbar_wait(&f_full[s], (uint32_t)((it / FST) & 1));
      const unsigned char* stg = ring + s * L::F_STAGE;
      const IO* t_w = reinterpret_cast<const IO*>(stg + L::F_OFF_W) + lane;
      const IO* t_lam = reinterpret_cast<const IO*>(stg + L::F_OFF_LAM) + lane;
      const IO* t_tt = reinterpret_cast<const IO*>(stg + L::F_OFF_TT) + lane;
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
      mbar_wait(&fac_empty[fb % L::NFB], (uint32_t)(((fb / L::NFB) & 1) ^ 1));
      unsigned char* F = fbuf0 + (fb % L::NFB) * L::FBUF;
      double* FA = reinterpret_cast<double*>(F + L::FB_A) + lane;
      double* FMU = reinterpret_cast<double*>(F + L::FB_MU) + lane;
      IO* FW = reinterpret_cast<IO*>(F + L::FB_W) + lane;
      publish_pre_mu(FMU);
      auto up_rows = [&](auto edge_tag) {
        constexpr bool EDGE = decltype(edge_tag)::value;
#pragma unroll FROW_UNROLL
        for (int k = 0; k < K; ++k) {
          const int t = t0 + k;
          const IO wio = t_w[k * 32];
          const double w = to_f64<IO>(wio);
          const double lraw = PD ? to_f64<IO>(t_lam[k * 32]) : lam_s;
          double A[D], Dt, idt, mu_t[D], c0;
          factor_row(t_tt, k, t, w, lraw, A, Dt, idt, mu_t, c0, EDGE);
#pragma unroll
          for (int j = 0; j < D; ++j) FA[(k * D + j) * 32] = A[j];
          if constexpr (IRR) {
#pragma unroll
            for (int j = 0; j < D; ++j) FMU[((k + D) * D + j) * 32] = mu_t[j];
          }
          FW[k * 32] = wio;
          if (!BWD && (!EDGE || t < T)) {
            nobs += (wio > IO(0));
            if (bad == 0 && !pivot_ok(Dt)) bad = t + 1;
          }
        }
      };
      if (t0 + K > TmD) up_rows(std::true_type{});
      else up_rows(std::false_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(&fac_full[fb % L::NFB]);  // release: this warp's smem writes
      if (lane == 0 && it + FST < ntiles) {
        fence_proxy_async_smem();
        issue(it + FST);
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
    // ---- down sweep: recompute and publish each chunk's factor rows.  The factor checkpoint of
    // the next chunk is loaded one chunk ahead (its latency leaves the recurrence's chain).
    double ckn[NFAC];
    auto load_ck = [&](int c) {
      const double* ckf = p.ck_fac + (long long)c * NFAC * B + b;
#pragma unroll
      for (int f = 0; f < NFAC; ++f) ckn[f] = ld_pred_f64(ckf + (long long)f * B, valid);
    };
    load_ck(C - 1);
    for (int c = C - 1; c >= 0; --c, ++it, ++fb) {
      const int s = it % FST;
      {
        int f = 0;
#pragma unroll
        for (int i = 0; i < D; ++i) st.dl[i] = ckn[f++];
#pragma unroll
        for (int m = 0; m < D - 1; ++m)
#pragma unroll
          for (int k = 0; k < D - 1 - m; ++k) st.ap[m][k] = ckn[f++];
      }
      if (c > 0) load_ck(c - 1);
      mbar_wait(&f_full[s], (uint32_t)((it / FST) & 1));
      const unsigned char* stg = ring + s * L::F_STAGE;
      const IO* t_w = reinterpret_cast<const IO*>(stg + L::F_OFF_W) + lane;
      const IO* t_lam = reinterpret_cast<const IO*>(stg + L::F_OFF_LAM) + lane;  // row k <-> t0 - D + k
      const IO* t_tt = reinterpret_cast<const IO*>(stg + L::F_OFF_TT) + lane;
      const int t0 = c * K;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const int tj = t0 - 1 - i;
        st.v[i] = 0.0;
        const double lraw = PD ? to_f64<IO>(t_lam[(D - 1 - i) * 32]) : lam_s;
        double l;
        if constexpr (IRR) {
          double c0;
          tile_col<D, IO, NW>(t_tt, -1 - i, tj, T, S.mu[i], c0);
          l = (tj >= 0 && tj < TmD) ? lraw * c0 * c0 : 0.0;
        } else {
          l = PD ? lraw : ((tj >= 0 && tj < TmD) ? lam_s : 0.0);
        }
        st.lm[i] = l;
        st.id[i] = (tj < 0) ? 1.0 : rcp64<NW>(l + st.dl[i]);
      }
      mbar_wait(&fac_empty[fb % L::NFB], (uint32_t)(((fb / L::NFB) & 1) ^ 1));
      unsigned char* F = fbuf0 + (fb % L::NFB) * L::FBUF;
      double* FA = reinterpret_cast<double*>(F + L::FB_A) + lane;
      double* FI = reinterpret_cast<double*>(F + L::FB_ID) + lane;
      double* FMU = reinterpret_cast<double*>(F + L::FB_MU) + lane;
      double* FC0 = reinterpret_cast<double*>(F + L::FB_C0) + lane;
      IO* FW = reinterpret_cast<IO*>(F + L::FB_W) + lane;
      publish_pre_mu(FMU);
      auto down_rows = [&](auto edge_tag) {
        constexpr bool EDGE = decltype(edge_tag)::value;
#pragma unroll FROW_UNROLL
        for (int k = 0; k < K; ++k) {
          const int t = t0 + k;
          const IO wio = t_w[k * 32];
          const double w = to_f64<IO>(wio);
          const double lraw = PD ? to_f64<IO>(t_lam[(k + D) * 32]) : lam_s;
          double A[D], Dt, idt, mu_t[D], c0;
          factor_row(t_tt, k, t, w, lraw, A, Dt, idt, mu_t, c0, EDGE);
          const bool past = EDGE && t >= T;  // rows past the end: z = 0 (q = 0, A = 0)
#pragma unroll
          for (int j = 0; j < D; ++j) FA[(k * D + j) * 32] = past ? 0.0 : A[j];
          FI[k * 32] = past ? 0.0 : idt + poison;
          if constexpr (IRR) {
#pragma unroll
            for (int j = 0; j < D; ++j) FMU[((k + D) * D + j) * 32] = mu_t[j];
            FC0[k * 32] = c0;
          }
          FW[k * 32] = wio;
        }
      };
      if (t0 + K > TmD) down_rows(std::true_type{});
      else down_rows(std::false_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(&fac_full[fb % L::NFB]);
      if (lane == 0 && it + FST < ntiles) {
        fence_proxy_async_smem();
        issue(it + FST);
      }
    }
    if (BWD && !PD) __syncthreads();  // matches the band warps' scalar-lambda reduction
    return;
  }

  // ============================================================== band warps (two bands each)
  const int bj = warp;
  const int cb0 = bj * BPW;
  const int nbw = min(BPW, nb - cb0);  // bands of this warp (the last warp may hold fewer)
  unsigned char* ring = smem + L::OFF_BAND + bj * L::B_WARP;
  double* redw0 = reinterpret_cast<double*>(smem + L::OFF_BAND + nw * L::B_WARP);  // [2][nw][K][32] (PD bwd)
  double* redS = redw0 + (BWD && PD ? L::RSLOTS * nw * K * 32 : 0);                  // [nw][32]
  uint64_t* bars = b_full[bj];
  auto issue = [&](int i) {
    const bool up = i < C;
    const int c = up ? i : 2 * C - 1 - i;
    const int t0 = c * K;
    unsigned char* stg = ring + (i % ST) * L::B_STAGE;
    mbar_arrive_expect_tx(&bars[i % ST], nbw * K * L::ROW);
    for (int u = 0; u < nbw; ++u) tma_load_3d(stg + u * K * L::ROW, &p.tm_rhs, (int)bw, t0, cb0 + u, &bars[i % ST]);
  };
  if (lane == 0)
    for (int i = 0; i < ST && i < ntiles; ++i) issue(i);
  __syncwarp();
  double* const ck_rhs = (BWD ? p.ck_rhs_b : p.ck_rhs_f) + b;  // [c][nb][d][B]
  const long long ck_stride = (long long)nb * D * B;
  IO* const out0 = reinterpret_cast<IO*>(p.out0);  // z (fwd) / grad_y (bwd): [nb][T][B]
  IO* const out1 = reinterpret_cast<IO*>(p.out1);  // D z cache (fwd): [nb][T-d][B]; grad_lambda (bwd)
  const IO* const dzc = reinterpret_cast<const IO*>(p.dz_cache);  // bwd: [nb][T-d][B]
  double v[BPW][D];
#pragma unroll
  for (int u = 0; u < BPW; ++u)
#pragma unroll
    for (int i = 0; i < D; ++i) v[u][i] = 0.0;
  int it = 0, fb = 0;
  // ---- up sweep: v_t = b_t - sum_j (M_j + A_{t,j}) v_{t-j}, per band
  for (int c = 0; c < C; ++c, ++it, ++fb) {
    const int s = it % ST;
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const IO* t_rhs = reinterpret_cast<const IO*>(ring + s * L::B_STAGE) + lane;
    const int t0 = c * K;
    if (valid) {
#pragma unroll
      for (int u = 0; u < BPW; ++u) {
        if (u >= nbw) break;
        double* ck = ck_rhs + (long long)c * ck_stride + (long long)(cb0 + u) * D * B;
#pragma unroll
        for (int i = 0; i < D; ++i) ck[(long long)i * B] = v[u][i];
      }
    }
    mbar_wait(&fac_full[fb % L::NFB], (uint32_t)((fb / L::NFB) & 1));
    const unsigned char* F = fbuf0 + (fb % L::NFB) * L::FBUF;
    const double* FA = reinterpret_cast<const double*>(F + L::FB_A) + lane;
    const double* FMU = reinterpret_cast<const double*>(F + L::FB_MU) + lane;
    const IO* FW = reinterpret_cast<const IO*>(F + L::FB_W) + lane;
    auto up_rows = [&](auto tail_tag) {
      constexpr bool TAIL = decltype(tail_tag)::value;  // the chunk reaches row T: stop there
      const int n = T - t0;
#pragma unroll BROW_UNROLL
      for (int k = 0; k < K; ++k) {
        if (TAIL && k >= n) break;
        const IO wio = FW[k * 32];
        const double w = to_f64<IO>(wio);
#pragma unroll
        for (int u = 0; u < BPW; ++u) {
          double vv = rhs_times_w<IO, BWD>(t_rhs[(u * K + k) * 32], wio, w);
#pragma unroll
          for (int j = D; j >= 1; --j) {  // M~[t][t-j] = mu_{t-j}[j] (IRR), else M_j
            const double mj = IRR ? FMU[((k + D - j) * D + j - 1) * 32] : Mj(D, j);
            if (j > 1) {
              vv = fma(-mj, v[u][j - 1], vv);
              vv = fma(-FA[(k * D + j - 1) * 32], v[u][j - 1], vv);
            } else {  // (L = M + A first, as ldl_step)
              vv = fma(-(mj + FA[k * D * 32]), v[u][0], vv);
            }
          }
#pragma unroll
          for (int i = D - 1; i >= 1; --i) v[u][i] = v[u][i - 1];
          v[u][0] = vv;
        }
      }
    };
    if (t0 + K > T) up_rows(std::true_type{});
    else up_rows(std::false_type{});
    __syncwarp();
    if (lane == 0) mbar_arrive(&fac_empty[fb % L::NFB]);
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue(it + ST);
    }
  }
  // ---- down sweep
  double cA[D][D], zw[BPW][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) cA[i][j] = 0.0;
#pragma unroll
  for (int u = 0; u < BPW; ++u)
#pragma unroll
    for (int i = 0; i < D; ++i) zw[u][i] = 0.0;
  double lam_acc = 0.0;
  double vn[BPW][D];
  auto load_v = [&](int c) {
#pragma unroll
    for (int u = 0; u < BPW; ++u) {
      const double* ck = ck_rhs + (long long)c * ck_stride + (long long)(cb0 + u) * D * B;
      const bool ok = valid && u < nbw;
#pragma unroll
      for (int i = 0; i < D; ++i) vn[u][i] = ld_pred_f64(ck + (long long)i * B, ok);
    }
  };
  load_v(C - 1);
  // backward: D z rows of both bands, loaded one chunk ahead of the back substitution that uses them
  IO dzn[BPW][K];
  auto load_dz = [&](int c) {
    const int t0 = c * K;
    auto rows = [&](auto tail_tag) {
      constexpr bool TAIL = decltype(tail_tag)::value;
#pragma unroll
      for (int u = 0; u < BPW; ++u) {
        const IO* src = dzc + ((long long)(cb0 + u) * TmD + t0) * B + b;
        const bool ok = valid && u < nbw;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          dzn[u][k] = (ok && (!TAIL || t0 + k < TmD)) ? *src : IO(0);
          src += B;
        }
      }
    };
    if (t0 + K > TmD) rows(std::true_type{});
    else rows(std::false_type{});
  };
  if (BWD) load_dz(C - 1);
  for (int c = C - 1; c >= 0; --c, ++it, ++fb) {
    const int s = it % ST;
    const int t0 = c * K;
    // TAIL: the chunk holds rows >= T - D (the last d rows have no D z row; rows >= T none at all)
    const bool tail = t0 + K > TmD;
    IO dzv[BPW][K];
    double* const redw = redw0 + (c & (L::RSLOTS - 1)) * nw * K * 32;
    if (BWD) {
#pragma unroll
      for (int u = 0; u < BPW; ++u)
#pragma unroll
        for (int k = 0; k < K; ++k) dzv[u][k] = dzn[u][k];
      if (c > 0) load_dz(c - 1);
    }
    // this chunk's forward-substitution checkpoint (loaded one chunk ahead), then the next one's
#pragma unroll
    for (int u = 0; u < BPW; ++u)
#pragma unroll
      for (int i = 0; i < D; ++i) v[u][i] = vn[u][i];
    if (c > 0) load_v(c - 1);
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const IO* t_rhs = reinterpret_cast<const IO*>(ring + s * L::B_STAGE) + lane;
    mbar_wait(&fac_full[fb % L::NFB], (uint32_t)((fb / L::NFB) & 1));
    const unsigned char* F = fbuf0 + (fb % L::NFB) * L::FBUF;
    const double* FA = reinterpret_cast<const double*>(F + L::FB_A) + lane;
    const double* FI = reinterpret_cast<const double*>(F + L::FB_ID) + lane;
    const double* FMU = reinterpret_cast<const double*>(F + L::FB_MU) + lane;
    const double* FC0 = reinterpret_cast<const double*>(F + L::FB_C0) + lane;
    const IO* FW = reinterpret_cast<const IO*>(F + L::FB_W) + lane;
    double q[BPW][K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const IO wio = FW[k * 32];
      const double w = to_f64<IO>(wio);
      const double idk = FI[k * 32];
#pragma unroll
      for (int u = 0; u < BPW; ++u) {
        double vv = rhs_times_w<IO, BWD>(t_rhs[(u * K + k) * 32], wio, w);
#pragma unroll
        for (int j = D; j >= 1; --j) {
          const double mj = IRR ? FMU[((k + D - j) * D + j - 1) * 32] : Mj(D, j);
          if (j > 1) {
            vv = fma(-mj, v[u][j - 1], vv);
            vv = fma(-FA[(k * D + j - 1) * 32], v[u][j - 1], vv);
          } else {
            vv = fma(-(mj + FA[k * D * 32]), v[u][0], vv);
          }
        }
#pragma unroll
        for (int i = D - 1; i >= 1; --i) v[u][i] = v[u][i - 1];
        v[u][0] = vv;
        q[u][k] = vv * idk;  // rows past T: FI = 0 -> q = 0
      }
    }
    auto back_rows = [&](auto tail_tag) {
      constexpr bool TAIL = decltype(tail_tag)::value;
      // output rows walked downwards from row t0 + K - 1
      IO* o0[BPW];
      IO* o1[BPW];
#pragma unroll
      for (int u = 0; u < BPW; ++u) {
        o0[u] = out0 + ((long long)(cb0 + u) * T + t0 + K - 1) * B + b;
        o1[u] = out1 + ((long long)(cb0 + u) * TmD + t0 + K - 1) * B + b;
      }
#pragma unroll
      for (int k = K - 1; k >= 0; --k) {
        const int t = t0 + k;
        const IO wio = FW[k * 32];
        double a[D];
#pragma unroll
        for (int j = 1; j <= D; ++j) a[j - 1] = (k + j < K) ? FA[((k + j) * D + j - 1) * 32] : cA[k + j - K][j - 1];
        double ls = 0.0;  // this warp's bands' -(D u)(D z) at row t (per-date backward)
#pragma unroll
        for (int u = 0; u < BPW; ++u) {
          double z = q[u][k];
#pragma unroll
          for (int j = D; j >= 1; --j) {  // M~[t+j][t] = mu_t[j] (IRR), else M_j; j = 1: L = M + A first
            const double mj = IRR ? FMU[((k + D) * D + j - 1) * 32] : Mj(D, j);
            if (j > 1) {
              z = fma(-mj, zw[u][j - 1], z);
              z = fma(-a[j - 1], zw[u][j - 1], z);
            } else {
              z = fma(-(mj + a[0]), zw[u][0], z);
            }
          }
          double dz;
          if constexpr (IRR) {  // (D z)_t = c_{t,0} (z_t + sum_j mu_t[j] z_{t+j})
            double du = z;
#pragma unroll
            for (int j = 1; j <= D; ++j) du = fma(FMU[((k + D) * D + j - 1) * 32], zw[u][j - 1], du);
            dz = FC0[k * 32] * du;
          } else {
            dz = Cj(D, 0) * z;
#pragma unroll
            for (int j = 1; j <= D; ++j) dz = fma(Cj(D, j), zw[u][j - 1], dz);
          }
#pragma unroll
          for (int i = D - 1; i >= 1; --i) zw[u][i] = zw[u][i - 1];
          zw[u][0] = z;
          const bool ok = valid && u < nbw;
          const bool in_t = !TAIL || t < T;
          const bool in_dz = !TAIL || t < TmD;
          if (!BWD) {
            if (ok && in_t) *o0[u] = from_f64<IO>(z);
            if (ok && in_dz) *o1[u] = from_f64<IO>(dz);
          } else {
            if (sizeof(IO) == 4 && PD && !IRR) {  // (as the single-series kernels of each grid)
              if (ok && in_t) *o0[u] = wio * from_f64<IO>(z);
              if (u < nbw) ls += to_f64<IO>(-(from_f64<IO>(dz) * dzv[u][k]));
            } else {
              if (ok && in_t) *o0[u] = from_f64<IO>(to_f64<IO>(wio) * z);
              const double g = -dz * to_f64<IO>(dzv[u][k]);
              if (u < nbw) {
                if (PD) ls += g;
                else if (in_dz) lam_acc += g;
              }
            }
          }
          o0[u] -= B;
          o1[u] -= B;
        }
        if (BWD && PD) redw[(bj * K + k) * 32 + lane] = ls;  // slot c & 1
      }
    };
    if (tail) back_rows(std::true_type{});
    else back_rows(std::false_type{});
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) cA[i][j] = FA[(i * D + j) * 32];
    __syncwarp();
    if (lane == 0) mbar_arrive(&fac_empty[fb % L::NFB]);
    if (BWD && PD) {
      // grad_lambda_r = sum over band warps (fixed order) of their two bands' -(D u)(D z)
      // RSLOTS = 2: one barrier per chunk (slot c & 1 is written again two chunks later, after every warp has
      // passed the next chunk's barrier, i.e. finished reducing this one); RSLOTS = 4: one barrier per two
      // chunks, reducing both (a slot is rewritten four chunks later, past the next pair's barrier)
      const bool red_now = L::RSLOTS == 2 || ((C - 1 - c) & 1) == 1 || c == 0;
      if (red_now) {
        named_bar_sync(1, 32 * nw);
        const int c_hi = (L::RSLOTS == 2 || ((C - 1 - c) & 1) == 0) ? c : c + 1;  // (c == 0 alone when C is odd)
        for (int cc = c_hi; cc >= c; --cc) {
          const double* rw = redw0 + (cc & (L::RSLOTS - 1)) * nw * K * 32;
          for (int k = bj; k < K; k += nw) {
            const int t = cc * K + k;
            double acc = 0.0;
            for (int j = 0; j < nw; ++j) acc += rw[(j * K + k) * 32 + lane];
            if (valid && t < TmD) out1[(long long)t * B + b] = from_f64<IO>(acc);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue(it + ST);
    }
  }
  if (BWD && !PD) {
    redS[bj * 32 + lane] = lam_acc;
    __syncthreads();
    if (bj == 0) {
      double acc = 0.0;
      for (int j = 0; j < nw; ++j) acc += redS[j * 32 + lane];
      if (valid) out1[b] = from_f64<IO>(acc);
    }
  }
}

}  // namespace whit
