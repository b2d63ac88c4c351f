// libwhit twisted (two-ended) factorisation for small batches (DESIGN §5 "small batches").
//
// One series per lane as in whit_kernel, but each group of 32 series is split in time between a PAIR of
// warps that work concurrently: with the twist block S = [m, m+d) (m a multiple of K),
//   * the TOP warp factors Omega_top = W_[0,m) + sum_{r<m} lambda_r d_r d_r^T on dates [0, m+d) -- the
//     standard deviation-form LDL^T (R-10) run forward, with w, W y and lambda~ cut at row m by the TMA
//     tensor maps (rows >= m read as zero);
//   * the BOTTOM warp factors Omega_bot = W_[m,T) + sum_{r>=m} lambda_r d_r d_r^T on dates [m, T) in
//     REVERSED time: reversing the dates turns the difference operator into (-1)^d times itself (R-3), so the
//     reversed block is again a standard Whittaker matrix, with lambda~''(t) = lambda_{t-d} (t >= m+d) -- the
//     same recurrence, reading each staged tile bottom-up;
//   * Omega = Omega_top + Omega_bot and the blocks [0,m) and [m+d,T) do not couple, so eliminating both
//     leaves the d x d system  (Sigma_top + Sigma_bot) z_S = r_top + r_bot  with Sigma_x = L_SS D_S L_SS^T
//     and r_x = L_SS v_S read off each half's recurrence state after its last row (both are data-scale:
//     the lambda-scale part of Omega never enters);
//   * both warps exchange (Sigma_x, r_x) through shared memory, solve the d x d system identically (same
//     operation order, bitwise the same z_S), and back-substitute their own halves outward from S.
// Each warp runs T/2 rows instead of T: half the latency per series and twice the warps, so batches that
// fill the 148 SMs only ~1-2 times (the homo config, strong-scaling shards) lose much less to the wave
// tail.  Checkpoints (R-mode) as in whit_kernel: top chunk c -> slot c, bottom chunk c'' -> slot C1 + c''.
//
// A pair whose halves are not safely positive definite on their own (a half with fewer than 2d observed
// days -- its Schur complement onto S would be singular or nearly so -- or any failing pivot, or a non-SPD
// d x d block) writes twflag = 0 and leaves the whole 32-series group to whit_kernel, launched right after
// with p.tw_filter set: the exact LAPACK-style status (R-8) always comes from the sequential factorisation.
#pragma once
#include "whit_kernels.cuh"

namespace whit {

template <int D, typename IO, bool PD, bool BWD>
struct TwLayout {
  static constexpr int K = Tile<IO, D, false>::K;  // chunk rows as the single-series kernels
#ifndef WHIT_TW_ST
#define WHIT_TW_ST 2
#endif
  static constexpr int ST = sizeof(IO) == 4 ? WHIT_TW_ST : 2;  // (fp64 tiles: two stages fill the CTA budget)
  static constexpr int PAIRS = 2;  // warp pairs per CTA
  static constexpr int ROW = 32 * (int)sizeof(IO);
  static constexpr int OFF_RHS = 0;
  static constexpr int OFF_W = K * ROW;
  static constexpr int OFF_LAM = 2 * K * ROW;                          // (K + d)-row lambda box
  static constexpr int OFF_DZ = OFF_LAM + (PD ? (K + D) * ROW : 0);
  static constexpr int STAGE = (OFF_DZ + (BWD ? K * ROW : 0) + 127) / 128 * 128;
#ifndef WHIT_TW_DIRECT  // outputs by direct coalesced stores (no staging planes: 12 warps/SM in both directions)
#define WHIT_TW_DIRECT 0
#endif
  static constexpr bool DIRECT = WHIT_TW_DIRECT;
  static constexpr int OUT = DIRECT ? 0 : K * ROW;
  static constexpr int NX = D * (D + 1) / 2 + D + 2;                   // exchange fields (fp64) per lane
  static constexpr int XCH = NX * 32 * 8;
  static constexpr int WARP_SMEM = ST * STAGE + 2 * OUT + XCH;
  static constexpr int SMEM = 2 * PAIRS * WARP_SMEM;
  static constexpr uint32_t BYTES = (2 * K + (PD ? K + D : 0) + (BWD ? K : 0)) * ROW;
};

#ifndef WHIT_TW_STAGE  // debug: stop after stage n (1 init, 2 first tiles, 3 up sweep, 4 exchange, 5 all but the down sweep); 0 = full
#define WHIT_TW_STAGE 0
#endif
#ifndef WHIT_TW_MAXREG
#define WHIT_TW_MAXREG 168
#endif

// Per-direction sweep bodies in "processing space": step p = 0..K-1 of a chunk visits tile row
// k = p (top) or K-1-p (bottom, REV), date t = t_lo + k.
template <int D, typename IO, bool PD, bool BWD, bool REV>
struct TwSweep {
  using L = TwLayout<D, IO, PD, BWD>;
  static constexpr int K = L::K;
  static __device__ __forceinline__ int krow(int p) { return REV ? K - 1 - p : p; }
  // the row's own lambda~: top, lambda box at t0-d (index k+d = row t, cut at m by the map); bottom,
  // box at t_lo-d in the map based at row m (index k = lambda_{t-d}, zero below m)
  static __device__ __forceinline__ double lam_own(const IO* t_lam, int k, int t, int m, double lam_s) {
    if (PD) return to_f64<IO>(t_lam[(REV ? k : k + D) * 32]);
    return REV ? ((t >= m + D) ? lam_s : 0.0) : ((t < m) ? lam_s : 0.0);
  }
  // is date t outside this half's sub-problem (top: t >= m+d; bottom: t < m)
  static __device__ __forceinline__ bool outside(int t, int m) { return REV ? (t < m) : (t >= m + D); }

  template <bool EDGE>
  static __device__ __forceinline__ void up_chunk(FState<D>& st, const unsigned char* stg, int lane, int t_lo, int m,
                                                  double lam_s, int& nobs, int& bad) {
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + lane;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int k = krow(p), t = t_lo + k;
      if (EDGE && outside(t, m)) break;
      const IO wio = t_w[k * 32];
      const double w = to_f64<IO>(wio);
      const double lt = lam_own(t_lam, k, t, m, lam_s);
      const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, w);
      double A[D], Dt, idt, vt;
      ldl_step<D, Newton<IO, D>::N>(st, w, lt, bb, A, Dt, idt, vt);
      if (!BWD) {
        nobs += (wio > IO(0));
        if (bad == 0 && !pivot_ok(Dt)) bad = t + 1;
      }
    }
  }

  // Recompute the chunk's factor from the restored state, then back-substitute (dates outward from S) and
  // stage the outputs at their tile rows: top z_t, (D z)_t; bottom z_t, (D z)_{t-d}; backward w u and
  // -(D u)(D z) (per date) or the scalar partial sum.  EDGE: the chunk holding S -- rows outside the half
  // are zero, S rows take z_S.
  template <bool EDGE>
  static __device__ __forceinline__ void down_chunk(FState<D>& st, double (&cA)[D][D], double (&zw)[D],
                                                    double& lam_acc, const unsigned char* stg, int lane, int t_lo,
                                                    int m, double lam_s, const double (&zS)[D], IO* so0, IO* so1,
                                                    IO* g0, IO* g1, long long B, bool valid) {
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::OFF_RHS) + lane;
    const IO* t_w = reinterpret_cast<const IO*>(stg + L::OFF_W) + lane;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;
    const IO* t_dz = reinterpret_cast<const IO*>(stg + L::OFF_DZ) + lane;
    double q[K];
    double Ak[K][D];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int k = krow(p), t = t_lo + k;
      const IO wio = t_w[k * 32];
      const double w = to_f64<IO>(wio);
      const double lt = lam_own(t_lam, k, t, m, lam_s);
      const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, w);
      double Dt, idt, vt;
      ldl_step<D, Newton<IO, D>::N>(st, w, lt, bb, Ak[p], Dt, idt, vt);
      q[p] = vt * idt;
      if (EDGE && outside(t, m)) {
        q[p] = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) Ak[p][j] = 0.0;
      }
    }
#pragma unroll
    for (int p = K - 1; p >= 0; --p) {
      const int k = krow(p), t = t_lo + k;
      double z = q[p];
#pragma unroll
      for (int j = D; j >= 1; --j) {
        const double a = (p + j < K) ? Ak[p + j][j - 1] : cA[p + j - K][j - 1];
        if (j > 1) {
          z = fma(-Mj(D, j), zw[j - 1], z);
          z = fma(-a, zw[j - 1], z);
        } else {
          z = fma(-(Mj(D, 1) + a), zw[0], z);  // (L = M + A first, as Sweep::back_row)
        }
      }
      if (EDGE && t >= m && t < m + D) {
        // S row: the twist solution (select, no dynamic register indexing)
#pragma unroll
        for (int a = 0; a < D; ++a) z = (t == m + a) ? zS[a] : z;
      }
      // top: (D z)_t = sum_j c_j z_{t+j};  bottom: (D z)_{t-d} = c_d z_t + sum_{j>=1} c_{d-j} z_{t-j}
      double dz = (REV ? Cj(D, D) : Cj(D, 0)) * z;
#pragma unroll
      for (int j = 1; j <= D; ++j) dz = fma(REV ? Cj(D, D - j) : Cj(D, j), zw[j - 1], dz);
#pragma unroll
      for (int i = D - 1; i >= 1; --i) zw[i] = zw[i - 1];
      zw[0] = z;
      IO o0v, o1v = IO(0);
      if (!BWD) {
        o0v = from_f64<IO>(z);
        o1v = from_f64<IO>(dz);
      } else {
        const double w = to_f64<IO>(t_w[k * 32]);
        o0v = (sizeof(IO) == 4) ? t_w[k * 32] * from_f64<IO>(z) : from_f64<IO>(w * z);
        if (PD) {
          o1v = (sizeof(IO) == 4) ? IO(-(from_f64<IO>(dz) * t_dz[k * 32]))
                                  : from_f64<IO>(-dz * to_f64<IO>(t_dz[k * 32]));
        } else {
          const bool row_ok = REV ? (t >= m + D) : (t < m);  // this half's difference rows
          if (!EDGE || row_ok) lam_acc += -dz * to_f64<IO>(t_dz[k * 32]);
        }
      }
      if (L::DIRECT) {  // this half's rows only: z / grad_y at t, D z / grad_lambda at r (top r = t, bottom t - d)
        const int r = REV ? t - D : t;
        const bool own_t = !EDGE || (REV ? t >= m : t < m);
        const bool own_r = !EDGE || (REV ? r >= m : r < m);
        if (valid && own_t) g0[(long long)k * B] = o0v;
        if (valid && (!BWD || PD) && own_r) g1[(long long)k * B] = o1v;
      } else {
        so0[k * 32] = o0v;
        so1[k * 32] = o1v;
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) cA[i][j] = Ak[i][j];
  }
};

// Issue tile i of one warp (up tiles 0..Cn-1, then down tiles Cn-1..0).  Chunk c: top dates [cK, cK+K),
// bottom dates [T-(c+1)K, T-cK) in maps based at row m.
template <int D, typename IO, bool PD, bool BWD, bool REV>
__device__ __forceinline__ void tw_issue(const Params& p, unsigned char* stage, uint64_t* bar, int i, int Cn,
                                         int bw) {
  using L = TwLayout<D, IO, PD, BWD>;
  const int c = i < Cn ? i : 2 * Cn - 1 - i;
  mbar_arrive_expect_tx(bar, L::BYTES);
  if (!REV) {
    const int t0 = c * L::K;
    tma_load_2d(stage + L::OFF_RHS, &p.tm_rhs, bw, t0, bar);
    tma_load_2d(stage + L::OFF_W, &p.tm_w, bw, t0, bar);
    if (PD) tma_load_2d(stage + L::OFF_LAM, &p.tm_lam_dn, bw, t0 - D, bar);
    if (BWD) tma_load_2d(stage + L::OFF_DZ, &p.tm_dz, bw, t0, bar);
  } else {
    const int r_lo = p.T - (c + 1) * L::K - p.tw_m;  // chunk's first date relative to row m
    tma_load_2d(stage + L::OFF_RHS, &p.tmb_rhs, bw, r_lo, bar);
    tma_load_2d(stage + L::OFF_W, &p.tmb_w, bw, r_lo, bar);
    if (PD) tma_load_2d(stage + L::OFF_LAM, &p.tmb_lam, bw, r_lo - D, bar);
    if (BWD) tma_load_2d(stage + L::OFF_DZ, &p.tmb_dz, bw, r_lo - D, bar);
  }
}

template <int D, typename IO, bool PD, bool BWD, bool REV, bool HIREG>
__device__ __forceinline__ void tw_half(const Params& p, unsigned char* ring, uint64_t* bars, double* xme,
                                        const double* xother, int pair_bar, int lane, long long bw, bool valid,
                                        long long b, double lam_s) {
  using L = TwLayout<D, IO, PD, BWD>;
  using S = TwSweep<D, IO, PD, BWD, REV>;
  constexpr int K = L::K, ST = L::ST, NFAC = Ck<D>::NFAC;
  const int T = p.T, m = p.tw_m;
  const long long B = p.B;
  const int Cn = REV ? p.tw_C2 : p.tw_C1;
  const int slot0 = REV ? p.tw_C1 : 0;
  const int ntiles = 2 * Cn;
  IO* so0 = reinterpret_cast<IO*>(ring + ST * L::STAGE);
  IO* so1 = reinterpret_cast<IO*>(ring + ST * L::STAGE + L::OUT);
  auto t_lo_of = [&](int c) { return REV ? T - (c + 1) * K : c * K; };
  // chunks that hold S rows (or rows outside the half): top -- its last chunk (m is a multiple of K);
  // bottom -- its last one or two (S may straddle their boundary)
  auto edge = [&](int c) { return REV ? (t_lo_of(c) < m + D) : (t_lo_of(c) + K > m); };
  if (lane == 0) {
    for (int s = 0; s < ST && s < ntiles; ++s) tw_issue<D, IO, PD, BWD, REV>(p, ring + s * L::STAGE, &bars[s], s, Cn, (int)bw);
  }
  __syncwarp();
  if (WHIT_TW_STAGE == 2) {
    for (int j = 0; j < ST && j < ntiles; ++j) mbar_wait(&bars[j], 0);
    return;
  }
  double* const ck_rhs = (BWD ? p.ck_rhs_b : p.ck_rhs_f) + b;

  FState<D> st;
  state_init<D>(st);
  int nobs = 0, bad = 0, it = 0;
  // ------------------------------------------------------------ up sweep (factor + forward substitution)
  for (int c = 0; c < Cn; ++c, ++it) {
    const int s = it % ST;
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * L::STAGE;
    if (valid) {
      if (!BWD) {
        double* ck = p.ck_fac + (long long)(slot0 + c) * NFAC * B + b;
        int f = 0;
#pragma unroll
        for (int i = 0; i < D; ++i) ck[(long long)(f++) * B] = st.dl[i];
#pragma unroll
        for (int mm = 0; mm < D - 1; ++mm)
#pragma unroll
          for (int k = 0; k < D - 1 - mm; ++k) ck[(long long)(f++) * B] = st.ap[mm][k];
      }
      double* ck = ck_rhs + (long long)(slot0 + c) * D * B;
#pragma unroll
      for (int i = 0; i < D; ++i) ck[(long long)i * B] = st.v[i];
    }
    if (edge(c)) S::template up_chunk<true>(st, stg, lane, t_lo_of(c), m, lam_s, nobs, bad);
    else S::template up_chunk<false>(st, stg, lane, t_lo_of(c), m, lam_s, nobs, bad);
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      tw_issue<D, IO, PD, BWD, REV>(p, ring + s * L::STAGE, &bars[s], it + ST, Cn, (int)bw);
    }
  }

  if (WHIT_TW_STAGE == 3) {
    for (int j = it; j < ntiles && j < it + ST; ++j) mbar_wait(&bars[j % ST], (uint32_t)((j / ST) & 1));
    return;
  }
  // ------------------------------------------------------------ the twist: Sigma_x, r_x of this half
  // S index a = date - m.  Top: state row i <-> date m+d-1-i, L_SS lower;  bottom: i <-> date m+i, its
  // reversed-time factor is "upper" in date order.  Sigma_x = L D L^T over S, r_x = L v.
  {
    double Lm[D][D], Dd[D], vv[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int i = REV ? a : D - 1 - a;
      Dd[a] = st.dl[i];  // lambda~ = 0 on S rows of both halves: D_t = Delta_t
      vv[a] = st.v[i];
#pragma unroll
      for (int c = 0; c < D; ++c) Lm[a][c] = (a == c) ? 1.0 : 0.0;
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        if (!REV && c < a) Lm[a][c] = Mj(D, a - c) + st.ap[D - 1 - a][a - c - 1];
        if (REV && c > a) Lm[a][c] = Mj(D, c - a) + st.ap[a][c - a - 1];
      }
    int f = 0;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int bq = 0; bq <= a; ++bq) {
        double sacc = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) sacc = fma(Lm[a][c] * Dd[c], Lm[bq][c], sacc);
        xme[(f++) * 32 + lane] = sacc;
      }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double racc = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) racc = fma(Lm[a][c], vv[c], racc);
      xme[(f++) * 32 + lane] = racc;
    }
    // health of this half for the pair's decision (forward only; the backward follows twflag)
    const bool ok_half = !valid || (bad == 0 && nobs >= 2 * D);
    xme[f * 32 + lane] = ok_half ? 1.0 : 0.0;
  }
  __syncwarp();  // bar.sync is .aligned: the warp must arrive converged (lane 0 may still be issuing)
  named_bar_sync(pair_bar, 64);
  // both warps: Sigma = Sigma_top + Sigma_bot, r = r_top + r_bot (in that order), LDL^T solve of d x d
  const double* xt = REV ? xother : xme;
  const double* xb = REV ? xme : xother;
  double zS[D];
  bool ok;
  {
    double Sg[D][D], r[D];
    int f = 0;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int bq = 0; bq <= a; ++bq) {
        Sg[a][bq] = xt[f * 32 + lane] + xb[f * 32 + lane];
        Sg[bq][a] = Sg[a][bq];
        ++f;
      }
#pragma unroll
    for (int a = 0; a < D; ++a, ++f) r[a] = xt[f * 32 + lane] + xb[f * 32 + lane];
    ok = BWD || (xt[f * 32 + lane] != 0.0 && xb[f * 32 + lane] != 0.0);
    double Ld[D][D], Dp[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double dd = Sg[i][i];
#pragma unroll
      for (int k = 0; k < i; ++k) dd = fma(-Ld[i][k] * Dp[k], Ld[i][k], dd);
      Dp[i] = dd;
      ok = ok && pivot_ok(dd);
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        double e = Sg[j][i];
#pragma unroll
        for (int k = 0; k < i; ++k) e = fma(-Ld[j][k] * Dp[k], Ld[i][k], e);
        Ld[j][i] = e / dd;
      }
    }
    double y[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double yy = r[i];
#pragma unroll
      for (int k = 0; k < i; ++k) yy = fma(-Ld[i][k], y[k], yy);
      y[i] = yy;
    }
#pragma unroll
    for (int i = D - 1; i >= 0; --i) {
      double zz = y[i] / Dp[i];
#pragma unroll
      for (int k = i + 1; k < D; ++k) zz = fma(-Ld[k][i], zS[k], zz);
      zS[i] = zz;
    }
  }
  if (WHIT_TW_STAGE == 4) {
    for (int j = it; j < ntiles && j < it + ST; ++j) mbar_wait(&bars[j % ST], (uint32_t)((j / ST) & 1));
    return;
  }
  if (!BWD) {
    const bool pair_ok = __all_sync(0xffffffffu, ok || !valid);
    if (!pair_ok) {
      // leave the group to whit_kernel (launched next): drain the speculatively issued tiles and stop
      if (!REV && lane == 0) p.twflag[bw >> 5] = 0;
      for (int j = it; j < ntiles && j < it + ST; ++j) mbar_wait(&bars[j % ST], (uint32_t)((j / ST) & 1));
      return;
    }
    if (!REV) {
      if (lane == 0) p.twflag[bw >> 5] = 1;
      if (valid) p.info[b] = 0;
    }
  }

  if (WHIT_TW_STAGE == 5) {  // debug timing: everything but the down sweep (the group counts as solved)
    for (int j = it; j < ntiles && j < it + ST; ++j) mbar_wait(&bars[j % ST], (uint32_t)((j / ST) & 1));
    return;
  }
  // ------------------------------------------------------------ down sweep (outward from S)
  double cA[D][D], zw[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    zw[i] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) cA[i][j] = 0.0;
  }
  double lam_acc = 0.0;
  // checkpoints of the next chunk, loaded one chunk ahead by predicated loads (ld_pred_f64): 8,192 hetero series
  // 0.72 -> 0.61 ms per fwd+bwd step.  Not in the 168-register scalar-lambda forward, where the prefetch registers
  // spill (its chunk then waits on its own checkpoint load, as before: 0.348 vs 0.363 ms)
  constexpr bool CKPRE = PD || BWD || HIREG;
  double pck[NFAC], pv[D];
  auto load_ck = [&](int c) {
    const double* ckf = p.ck_fac + (long long)(slot0 + c) * NFAC * B + b;
    const double* ckr = ck_rhs + (long long)(slot0 + c) * D * B;
#pragma unroll
    for (int f = 0; f < NFAC; ++f) pck[f] = ld_pred_f64(ckf + (long long)f * B, valid);
#pragma unroll
    for (int i = 0; i < D; ++i) pv[i] = ld_pred_f64(ckr + (long long)i * B, valid);
  };
  if (CKPRE) load_ck(Cn - 1);
  for (int c = Cn - 1; c >= 0; --c, ++it) {
    const int s = it % ST;
    // restore the state entering step p = 0 of chunk c from its checkpoint
    {
      if (!CKPRE) load_ck(c);
      int f = 0;
#pragma unroll
      for (int i = 0; i < D; ++i) st.dl[i] = pck[f++];
#pragma unroll
      for (int mm = 0; mm < D - 1; ++mm)
#pragma unroll
        for (int k = 0; k < D - 1 - mm; ++k) st.ap[mm][k] = pck[f++];
#pragma unroll
      for (int i = 0; i < D; ++i) st.v[i] = pv[i];
    }
    if (CKPRE && c > 0) load_ck(c - 1);
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * L::STAGE;
    const IO* t_lam = reinterpret_cast<const IO*>(stg + L::OFF_LAM) + lane;
    const int t_lo = t_lo_of(c);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      // the row visited i+1 steps before the chunk: top date t_lo-1-i, bottom date t_lo+K+i
      const int tj = REV ? t_lo + K + i : t_lo - 1 - i;
      const bool virt = REV ? (tj >= T) : (tj < 0);
      double l;
      if (PD) l = to_f64<IO>(t_lam[(REV ? K + i : D - 1 - i) * 32]);
      else l = REV ? ((tj >= m + D && tj < T) ? lam_s : 0.0) : ((tj >= 0 && tj < m) ? lam_s : 0.0);
      st.lm[i] = l;
      st.id[i] = virt ? 1.0 : rcp64<Newton<IO, D>::N>(l + st.dl[i]);
    }
    if (!L::DIRECT) {
      if (lane == 0) bulk_wait_read0();  // staging tiles free again
      __syncwarp();
    }
    // this chunk's output rows (direct stores): g0 at row t_lo, g1 at row t_lo (top) / t_lo - d (bottom)
    IO* const g0 = reinterpret_cast<IO*>(p.out0) + b + (long long)t_lo * B;
    IO* const g1 = reinterpret_cast<IO*>(p.out1) + b + (long long)(REV ? t_lo - D : t_lo) * B;
    if (edge(c))
      S::template down_chunk<true>(st, cA, zw, lam_acc, stg, lane, t_lo, m, lam_s, zS, so0 + lane, so1 + lane, g0, g1,
                                   B, valid);
    else
      S::template down_chunk<false>(st, cA, zw, lam_acc, stg, lane, t_lo, m, lam_s, zS, so0 + lane, so1 + lane, g0,
                                    g1, B, valid);
    if (!L::DIRECT && edge(c)) {
      // chunks at S: a tensor store would start outside its plane (top: at row m; bottom: below row m),
      // so each lane writes its own rows of the staged tile directly, inside the half's rows only
      IO* o0 = reinterpret_cast<IO*>(p.out0);
      IO* o1 = reinterpret_cast<IO*>(p.out1);
      const IO* s0 = so0 + lane;
      const IO* s1 = so1 + lane;
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        const int t = t_lo + k, r = REV ? t - D : t;
        const bool own_t = REV ? (t >= m && t < T) : (t < m);
        const bool own_r = REV ? (r >= m && r < T - D) : (r < m);
        if (valid && own_t) o0[(long long)t * B + b] = s0[k * 32];
        if (valid && (!BWD || PD) && own_r) o1[(long long)r * B + b] = s1[k * 32];
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && !L::DIRECT && !edge(c)) {
      // top maps end at row m; bottom maps start at row m
      if (!REV) {
        tma_store_2d(&p.tm_out0, so0, (int)bw, t_lo);
        if (!BWD || PD) tma_store_2d(&p.tm_out1, so1, (int)bw, t_lo);
      } else {
        const int r_lo = t_lo - m;
        tma_store_2d(&p.tmb_out0, so0, (int)bw, r_lo);
        if (!BWD || PD) tma_store_2d(&p.tmb_out1, so1, (int)bw, r_lo - D);
      }
      bulk_commit();
    }
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      tw_issue<D, IO, PD, BWD, REV>(p, ring + s * L::STAGE, &bars[s], it + ST, Cn, (int)bw);
    }
  }
  if (lane == 0) bulk_wait0();
  if (BWD && !PD) {  // scalar lambda: dL/dlambda = top rows + bottom rows (in that order)
    if (REV) xme[(L::NX - 1) * 32 + lane] = lam_acc;
    __syncwarp();
    named_bar_sync(pair_bar, 64);
    if (!REV && valid) reinterpret_cast<IO*>(p.out1)[b] = from_f64<IO>(lam_acc + xother[(L::NX - 1) * 32 + lane]);
  }
}

// HIREG: the instantiation for launches whose warps fit one wave at 8 warps/SM (<= 592 groups): 255
// registers, no spills (the 168-register build spills up to 360 B at d = 3 and keeps 12 warps/SM, which only
// pays once the twisted warps fill that wave)
template <int D, typename IO, bool PD, bool BWD, bool HIREG = false>
__global__ void __maxnreg__((HIREG ? 255 : WHIT_TW_MAXREG)) whit_tw_kernel(const __grid_constant__ Params p) {
  using L = TwLayout<D, IO, PD, BWD>;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[2 * L::PAIRS][L::ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1;  // half 0: top, 1: bottom
  const long long B = p.B;
  const long long bw = ((long long)(blockIdx.x + p.tw_cta0) * L::PAIRS + pair) * 32;
  if (bw >= B) return;  // both warps of the pair leave together (no barrier is pending)
  const long long b = bw + lane;
  const bool valid = b < B;
  if (BWD && p.twflag[bw >> 5] == 0) return;  // this group went through whit_kernel
  unsigned char* ring = smem + warp * L::WARP_SMEM;
  double* xme = reinterpret_cast<double*>(ring + L::ST * L::STAGE + 2 * L::OUT);
  const double* xother = reinterpret_cast<const double*>(smem + (warp ^ 1) * L::WARP_SMEM + L::ST * L::STAGE + 2 * L::OUT);
  uint64_t* bars = full_bar[warp];
  if (lane == 0) {
    for (int s = 0; s < L::ST; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const double lam_s = (!PD && valid) ? to_f64<IO>(reinterpret_cast<const IO*>(p.lam_scalar)[b]) : 0.0;
  const int pair_bar = 1 + pair;
  if (WHIT_TW_STAGE == 1) return;
  if (half == 0)
    tw_half<D, IO, PD, BWD, false, HIREG>(p, ring, bars, xme, xother, pair_bar, lane, bw, valid, b, lam_s);
  else
    tw_half<D, IO, PD, BWD, true, HIREG>(p, ring, bars, xme, xother, pair_bar, lane, bw, valid, b, lam_s);
}

}  // namespace whit
