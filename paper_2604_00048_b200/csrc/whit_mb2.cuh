// libwhit multi-band kernel with a shared factor warp (NEXT-1, P:28 / P:147: the C bands of a
// pixel share W and Lambda, hence Omega and its factor).
//
// CTA = C band warps + 1 factor warp over 32 pixels:
//  * the factor warp streams w and lambda (its own TMA ring), runs the deviation-form LDL^T
//    (ldl_step, R-10) once per pixel and publishes, per K-row chunk, the rows
//    (A_{t,1..d}, 1/D_t, w_t) into one of two shared-memory factor buffers (mbarriers
//    fac_full / fac_empty); it writes the factor checkpoints and, in the down sweep, recomputes
//    each chunk's factor from them;
//  * each band warp streams only its band's right-hand side (y, or g and D z) and runs the
//    4-flop forward-substitution recurrence and the back substitution with the published rows.
// The band warps execute exactly the fp64 operation sequence of the single-band kernel, so every
// band's z, grad_y equal the independent-series results bit for bit; grad_lambda is the band sum
// (fp64, band order) reduced in shared memory.
#pragma once
#include "whit_kernels.cuh"

namespace whit {

template <int D, typename IO, bool PD, bool BWD>
struct MB2Layout {
  static constexpr int K = D <= 2 ? 16 : 8, ST = 2;
  static constexpr int ROW = 32 * (int)sizeof(IO);
  // factor warp ring: w K rows + lambda K+d rows
  static constexpr int F_OFF_W = 0, F_OFF_LAM = K * ROW;
  static constexpr int F_STAGE = (F_OFF_LAM + (PD ? (K + D) * ROW : 0) + 127) / 128 * 128;
  // band warp ring: rhs K rows (+ D z K rows in the backward)
  static constexpr int B_OFF_RHS = 0, B_OFF_DZ = K * ROW;
  static constexpr int B_STAGE = ((BWD ? 2 : 1) * K * ROW + 127) / 128 * 128;
  static constexpr int OUT = K * ROW;
  static constexpr int B_WARP = ST * B_STAGE + 2 * OUT;  // ring + 2 staged output planes
  // factor buffer: per row k: A[k][0..D-1], iD[k] (fp64), w[k] (IO), lane-contiguous
  static constexpr int FB_A = 0, FB_ID = D * K * 32 * 8, FB_W = (D + 1) * K * 32 * 8;
  static constexpr int FBUF = (FB_W + K * 32 * (int)sizeof(IO) + 127) / 128 * 128;
  static constexpr uint32_t F_BYTES_UP = (K + (PD ? K : 0)) * ROW;
  static constexpr uint32_t F_BYTES_DN = (K + (PD ? K + D : 0)) * ROW;
  static constexpr uint32_t B_BYTES_UP = K * ROW;
  static constexpr uint32_t B_BYTES_DN = (BWD ? 2 : 1) * K * ROW;
  // smem: factor ring | factor buffers x2 | band warps | reduction tile (fp64) + scalar slots
  static constexpr int OFF_FB = ST * F_STAGE;
  static constexpr int OFF_BAND = OFF_FB + 2 * FBUF;
  static constexpr int smem(int nb) { return OFF_BAND + nb * B_WARP + K * 32 * 8 + nb * 32 * 8; }
};

template <int D, typename IO, bool PD, bool BWD>
__global__ void __maxnreg__(168) whit_mb2_kernel(const __grid_constant__ Params p) {
  using L = MB2Layout<D, IO, PD, BWD>;
  constexpr int K = L::K, ST = L::ST, NFAC = Ck<D>::NFAC, NW = Newton<IO>::N;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t f_full[ST];           // factor warp's TMA ring
  __shared__ __align__(8) uint64_t b_full[kMaxBands][ST];  // band warps' TMA rings
  __shared__ __align__(8) uint64_t fac_full[2], fac_empty[2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = p.nb, T = p.T, C = p.C, TmD = T - D;
  const long long B = p.B;
  const long long bw = (long long)blockIdx.x * 32;
  if (bw >= B) return;  // whole CTA
  const long long b = bw + lane;
  const bool valid = b < B;
  const bool fwarp = warp == nb;  // the factor warp
  const int ntiles = 2 * C;
  unsigned char* fbuf0 = smem + L::OFF_FB;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&fac_full[i], 1);
      mbar_init(&fac_empty[i], nb);
    }
  }
  if (lane == 0) {
    if (fwarp) {
      for (int s = 0; s < ST; ++s) mbar_init(&f_full[s], 1);
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
      unsigned char* stg = ring + (i % ST) * L::F_STAGE;
      mbar_arrive_expect_tx(&f_full[i % ST], up ? L::F_BYTES_UP : L::F_BYTES_DN);
      tma_load_2d(stg + L::F_OFF_W, &p.tm_w, (int)bw, t0, &f_full[i % ST]);
      if (PD) {
        if (up) tma_load_2d(stg + L::F_OFF_LAM, &p.tm_lam_up, (int)bw, t0, &f_full[i % ST]);
        else tma_load_2d(stg + L::F_OFF_LAM, &p.tm_lam_dn, (int)bw, t0 - D, &f_full[i % ST]);
      }
    };
    if (lane == 0)
      for (int i = 0; i < ST && i < ntiles; ++i) issue(i);
    __syncwarp();
    const double lam_s = (!PD && valid) ? to_f64<IO>(reinterpret_cast<const IO*>(p.lam_scalar)[b]) : 0.0;
    FState<D> st;
    state_init<D>(st);
    int nobs = 0;
    bool allpos = true;
    int it = 0, fb = 0;  // fb: factor-buffer sequence number
    // ---- up sweep
    for (int c = 0; c < C; ++c, ++it, ++fb) {
      const int s = it % ST;
      mbar_wait(&f_full[s], (uint32_t)((it / ST) & 1));
      const unsigned char* stg = ring + s * L::F_STAGE;
      const IO* t_w = reinterpret_cast<const IO*>(stg + L::F_OFF_W) + lane;
      const IO* t_lam = reinterpret_cast<const IO*>(stg + L::F_OFF_LAM) + lane;
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
      mbar_wait(&fac_empty[fb & 1], (uint32_t)(((fb >> 1) & 1) ^ 1));
      unsigned char* F = fbuf0 + (fb & 1) * L::FBUF;
      double* FA = reinterpret_cast<double*>(F + L::FB_A) + lane;
      IO* FW = reinterpret_cast<IO*>(F + L::FB_W) + lane;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int t = t0 + k;
        const IO wio = t_w[k * 32];
        const double w = to_f64<IO>(wio);
        double lt = PD ? to_f64<IO>(t_lam[k * 32]) : lam_s;
        if (!PD) lt = (t < TmD) ? lt : 0.0;
        double A[D], Dt, idt, vt;
        ldl_step<D, NW>(st, w, lt, 0.0, A, Dt, idt, vt);
#pragma unroll
        for (int j = 0; j < D; ++j) FA[(k * D + j) * 32] = A[j];
        FW[k * 32] = wio;
        if (!BWD && t < T) {
          nobs += (wio > IO(0));
          allpos = allpos && (Dt > 0.0);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&fac_full[fb & 1]);  // release: this warp's smem writes
      if (lane == 0 && it + ST < ntiles) {
        fence_proxy_async_smem();
        issue(it + ST);
      }
    }
    bool failed;
    if (!BWD) {
      if (valid) p.info[b] = (nobs < D) ? (T - D + 1) : (allpos ? 0 : -1);
      failed = (nobs < D) || !allpos;
    } else {
      failed = valid ? (p.info[b] != 0) : true;
    }
    const double poison = failed ? qnan() : 0.0;
    // ---- down sweep: recompute and publish each chunk's factor rows
    for (int c = C - 1; c >= 0; --c, ++it, ++fb) {
      const int s = it % ST;
      mbar_wait(&f_full[s], (uint32_t)((it / ST) & 1));
      const unsigned char* stg = ring + s * L::F_STAGE;
      const IO* t_w = reinterpret_cast<const IO*>(stg + L::F_OFF_W) + lane;
      const IO* t_lam = reinterpret_cast<const IO*>(stg + L::F_OFF_LAM) + lane;  // row k <-> t0 - D + k
      const int t0 = c * K;
      if (valid) {
        const double* ckf = p.ck_fac + (long long)c * NFAC * B + b;
        int f = 0;
#pragma unroll
        for (int i = 0; i < D; ++i) st.dl[i] = ckf[(long long)(f++) * B];
#pragma unroll
        for (int m = 0; m < D - 1; ++m)
#pragma unroll
          for (int k = 0; k < D - 1 - m; ++k) st.ap[m][k] = ckf[(long long)(f++) * B];
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const int tj = t0 - 1 - i;
        st.v[i] = 0.0;
        const double l = PD ? to_f64<IO>(t_lam[(D - 1 - i) * 32]) : ((tj >= 0 && tj < TmD) ? lam_s : 0.0);
        st.lm[i] = l;
        st.id[i] = (tj < 0) ? 1.0 : rcp64<NW>(l + st.dl[i]);
      }
      mbar_wait(&fac_empty[fb & 1], (uint32_t)(((fb >> 1) & 1) ^ 1));
      unsigned char* F = fbuf0 + (fb & 1) * L::FBUF;
      double* FA = reinterpret_cast<double*>(F + L::FB_A) + lane;
      double* FI = reinterpret_cast<double*>(F + L::FB_ID) + lane;
      IO* FW = reinterpret_cast<IO*>(F + L::FB_W) + lane;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int t = t0 + k;
        const IO wio = t_w[k * 32];
        const double w = to_f64<IO>(wio);
        double lt = PD ? to_f64<IO>(t_lam[(k + D) * 32]) : lam_s;
        if (!PD) lt = (t < TmD) ? lt : 0.0;
        double A[D], Dt, idt, vt;
        ldl_step<D, NW>(st, w, lt, 0.0, A, Dt, idt, vt);
        const bool past = t >= T;  // rows past the end: z = 0 (q = 0, A = 0)
#pragma unroll
        for (int j = 0; j < D; ++j) FA[(k * D + j) * 32] = past ? 0.0 : A[j];
        FI[k * 32] = past ? 0.0 : idt + poison;
        FW[k * 32] = wio;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&fac_full[fb & 1]);
      if (lane == 0 && it + ST < ntiles) {
        fence_proxy_async_smem();
        issue(it + ST);
      }
    }
    if (!(BWD && !PD)) return;
    __syncthreads();  // scalar-lambda reduction below (band warps) -- matched
    return;
  }

  // ============================================================== band warps
  const int band = warp;
  unsigned char* ring = smem + L::OFF_BAND + band * L::B_WARP;
  IO* so0 = reinterpret_cast<IO*>(ring + ST * L::B_STAGE);
  IO* so1 = reinterpret_cast<IO*>(ring + ST * L::B_STAGE + L::OUT);
  double* red = reinterpret_cast<double*>(smem + L::OFF_BAND + nb * L::B_WARP);
  double* redS = red + K * 32;
  uint64_t* bars = b_full[band];
  auto issue = [&](int i) {
    const bool up = i < C;
    const int c = up ? i : 2 * C - 1 - i;
    const int t0 = c * K;
    unsigned char* stg = ring + (i % ST) * L::B_STAGE;
    mbar_arrive_expect_tx(&bars[i % ST], up ? L::B_BYTES_UP : L::B_BYTES_DN);
    tma_load_3d(stg + L::B_OFF_RHS, &p.tm_rhs, (int)bw, t0, band, &bars[i % ST]);
    if (BWD && !up) tma_load_3d(stg + L::B_OFF_DZ, &p.tm_dz, (int)bw, t0, band, &bars[i % ST]);
  };
  if (lane == 0)
    for (int i = 0; i < ST && i < ntiles; ++i) issue(i);
  __syncwarp();
  double* const ck_rhs = (BWD ? p.ck_rhs_b : p.ck_rhs_f) + (long long)band * D * B + b;
  const long long ck_stride = (long long)nb * D * B;
  double v[D];
#pragma unroll
  for (int i = 0; i < D; ++i) v[i] = 0.0;
  int it = 0, fb = 0;
  // ---- up sweep: v_t = b_t - sum_j (M_j + A_{t,j}) v_{t-j}
  for (int c = 0; c < C; ++c, ++it, ++fb) {
    const int s = it % ST;
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const IO* t_rhs = reinterpret_cast<const IO*>(ring + s * L::B_STAGE + L::B_OFF_RHS) + lane;
    const int t0 = c * K;
    if (valid) {
      double* ck = ck_rhs + (long long)c * ck_stride;
#pragma unroll
      for (int i = 0; i < D; ++i) ck[(long long)i * B] = v[i];
    }
    mbar_wait(&fac_full[fb & 1], (uint32_t)((fb >> 1) & 1));
    const unsigned char* F = fbuf0 + (fb & 1) * L::FBUF;
    const double* FA = reinterpret_cast<const double*>(F + L::FB_A) + lane;
    const IO* FW = reinterpret_cast<const IO*>(F + L::FB_W) + lane;
    const int n = min(K, T - t0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k >= n) break;
      const IO wio = FW[k * 32];
      const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, to_f64<IO>(wio));
      double vv = bb;
#pragma unroll
      for (int j = D; j >= 1; --j) {
        vv = fma(-Mj(D, j), v[j - 1], vv);
        vv = fma(-FA[(k * D + j - 1) * 32], v[j - 1], vv);
      }
#pragma unroll
      for (int i = D - 1; i >= 1; --i) v[i] = v[i - 1];
      v[0] = vv;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&fac_empty[fb & 1]);
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue(it + ST);
    }
  }
  // ---- down sweep
  double cA[D][D], zw[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    zw[i] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) cA[i][j] = 0.0;
  }
  double lam_acc = 0.0;
  const int TmDs = TmD;
  for (int c = C - 1; c >= 0; --c, ++it, ++fb) {
    const int s = it % ST;
    mbar_wait(&bars[s], (uint32_t)((it / ST) & 1));
    const unsigned char* stg = ring + s * L::B_STAGE;
    const IO* t_rhs = reinterpret_cast<const IO*>(stg + L::B_OFF_RHS) + lane;
    const IO* t_dz = reinterpret_cast<const IO*>(stg + L::B_OFF_DZ) + lane;
    const int t0 = c * K;
    if (valid) {
      const double* ck = ck_rhs + (long long)c * ck_stride;
#pragma unroll
      for (int i = 0; i < D; ++i) v[i] = ck[(long long)i * B];
    }
    mbar_wait(&fac_full[fb & 1], (uint32_t)((fb >> 1) & 1));
    const unsigned char* F = fbuf0 + (fb & 1) * L::FBUF;
    const double* FA = reinterpret_cast<const double*>(F + L::FB_A) + lane;
    const double* FI = reinterpret_cast<const double*>(F + L::FB_ID) + lane;
    const IO* FW = reinterpret_cast<const IO*>(F + L::FB_W) + lane;
    double q[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const IO wio = FW[k * 32];
      const double bb = rhs_times_w<IO, BWD>(t_rhs[k * 32], wio, to_f64<IO>(wio));
      double vv = bb;
#pragma unroll
      for (int j = D; j >= 1; --j) {
        vv = fma(-Mj(D, j), v[j - 1], vv);
        vv = fma(-FA[(k * D + j - 1) * 32], v[j - 1], vv);
      }
#pragma unroll
      for (int i = D - 1; i >= 1; --i) v[i] = v[i - 1];
      v[0] = vv;
      q[k] = vv * FI[k * 32];  // rows past T: FI = 0 -> q = 0
    }
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      const int t = t0 + k;
      double z = q[k];
#pragma unroll
      for (int j = D; j >= 1; --j) {
        const double a = (k + j < K) ? FA[((k + j) * D + j - 1) * 32] : cA[k + j - K][j - 1];
        z = fma(-Mj(D, j), zw[j - 1], z);
        z = fma(-a, zw[j - 1], z);
      }
      double dz = Cj(D, 0) * z;
#pragma unroll
      for (int j = 1; j <= D; ++j) dz = fma(Cj(D, j), zw[j - 1], dz);
#pragma unroll
      for (int i = D - 1; i >= 1; --i) zw[i] = zw[i - 1];
      zw[0] = z;
      if (!BWD) {
        so0[k * 32 + lane] = from_f64<IO>(z);
        so1[k * 32 + lane] = from_f64<IO>(dz);
      } else {
        const IO wio = FW[k * 32];
        if (sizeof(IO) == 4 && PD) {
          so0[k * 32 + lane] = wio * from_f64<IO>(z);
          so1[k * 32 + lane] = -(from_f64<IO>(dz) * t_dz[k * 32]);
        } else {
          so0[k * 32 + lane] = from_f64<IO>(to_f64<IO>(wio) * z);
          const double g = -dz * to_f64<IO>(t_dz[k * 32]);
          if (PD) so1[k * 32 + lane] = from_f64<IO>(g);
          else if (t < TmDs) lam_acc += g;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) cA[i][j] = FA[(i * D + j) * 32];
    __syncwarp();
    if (lane == 0) mbar_arrive(&fac_empty[fb & 1]);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&p.tm_out0, so0, (int)bw, t0, band);
      if (!BWD) tma_store_3d(&p.tm_out1, so1, (int)bw, t0, band);
      bulk_commit();
    }
    if (BWD && PD) {
      // sum over bands of the staged -(D u_c)(D z_c), fp64 in band order, by the band warps
      named_bar_sync(1, 32 * nb);
      for (int k = band; k < K; k += nb) {
        double acc = 0.0;
        for (int cb = 0; cb < nb; ++cb)
          acc += to_f64<IO>(reinterpret_cast<const IO*>(smem + L::OFF_BAND + cb * L::B_WARP + ST * L::B_STAGE +
                                                        L::OUT)[k * 32 + lane]);
        red[k * 32 + lane] = acc;
      }
      named_bar_sync(1, 32 * nb);
      if (band == 0) {  // round + stage the reduced rows into band 0's so1 (already read), store
        for (int k = 0; k < K; ++k) so1[k * 32 + lane] = from_f64<IO>(red[k * 32 + lane]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&p.tm_out1, so1, (int)bw, t0);
          bulk_commit();
        }
      }
      named_bar_sync(1, 32 * nb);  // so1 tiles / red are reused next chunk
    }
    __syncwarp();
    if (lane == 0 && it + ST < ntiles) {
      fence_proxy_async_smem();
      issue(it + ST);
    }
  }
  if (lane == 0) bulk_wait0();
  if (BWD && !PD) {
    redS[band * 32 + lane] = lam_acc;
    __syncthreads();
    if (band == 0) {
      double acc = 0.0;
      for (int cb = 0; cb < nb; ++cb) acc += redS[cb * 32 + lane];
      if (valid) reinterpret_cast<IO*>(p.out1)[b] = from_f64<IO>(acc);
    }
  }
}

}  // namespace whit
