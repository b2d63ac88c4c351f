// libwhit host side: the C-ABI of include/libwhit.h (validation, workspace
// layout, TMA descriptor encoding, kernel dispatch).  No torch types, no
// exceptions across the boundary, no host synchronisation except
// whit_failures().
#include "libwhit.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "whit_launch.cuh"

#include <nvtx3/nvToolsExt.h>

using whit::Params;

// NVTX range around each compute entry point (tracing: ncu --nvtx / nsys timelines); a no-op without a tool.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#define WHIT_NVTX(name) NvtxRange whit_nvtx_range_(name)

namespace {
thread_local std::string g_err;
}  // namespace

// Shared with the host executor (whit_host.cu); hidden from the ABI.
whit_status whit_detail::fail(whit_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

using whit_detail::fail;

namespace {

// chunk length = TMA tile rows (whit::Tile<IO, d>::K)
int chunk_k(int d) { return d <= 2 ? whit::Tile<float, 2, false>::K : whit::Tile<float, 3, false>::K; }
// rows per chunk of the shared-factor multi-band kernel (MB2Layout::K)
int chunk_k_bands(int d, int nb) {
  if (nb <= 1) return chunk_k(d);
  return d == 1 ? whit::MB2Layout<1, float, true, false>::K
                : d == 2 ? whit::MB2Layout<2, float, true, false>::K : whit::MB2Layout<3, float, true, false>::K;
}
static_assert(whit::Tile<float, 1, false>::K == whit::Tile<double, 2, true>::K &&
                  whit::Tile<float, 3, false>::K == whit::Tile<double, 3, true>::K,
              "chunk length table out of sync with whit::Tile");

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
  size_t off_dz, off_ckfac, off_ckrf, off_ckrb, off_info, off_cnt, off_wbits, off_wflag, off_twflag, total;
};

// Workspace of nb bands x B pixels: D z cache [nb][T-d][B] (I/O dtype), factor
// checkpoints [C][NFAC][B] + forward / backward rhs checkpoints [C][nb][d][B]
// (fp64), info[B], a failure counter.
bool layout(int d, int64_t T, int64_t B, int nb, whit_dtype dt, WsLayout* L, int kk = 0) {
  if (d < 1 || d > 3 || T < d + 1 || B < 1 || nb < 1 || nb > whit::kMaxBands ||
      (dt != WHIT_F32 && dt != WHIT_F64))
    return false;
  const size_t esz = dt == WHIT_F32 ? 4 : 8;
  if (kk == 0) kk = chunk_k_bands(d, nb);
  // checkpoint slots: ceil(T/K) chunks, +2 for the twisted path's two halves (C1 + C2 <= C + 2)
  const int64_t C = (T + kk - 1) / kk + 2;
  const int nfac = d + d * (d - 1) / 2;
  size_t o = 0;
  L->off_dz = o;    o = align256(o + size_t(nb) * size_t(T - d) * size_t(B) * esz);
  L->off_ckfac = o; o = align256(o + size_t(C) * nfac * size_t(B) * 8);
  L->off_ckrf = o;  o = align256(o + size_t(C) * nb * d * size_t(B) * 8);
  L->off_ckrb = o;  o = align256(o + size_t(C) * nb * d * size_t(B) * 8);
  L->off_info = o;  o = align256(o + size_t(B) * 4);
  L->off_cnt = o;   o = align256(o + 8);
  // binary-W detection of the plain forward: the bit plane of W [ceil(T/32)][B] and one flag per warp
  L->off_wbits = o; o = align256(o + size_t((T + 31) / 32) * size_t(B) * 4);
  L->off_wflag = o; o = align256(o + size_t((B + 31) / 32) * 4);
  L->off_twflag = o; o = align256(o + size_t((B + 31) / 32) * 4);  // twisted path: per warp group
  L->total = o;
  return true;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// Map over [depth][rows][inner] (depth = 0: a 2-D [rows][inner] plane), box
// {32, box_rows(, 1)}; out-of-bounds elements (negative or >= rows, >= inner)
// read as zero and are clipped on store.
whit_status encode_map(CUtensorMap* m, const void* ptr, whit_dtype dt, int64_t inner, int64_t rows, int box_rows,
                       int depth = 0) {
  if (!get_encode()) return fail(WHIT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  const size_t esz = dt == WHIT_F32 ? 4 : 8;
  const cuuint32_t rank = depth > 0 ? 3 : 2;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(depth > 0 ? depth : 1)};
  cuuint64_t strides[2] = {cuuint64_t(inner) * esz, cuuint64_t(inner) * esz * cuuint64_t(rows)};
  cuuint32_t box[3] = {32u, cuuint32_t(box_rows), 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, dt == WHIT_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank,
                        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(WHIT_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", int(r));
  return WHIT_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Binary-W detection in the plain forward: on unless WHIT_WDET=0 in the environment (A/B runs).
bool wdet_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("WHIT_WDET");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

// Encoded TMA descriptors of a workspace, keyed by (pointer, dtype, shape, box): a training loop calls
// forward / backward with the same buffers every step, so cuTensorMapEncodeTiled runs once per buffer.
struct MapCache {
  static constexpr int N = 24;
  struct Key {
    const void* ptr;
    int64_t inner, rows;
    int box, depth, dt;
  } key[N];
  CUtensorMap map[N];
  int n = 0, next = 0;
};

struct whit_ws {
  mutable MapCache maps;
  int device;  // CUDA device current at creation (-1: none), made current around encodes/launches
  int d;
  int64_t T, B;
  int nb;      // bands per pixel sharing w, lambda (1 = independent series)
  int kk;      // checkpoint interval / tile rows (chunk_k(d), or 8 on an irregular grid)
  bool irr;    // irregular acquisition grid (NEXT-2): forward must be whit_forward_times
  const void* times;
  const uint32_t* wbits;  // bit-packed W of the last forward (whit_forward_wbits), else NULL
  bool wdet;              // the last forward was the plain float-W forward with binary-W detection on
  bool tw;                // the last forward ran the twisted path (+ its whit_kernel fallback)
  int tw_mode;            // whit_ws_set_twist: -1 auto (WHIT_TWIST / batch size), 0 never, 1 when the shape allows
  int hyb_g1;             // hybrid launch of the last forward: groups [0, g1) sequential, [g1, G) twisted (0: none)
  cudaStream_t aux = nullptr;            // hybrid launch: the twisted part's stream (created on first use)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  whit_dtype dt;
  whit_lambda_mode lm;
  char* buf;
  size_t bytes;
  cudaStream_t stream;
  WsLayout L;
  bool have_fwd;   // a forward ran and its checkpoints are intact (whit_backward may follow)
  bool have_info;  // info[] holds the status of the last forward or posterior variance (count_failures also
                   // counts the nonzero per-warp binary-W flags for whit_wbits_detected)
  const void* w;
  const void* lam;
  const void* z;
};

namespace {

whit_status wmap(const whit_ws* ws, CUtensorMap* m, const void* ptr, whit_dtype dt, int64_t inner, int64_t rows,
                 int box_rows, int depth = 0) {
  MapCache& c = ws->maps;
  const MapCache::Key k{ptr, inner, rows, box_rows, depth, int(dt)};
  for (int i = 0; i < c.n; ++i) {
    const MapCache::Key& e = c.key[i];
    if (e.ptr == k.ptr && e.inner == k.inner && e.rows == k.rows && e.box == k.box && e.depth == k.depth &&
        e.dt == k.dt) {
      *m = c.map[i];
      return WHIT_OK;
    }
  }
  const whit_status st = encode_map(m, ptr, dt, inner, rows, box_rows, depth);
  if (st != WHIT_OK) return st;
  const int slot = c.n < MapCache::N ? c.n++ : (c.next++ % MapCache::N);
  c.key[slot] = k;
  c.map[slot] = *m;
  return WHIT_OK;
}

// Makes the workspace's device current on the calling thread (autograd runs
// backward on its own device thread, where no context is bound yet) and
// restores the caller's device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (dev < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Every forward records, in one place, what its backward will consume: the weights it read (float
// plane or bit-packed), lambda, z, the dates of an irregular grid.  (A stale field -- e.g. the bit
// plane of an earlier whit_forward_wbits -- would silently steer the next backward.)
void mark_forward(whit_ws* ws, const void* w, const void* lam, const void* z, const uint32_t* wbits,
                  const void* times, bool wdet = false, bool tw = false, int hyb_g1 = 0) {
  ws->wdet = wdet;
  ws->tw = tw;
  ws->hyb_g1 = hyb_g1;
  ws->have_fwd = true;
  ws->have_info = true;
  ws->w = w;
  ws->lam = lam;
  ws->z = z;
  ws->wbits = wbits;
  ws->times = times;
}

using whit_detail::kSmemBudget;
using whit_detail::launch;
using whit_detail::launch_irr;
using whit_detail::launch_mb2;
using whit_detail::launch_var;

// Largest band count whose shared-factor CTA (whit_mb2_kernel) fits shared memory, for every
// (d, lambda mode, direction) of this dtype.
template <typename IO, int D, bool PD, bool BWD>
constexpr int max_bands_mb2() {
  int m = 0;
  for (int nb = 1; nb <= whit::kMaxBands; ++nb)
    if (whit::MB2Layout<D, IO, PD, BWD>::smem(nb) <= kSmemBudget &&
        whit::MB2Layout<D, IO, PD, BWD, true>::smem(nb) <= kSmemBudget)
      m = nb;
  return m;
}
template <typename IO, int D>
constexpr int max_bands_d() {
  const int v[] = {max_bands_mb2<IO, D, true, true>(), max_bands_mb2<IO, D, true, false>(),
                   max_bands_mb2<IO, D, false, true>(), max_bands_mb2<IO, D, false, false>()};
  int m = whit::kMaxBands;
  for (int x : v) m = x < m ? x : m;
  return m;
}
template <typename IO>
constexpr int max_bands_io() {
  const int v[] = {max_bands_d<IO, 1>(), max_bands_d<IO, 2>(), max_bands_d<IO, 3>()};
  int m = whit::kMaxBands;
  for (int x : v) m = x < m ? x : m;
  return m;
}
static_assert(max_bands_io<float>() == whit::kMaxBands && max_bands_io<double>() == whit::kMaxBands,
              "every multi-band kernel fits kMaxBands bands in one CTA");
int max_bands(whit_dtype dt) { return dt == WHIT_F32 ? max_bands_io<float>() : max_bands_io<double>(); }

template <typename IO, bool PD, bool BWD, bool MB>
whit_status dispatch_d(int d, const Params& p, cudaStream_t s) {
  if constexpr (MB) {
    switch (d) {
      case 1: return launch_mb2<1, IO, PD, BWD>(p, s);
      case 2: return launch_mb2<2, IO, PD, BWD>(p, s);
      case 3: return launch_mb2<3, IO, PD, BWD>(p, s);
    }
    return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
  } else {
  switch (d) {
    case 1: return launch<1, IO, PD, BWD>(p, s);
    case 2: return launch<2, IO, PD, BWD>(p, s);
    case 3: return launch<3, IO, PD, BWD>(p, s);
  }
  return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
  }
}

template <typename IO, bool BWD, bool MB>
whit_status dispatch_pd(const whit_ws* ws, const Params& p) {
  return ws->lm == WHIT_LAMBDA_PER_DATE ? dispatch_d<IO, true, BWD, MB>(ws->d, p, ws->stream)
                                        : dispatch_d<IO, false, BWD, MB>(ws->d, p, ws->stream);
}

template <typename IO, bool PD, bool BWD>
whit_status dispatch_wb_d(int d, const Params& p, cudaStream_t s) {
  switch (d) {
    case 1: return launch<1, IO, PD, BWD, false, true>(p, s);
    case 2: return launch<2, IO, PD, BWD, false, true>(p, s);
    case 3: return launch<3, IO, PD, BWD, false, true>(p, s);
  }
  return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
}

template <bool BWD>
whit_status dispatch_wb(const whit_ws* ws, const Params& p) {
  const bool pd = ws->lm == WHIT_LAMBDA_PER_DATE;
  if (ws->dt == WHIT_F32)
    return pd ? dispatch_wb_d<float, true, BWD>(ws->d, p, ws->stream) : dispatch_wb_d<float, false, BWD>(ws->d, p, ws->stream);
  return pd ? dispatch_wb_d<double, true, BWD>(ws->d, p, ws->stream) : dispatch_wb_d<double, false, BWD>(ws->d, p, ws->stream);
}

template <bool BWD>
whit_status dispatch(const whit_ws* ws, const Params& p) {
  const bool mb = ws->nb > 1;
  if (ws->dt == WHIT_F32)
    return mb ? dispatch_pd<float, BWD, true>(ws, p) : dispatch_pd<float, BWD, false>(ws, p);
  return mb ? dispatch_pd<double, BWD, true>(ws, p) : dispatch_pd<double, BWD, false>(ws, p);
}

template <typename IO, bool PD>
whit_status dispatch_loss_d(int d, const Params& p, cudaStream_t s) {
  switch (d) {
    case 1: return launch<1, IO, PD, false, true>(p, s);
    case 2: return launch<2, IO, PD, false, true>(p, s);
    case 3: return launch<3, IO, PD, false, true>(p, s);
  }
  return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
}

template <typename IO, bool PD>
whit_status dispatch_var_d(int d, const Params& p, cudaStream_t s) {
  switch (d) {
    case 1: return launch_var<1, IO, PD>(p, s);
    case 2: return launch_var<2, IO, PD>(p, s);
    case 3: return launch_var<3, IO, PD>(p, s);
  }
  return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
}

// Fill the tensor maps and plain pointers common to both directions.
whit_status fill_params(const whit_ws* ws, Params* p, const void* rhs, const void* w, const void* lam) {
  std::memset(p, 0, sizeof *p);
  const int d = ws->d;
  const int kK = ws->kk;
  whit_status st;
  if ((st = wmap(ws, &p->tm_rhs, rhs, ws->dt, ws->B, ws->T, kK, ws->nb)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p->tm_w, w, ws->dt, ws->B, ws->T, kK)) != WHIT_OK) return st;
  if (ws->lm == WHIT_LAMBDA_PER_DATE) {
    if ((st = wmap(ws, &p->tm_lam_up, lam, ws->dt, ws->B, ws->T - d, kK)) != WHIT_OK) return st;
    if ((st = wmap(ws, &p->tm_lam_dn, lam, ws->dt, ws->B, ws->T - d, kK + d)) != WHIT_OK) return st;
    p->lam_plane = lam;
  } else {
    p->lam_scalar = lam;
  }
  p->ck_fac = reinterpret_cast<double*>(ws->buf + ws->L.off_ckfac);
  p->ck_rhs_f = reinterpret_cast<double*>(ws->buf + ws->L.off_ckrf);
  p->ck_rhs_b = reinterpret_cast<double*>(ws->buf + ws->L.off_ckrb);
  p->info = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_info);
  p->B = ws->B;
  p->T = int(ws->T);
  p->C = int((ws->T + kK - 1) / kK);
  p->nb = ws->nb;
  return WHIT_OK;
}

template <typename IO, bool PD, bool BWD>
whit_status dispatch_irr_d(int d, bool mb, const Params& p, cudaStream_t s) {
  if (mb) {  // C > 1 bands on the uneven grid: shared-factor kernel with the dates stencils
    switch (d) {
      case 1: return launch_mb2<1, IO, PD, BWD, true>(p, s);
      case 2: return launch_mb2<2, IO, PD, BWD, true>(p, s);
      case 3: return launch_mb2<3, IO, PD, BWD, true>(p, s);
    }
    return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
  }
  switch (d) {
    case 1: return launch_irr<1, IO, PD, BWD>(p, s);
    case 2: return launch_irr<2, IO, PD, BWD>(p, s);
    case 3: return launch_irr<3, IO, PD, BWD>(p, s);
  }
  return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
}

template <bool BWD>
whit_status dispatch_irr(const whit_ws* ws, const Params& p) {
  const bool pd = ws->lm == WHIT_LAMBDA_PER_DATE, mb = ws->nb > 1;
  if (ws->dt == WHIT_F32)
    return pd ? dispatch_irr_d<float, true, BWD>(ws->d, mb, p, ws->stream)
              : dispatch_irr_d<float, false, BWD>(ws->d, mb, p, ws->stream);
  return pd ? dispatch_irr_d<double, true, BWD>(ws->d, mb, p, ws->stream)
            : dispatch_irr_d<double, false, BWD>(ws->d, mb, p, ws->stream);
}

// ---------------------------------------------------------------- twisted path (whit_twist.cuh)
// Split row m: a multiple of K near the middle, so the top half runs m + d rows and the bottom T - m.
int tw_split(const whit_ws* ws) { return ws->kk * int((ws->T - ws->d) / (2 * ws->kk)); }

// Small batches take the twisted path: a warp group's 32 series are split in time between two warps, which
// halves the per-series latency and doubles the warps in flight.  It wins while its 2 x B/32 warps fit one
// wave of 12 warps on each of the 148 SMs -- scalar lambda: B <= 28,416 (8,192: 1.0 -> 1.9x); per-date lambda,
// whose sequential kernel fills that wave better: B <= 24,864 (at 28,416 the sequential kernel is 5 % faster);
// beyond that a twisted tail wave costs more than it saves (profiles/r2_twist_tune.log).
// WHIT_TWIST=0 never, =1 whenever the shape allows; whit_ws_set_twist overrides both per workspace.
bool tw_pick(const whit_ws* ws) {
  if (ws->nb != 1 || ws->irr) return false;
  const int m = tw_split(ws);
  if (m < ws->kk || ws->T - m - ws->d < ws->kk) return false;  // each half needs a chunk beyond S
  static const int env_mode = [] {
    const char* e = std::getenv("WHIT_TWIST");
    return e ? (e[0] == '0' ? 0 : e[0] == '1' ? 1 : 2) : 2;
  }();
  const int mode = ws->tw_mode == 2 ? 0 : ws->tw_mode >= 0 ? ws->tw_mode : env_mode;
  if (mode == 0) return false;
  if (mode == 1) return true;
  return ws->B <= 148LL * 12 * (ws->lm == WHIT_LAMBDA_PER_DATE ? 14 : 16);
}

// Hybrid launch for batches just past one wave of whit_kernel (1,776 < G <= 2,400 groups of 32, e.g. homo's
// 2,048): the first g1 groups run the sequential kernel (its wave) while the remaining groups run twisted
// on a second stream, filling the slots the first wave leaves and finishing the tail in half the latency
// (homo 22.6 -> 23.9 M series/s in the two-stream probe, tools/kdev/hybrid_probe.py).  Auto mode only.
// The sequential part's group count (even: two groups per twisted CTA), by lambda mode -- re-tuned once the
// twisted tail ran the 255-register build (profiles/r2_hybrid_g1.log, M series/s at 1,632 -> here): homo
// 65,536 26.0 -> 26.7 (1,728), hetero-shaped 65,536 25.4 -> 25.5 (1,504).
int hyb_g1_of(const whit_ws* ws) { return ws->lm == WHIT_LAMBDA_PER_DATE ? 1504 : 1728; }
int hyb_pick(const whit_ws* ws) {
  if (ws->nb != 1 || ws->irr) return 0;
  if (ws->tw_mode == 2) {  // forced (tests): whenever there are groups beyond the split
    const int m = tw_split(ws), g1 = hyb_g1_of(ws);
    return (m >= ws->kk && ws->T - m - ws->d >= ws->kk && (ws->B + 31) / 32 > g1) ? g1 : 0;
  }
  if (ws->tw_mode >= 0) return 0;
  const char* e = std::getenv("WHIT_TWIST");
  if (e && (e[0] == '0' || e[0] == '1')) return 0;
  const char* h = std::getenv("WHIT_HYBRID");
  if (h && h[0] == '0') return 0;
  const int hmax = (h && h[0] >= '2' && h[0] <= '9') ? 1 << 30 : 2400;  // WHIT_HYBRID=2: any G > 1,776 (A/B)
  const int m = tw_split(ws);
  if (m < ws->kk || ws->T - m - ws->d < ws->kk) return 0;
  const long long G = (ws->B + 31) / 32;
  static const int g1_env = [] {  // WHIT_HYB_G1: the sequential part's group count (dev A/B; even)
    const char* v = std::getenv("WHIT_HYB_G1");
    const int x = v ? std::atoi(v) : 0;
    return (x >= 2 && x % 2 == 0) ? x : 0;
  }();
  const int g1 = g1_env ? g1_env : hyb_g1_of(ws);
  return (G > 148 * 12 && G <= hmax && G > g1) ? g1 : 0;
}

whit_status hyb_streams(whit_ws* ws) {
  if (ws->aux) return WHIT_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&ws->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ws->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ws->ev_join, cudaEventDisableTiming);
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "hybrid launch streams: %s", cudaGetErrorString(e));
  return WHIT_OK;
}

// Tensor maps of the two halves (2-D, box K rows; lambda box K + d): top planes cut at row m, bottom planes
// based at row m.  rhs: y (forward) / grad_z (backward); out0: z / grad_y; out1: the D z cache (forward) /
// grad_lambda per date (backward); dz: the D z cache (backward).
whit_status tw_fill(const whit_ws* ws, Params* p, const void* rhs, const void* w, const void* lam, void* out0,
                    void* out1, const void* dz, bool bwd) {
  std::memset(p, 0, sizeof *p);
  const int d = ws->d, K = ws->kk, m = tw_split(ws);
  const int64_t T = ws->T, B = ws->B;
  const size_t esz = ws->dt == WHIT_F32 ? 4 : 8;
  const size_t off = size_t(m) * size_t(B) * esz;  // byte offset of row m in a [rows][B] plane
  auto at = [&](const void* ptr) { return static_cast<const char*>(ptr) + off; };
  const bool pd = ws->lm == WHIT_LAMBDA_PER_DATE;
  whit_status st;
  if ((st = wmap(ws, &p->tm_rhs, rhs, ws->dt, B, m, K)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p->tm_w, w, ws->dt, B, m, K)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p->tmb_rhs, at(rhs), ws->dt, B, T - m, K)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p->tmb_w, at(w), ws->dt, B, T - m, K)) != WHIT_OK) return st;
  if (pd) {
    if ((st = wmap(ws, &p->tm_lam_dn, lam, ws->dt, B, m, K + d)) != WHIT_OK) return st;
    if ((st = wmap(ws, &p->tmb_lam, at(lam), ws->dt, B, T - d - m, K + d)) != WHIT_OK) return st;
  } else {
    p->lam_scalar = lam;
  }
  if ((st = wmap(ws, &p->tm_out0, out0, ws->dt, B, m, K)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p->tmb_out0, at(out0), ws->dt, B, T - m, K)) != WHIT_OK) return st;
  if (!bwd || pd) {
    if ((st = wmap(ws, &p->tm_out1, out1, ws->dt, B, m, K)) != WHIT_OK) return st;
    if ((st = wmap(ws, &p->tmb_out1, at(out1), ws->dt, B, T - d - m, K)) != WHIT_OK) return st;
  }
  if (bwd) {
    if ((st = wmap(ws, &p->tm_dz, dz, ws->dt, B, m, K)) != WHIT_OK) return st;
    if ((st = wmap(ws, &p->tmb_dz, at(dz), ws->dt, B, T - d - m, K)) != WHIT_OK) return st;
  }
  p->out0 = out0;  // (direct stores of the chunks at S)
  p->out1 = out1;  // D z / grad_lambda plane, or the scalar lambda gradient [B] (backward)
  p->ck_fac = reinterpret_cast<double*>(ws->buf + ws->L.off_ckfac);
  p->ck_rhs_f = reinterpret_cast<double*>(ws->buf + ws->L.off_ckrf);
  p->ck_rhs_b = reinterpret_cast<double*>(ws->buf + ws->L.off_ckrb);
  p->info = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_info);
  p->twflag = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_twflag);
  p->B = B;
  p->T = int(T);
  p->C = int((T + K - 1) / K);
  p->nb = 1;
  p->tw_m = m;
  p->tw_C1 = m / K + 1;
  p->tw_C2 = int((T - m + K - 1) / K);
  return WHIT_OK;
}

template <typename IO, bool PD, bool BWD, bool HIREG>
whit_status dispatch_tw_d(int d, const Params& p, cudaStream_t s) {
  switch (d) {
    case 1: return whit_detail::launch_tw<1, IO, PD, BWD, HIREG>(p, s);
    case 2: return whit_detail::launch_tw<2, IO, PD, BWD, HIREG>(p, s);
    case 3: return whit_detail::launch_tw<3, IO, PD, BWD, HIREG>(p, s);
  }
  return fail(WHIT_ERR_ARG, "d must be 1, 2 or 3");
}

// Twisted launches of at most one wave at 8 warps/SM (148 x 4 warp pairs = 592 groups of 32 series) take the
// 255-register build: no spills, and the lower occupancy costs nothing there (homo-shaped 8,192 series:
// 11.9 -> 13.8 M series/s, 16,384: 20.3 -> 23.6 M; at 24,576 the 168-register build is faster, 23.4 vs 18.8).
constexpr long long kTwHiregGroups = 148LL * 4;

template <bool BWD, bool HIREG>
whit_status dispatch_tw_r(const whit_ws* ws, const Params& p) {
  const bool pd = ws->lm == WHIT_LAMBDA_PER_DATE;
  if (ws->dt == WHIT_F32)
    return pd ? dispatch_tw_d<float, true, BWD, HIREG>(ws->d, p, ws->stream)
              : dispatch_tw_d<float, false, BWD, HIREG>(ws->d, p, ws->stream);
  return pd ? dispatch_tw_d<double, true, BWD, HIREG>(ws->d, p, ws->stream)
            : dispatch_tw_d<double, false, BWD, HIREG>(ws->d, p, ws->stream);
}

template <bool BWD>
whit_status dispatch_tw(const whit_ws* ws, const Params& p) {
  const long long groups = (ws->B + 31) / 32 - 2LL * p.tw_cta0;  // (hybrid: the groups past the sequential part)
  return groups <= kTwHiregGroups ? dispatch_tw_r<BWD, true>(ws, p) : dispatch_tw_r<BWD, false>(ws, p);
}

}  // namespace

extern "C" {

int whit_version(void) { return LIBWHIT_VERSION; }

const char* whit_status_string(whit_status s) {
  switch (s) {
    case WHIT_OK: return "WHIT_OK";
    case WHIT_ERR_ARG: return "WHIT_ERR_ARG";
    case WHIT_ERR_SHAPE: return "WHIT_ERR_SHAPE";
    case WHIT_ERR_ALIGN: return "WHIT_ERR_ALIGN";
    case WHIT_ERR_WS: return "WHIT_ERR_WS";
    case WHIT_ERR_CUDA: return "WHIT_ERR_CUDA";
    case WHIT_ERR_STATE: return "WHIT_ERR_STATE";
  }
  return "WHIT_UNKNOWN_STATUS";
}

const char* whit_last_error(void) { return g_err.c_str(); }

size_t whit_ws_bytes_bands(int d, int64_t T, int64_t B, int C, whit_dtype dtype, whit_lambda_mode lambda_mode) {
  WsLayout L;
  if (lambda_mode != WHIT_LAMBDA_SCALAR && lambda_mode != WHIT_LAMBDA_PER_DATE) return 0;
  if (!layout(d, T, B, C, dtype, &L)) return 0;
  return L.total;
}

size_t whit_ws_bytes(int d, int64_t T, int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode) {
  return whit_ws_bytes_bands(d, T, B, 1, dtype, lambda_mode);
}

static whit_status ws_create(whit_ws** out, int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                             whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes, void* cuda_stream, bool irr);

whit_status whit_ws_create_bands(whit_ws** out, int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                                 whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes, void* cuda_stream) {
  return ws_create(out, d, T, B, C, dtype, lambda_mode, dev_buf, dev_bytes, cuda_stream, false);
}

size_t whit_ws_bytes_times_bands(int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                                 whit_lambda_mode lambda_mode) {
  WsLayout L;
  if (lambda_mode != WHIT_LAMBDA_SCALAR && lambda_mode != WHIT_LAMBDA_PER_DATE) return 0;
  if (!layout(d, T, B, C, dtype, &L, 8)) return 0;
  return L.total;
}

size_t whit_ws_bytes_times(int d, int64_t T, int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode) {
  return whit_ws_bytes_times_bands(d, T, B, 1, dtype, lambda_mode);
}

whit_status whit_ws_create_times_bands(whit_ws** out, int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                                       whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes,
                                       void* cuda_stream) {
  return ws_create(out, d, T, B, C, dtype, lambda_mode, dev_buf, dev_bytes, cuda_stream, true);
}

whit_status whit_ws_create_times(whit_ws** out, int d, int64_t T, int64_t B, whit_dtype dtype,
                                 whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes, void* cuda_stream) {
  return ws_create(out, d, T, B, 1, dtype, lambda_mode, dev_buf, dev_bytes, cuda_stream, true);
}

static whit_status ws_create(whit_ws** out, int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                             whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes, void* cuda_stream,
                             bool irr) {
  if (!out) return fail(WHIT_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (d < 1 || d > 3) return fail(WHIT_ERR_ARG, "d = %d not in {1,2,3}", d);
  if (dtype != WHIT_F32 && dtype != WHIT_F64) return fail(WHIT_ERR_ARG, "bad dtype %d", int(dtype));
  if (C < 1 || C > max_bands(dtype))
    return fail(WHIT_ERR_ARG, "bands C = %d not in [1, %d] for this dtype", C, max_bands(dtype));
  if (lambda_mode != WHIT_LAMBDA_SCALAR && lambda_mode != WHIT_LAMBDA_PER_DATE)
    return fail(WHIT_ERR_ARG, "bad lambda mode %d", int(lambda_mode));
  if (T < d + 1) return fail(WHIT_ERR_SHAPE, "T = %lld < d + 1", (long long)T);
  if (T > (int64_t(1) << 30)) return fail(WHIT_ERR_SHAPE, "T = %lld too large", (long long)T);
  if (B < 1 || B >= (int64_t(1) << 31)) return fail(WHIT_ERR_SHAPE, "B = %lld out of range [1, 2^31)", (long long)B);
  if (B % (dtype == WHIT_F32 ? 4 : 2) != 0)
    return fail(WHIT_ERR_ALIGN, "B = %lld must be a multiple of %d (16-B row stride)", (long long)B,
                dtype == WHIT_F32 ? 4 : 2);
  WsLayout L;
  layout(d, T, B, C, dtype, &L, irr ? 8 : 0);
  if (!dev_buf) return fail(WHIT_ERR_WS, "workspace buffer is NULL");
  if (reinterpret_cast<uintptr_t>(dev_buf) & 255u) return fail(WHIT_ERR_ALIGN, "workspace buffer not 256-B aligned");
  if (dev_bytes < L.total)
    return fail(WHIT_ERR_WS, "workspace %zu bytes < required %zu", dev_bytes, L.total);
  whit_ws* ws = new (std::nothrow) whit_ws;
  if (!ws) return fail(WHIT_ERR_ARG, "host allocation failed");
  ws->d = d; ws->T = T; ws->B = B; ws->nb = C; ws->dt = dtype; ws->lm = lambda_mode;
  ws->irr = irr; ws->kk = irr ? 8 : chunk_k_bands(d, C); ws->times = nullptr; ws->wbits = nullptr;
  ws->buf = static_cast<char*>(dev_buf); ws->bytes = dev_bytes;
  ws->stream = static_cast<cudaStream_t>(cuda_stream);
  ws->L = L;
  ws->have_fwd = false; ws->have_info = false; ws->wdet = false; ws->tw = false; ws->tw_mode = -1; ws->hyb_g1 = 0;
  ws->w = ws->lam = ws->z = nullptr;
  ws->device = -1;
  int dev = -1;
  if (cudaGetDevice(&dev) == cudaSuccess) ws->device = dev;
  cudaGetLastError();  // creation is host-only: a missing GPU is not an error here
  *out = ws;
  return WHIT_OK;
}

whit_status whit_ws_create(whit_ws** out, int d, int64_t T, int64_t B, whit_dtype dtype,
                           whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes, void* cuda_stream) {
  return whit_ws_create_bands(out, d, T, B, 1, dtype, lambda_mode, dev_buf, dev_bytes, cuda_stream);
}

whit_status whit_ws_set_stream(whit_ws* ws, void* cuda_stream) {
  if (!ws) return fail(WHIT_ERR_ARG, "ws is NULL");
  ws->stream = static_cast<cudaStream_t>(cuda_stream);
  return WHIT_OK;
}

void whit_ws_destroy(whit_ws* ws) {
  if (!ws) return;
  if (ws->aux) {
    DeviceGuard guard(ws->device);
    cudaStreamDestroy(ws->aux);
    cudaEventDestroy(ws->ev_fork);
    cudaEventDestroy(ws->ev_join);
  }
  delete ws;
}

whit_status whit_forward_bands(const void* y, const void* w, const void* lambda, int d, int64_t T, int64_t B, int C,
                               void* z, whit_ws* ws) {
  WHIT_NVTX("whit_forward_bands");
  if (!ws) return fail(WHIT_ERR_ARG, "factor_ws is NULL");
  if (ws->irr) return fail(WHIT_ERR_STATE, "irregular-grid workspace: use whit_forward_times");
  if (!y || !w || !lambda || !z) return fail(WHIT_ERR_ARG, "NULL data pointer");
  if (d != ws->d || T != ws->T || B != ws->B || C != ws->nb)
    return fail(WHIT_ERR_SHAPE, "(d,T,B,C) = (%d,%lld,%lld,%d) != workspace (%d,%lld,%lld,%d)", d, (long long)T,
                (long long)B, C, ws->d, (long long)ws->T, (long long)ws->B, ws->nb);
  if (!aligned16(y) || !aligned16(w) || !aligned16(lambda) || !aligned16(z))
    return fail(WHIT_ERR_ALIGN, "data pointers must be 16-B aligned");
  if (z == y || z == w || z == lambda) return fail(WHIT_ERR_ARG, "z aliases an input");
  DeviceGuard guard(ws->device);
  if (!guard.ok) return fail(WHIT_ERR_CUDA, "cudaSetDevice(%d) failed", ws->device);
  Params p;
  whit_status st = fill_params(ws, &p, y, w, lambda);
  if (st != WHIT_OK) return st;
  const int kK = ws->kk;
  p.out0 = z;
  p.out1 = ws->buf + ws->L.off_dz;
  if ((st = wmap(ws, &p.tm_out0, z, ws->dt, B, T, kK, C)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_out1, ws->buf + ws->L.off_dz, ws->dt, B, T - d, kK, C)) != WHIT_OK) return st;
  if (const int g1 = C == 1 ? hyb_pick(ws) : 0) {
    // hybrid: groups [0, g1) by whit_kernel on the workspace stream (binary-W detection on), groups [g1, G) by
    // the twisted kernel + its whit_kernel fallback on the auxiliary stream, forked and joined by events
    if ((st = hyb_streams(ws)) != WHIT_OK) return st;
    Params pt;
    if ((st = tw_fill(ws, &pt, y, w, lambda, z, ws->buf + ws->L.off_dz, nullptr, false)) != WHIT_OK) return st;
    pt.tw_cta0 = g1 / 2;
    const bool wdet = wdet_enabled();
    Params ps = p;
    ps.g_hi = g1;
    if (wdet) {
      ps.wbits_out = reinterpret_cast<uint32_t*>(ws->buf + ws->L.off_wbits);
      ps.wbits = ps.wbits_out;
      ps.wflag = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_wflag);
    }
    p.twflag = pt.twflag;  // the fallback: whit_kernel over groups [g1, G) the twisted kernel handed back
    p.tw_filter = 1;
    ws->have_fwd = false;
    cudaStream_t main = ws->stream;
    cudaError_t e = cudaEventRecord(ws->ev_fork, main);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ws->aux, ws->ev_fork, 0);
    const long long G = (B + 31) / 32;
    if (e == cudaSuccess)  // groups [0, g1) count as solved for the fallback's filter; no stale W flags above g1
      e = cudaMemsetAsync(pt.twflag, 0x01, size_t(g1) * 4, ws->aux);
    if (e == cudaSuccess)
      e = cudaMemsetAsync(ws->buf + ws->L.off_wflag + size_t(g1) * 4, 0, size_t(G - g1) * 4, ws->aux);
    if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "hybrid fork: %s", cudaGetErrorString(e));
    st = dispatch<false>(ws, ps);
    ws->stream = ws->aux;
    if (st == WHIT_OK) st = dispatch_tw<false>(ws, pt);
    if (st == WHIT_OK) st = dispatch<false>(ws, p);
    ws->stream = main;
    // join even when a launch on the auxiliary stream failed: nothing it enqueued may outlive the call unordered
    e = cudaEventRecord(ws->ev_join, ws->aux);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(main, ws->ev_join, 0);
    if (st != WHIT_OK) return st;
    if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "hybrid join: %s", cudaGetErrorString(e));
    mark_forward(ws, w, lambda, z, nullptr, nullptr, wdet, true, g1);
    return WHIT_OK;
  }
  if (C == 1 && tw_pick(ws)) {
    // twisted kernel, then whit_kernel for the warp groups it handed back (twflag = 0)
    Params pt;
    if ((st = tw_fill(ws, &pt, y, w, lambda, z, ws->buf + ws->L.off_dz, nullptr, false)) != WHIT_OK) return st;
    ws->have_fwd = false;
    if ((st = dispatch_tw<false>(ws, pt)) != WHIT_OK) return st;
    p.twflag = pt.twflag;
    p.tw_filter = 1;
    if ((st = dispatch<false>(ws, p)) != WHIT_OK) return st;
    mark_forward(ws, w, lambda, z, nullptr, nullptr, false, true);
    return WHIT_OK;
  }
  const bool wdet = C == 1 && wdet_enabled();
  if (wdet) {
    p.wbits_out = reinterpret_cast<uint32_t*>(ws->buf + ws->L.off_wbits);
    p.wbits = p.wbits_out;
    p.wflag = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_wflag);
  }
  ws->have_fwd = false;
  st = dispatch<false>(ws, p);
  if (st != WHIT_OK) return st;
  mark_forward(ws, w, lambda, z, nullptr, nullptr, wdet);
  return WHIT_OK;
}

whit_status whit_forward_wbits(const void* y, const uint32_t* wbits, const void* lambda, int d, int64_t T, int64_t B,
                               void* z, whit_ws* ws) {
  WHIT_NVTX("whit_forward_wbits");
  if (!ws) return fail(WHIT_ERR_ARG, "factor_ws is NULL");
  if (ws->irr || ws->nb != 1) return fail(WHIT_ERR_STATE, "bit-packed W needs a single-band daily-grid workspace");
  if (!y || !wbits || !lambda || !z) return fail(WHIT_ERR_ARG, "NULL data pointer");
  if (d != ws->d || T != ws->T || B != ws->B)
    return fail(WHIT_ERR_SHAPE, "(d,T,B) = (%d,%lld,%lld) != workspace (%d,%lld,%lld)", d, (long long)T,
                (long long)B, ws->d, (long long)ws->T, (long long)ws->B);
  if (!aligned16(y) || !aligned16(wbits) || !aligned16(lambda) || !aligned16(z))
    return fail(WHIT_ERR_ALIGN, "data pointers must be 16-B aligned");
  if (z == y || z == (const void*)wbits || z == lambda) return fail(WHIT_ERR_ARG, "z aliases an input");
  DeviceGuard guard(ws->device);
  if (!guard.ok) return fail(WHIT_ERR_CUDA, "cudaSetDevice(%d) failed", ws->device);
  Params p;
  whit_status st = fill_params(ws, &p, y, y /* w map unused */, lambda);
  if (st != WHIT_OK) return st;
  p.wbits = wbits;
  const int kK = ws->kk;
  if ((st = wmap(ws, &p.tm_out0, z, ws->dt, B, T, kK, 1)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_out1, ws->buf + ws->L.off_dz, ws->dt, B, T - d, kK, 1)) != WHIT_OK) return st;
  ws->have_fwd = false;
  st = dispatch_wb<false>(ws, p);
  if (st != WHIT_OK) return st;
  mark_forward(ws, wbits, lambda, z, wbits, nullptr);
  return WHIT_OK;
}

whit_status whit_pack_mask(const void* w, int64_t T, int64_t B, whit_dtype dtype, uint32_t* bits, void* cuda_stream) {
  if (!w || !bits) return fail(WHIT_ERR_ARG, "NULL pointer");
  if (dtype != WHIT_F32 && dtype != WHIT_F64) return fail(WHIT_ERR_ARG, "bad dtype");
  if (T < 1 || B < 1) return fail(WHIT_ERR_SHAPE, "bad T / B");
  const long long rows = (T + 31) / 32;
  if (rows > 65535) return fail(WHIT_ERR_SHAPE, "T too large for the packing grid");
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  dim3 grid((unsigned)((B + 255) / 256), (unsigned)rows);
  if (dtype == WHIT_F32)
    whit::pack_mask<float><<<grid, 256, 0, s>>>(static_cast<const float*>(w), T, B, bits);
  else
    whit::pack_mask<double><<<grid, 256, 0, s>>>(static_cast<const double*>(w), T, B, bits);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "pack launch: %s", cudaGetErrorString(e));
  return WHIT_OK;
}

whit_status whit_forward_times_bands(const void* y, const void* w, const void* lambda, const void* times, int d,
                                     int64_t T, int64_t B, int C, void* z, whit_ws* ws) {
  WHIT_NVTX("whit_forward_times_bands");
  if (!ws) return fail(WHIT_ERR_ARG, "factor_ws is NULL");
  if (!ws->irr) return fail(WHIT_ERR_STATE, "workspace not created by whit_ws_create_times(_bands)");
  if (!y || !w || !lambda || !times || !z) return fail(WHIT_ERR_ARG, "NULL data pointer");
  if (d != ws->d || T != ws->T || B != ws->B || C != ws->nb)
    return fail(WHIT_ERR_SHAPE, "(d,T,B,C) = (%d,%lld,%lld,%d) != workspace (%d,%lld,%lld,%d)", d, (long long)T,
                (long long)B, C, ws->d, (long long)ws->T, (long long)ws->B, ws->nb);
  if (!aligned16(y) || !aligned16(w) || !aligned16(lambda) || !aligned16(times) || !aligned16(z))
    return fail(WHIT_ERR_ALIGN, "data pointers must be 16-B aligned");
  if (z == y || z == w || z == lambda || z == times) return fail(WHIT_ERR_ARG, "z aliases an input");
  DeviceGuard guard(ws->device);
  if (!guard.ok) return fail(WHIT_ERR_CUDA, "cudaSetDevice(%d) failed", ws->device);
  Params p;
  whit_status st = fill_params(ws, &p, y, w, lambda);
  if (st != WHIT_OK) return st;
  const int kK = ws->kk;
  p.out0 = z;  // multi-band kernel: direct stores
  p.out1 = ws->buf + ws->L.off_dz;
  if ((st = wmap(ws, &p.tm_out0, z, ws->dt, B, T, kK, C)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_out1, ws->buf + ws->L.off_dz, ws->dt, B, T - d, kK, C)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_lw, times, ws->dt, B, T, kK + 2 * d)) != WHIT_OK) return st;
  ws->have_fwd = false;
  st = dispatch_irr<false>(ws, p);
  if (st != WHIT_OK) return st;
  mark_forward(ws, w, lambda, z, nullptr, times);
  return WHIT_OK;
}

whit_status whit_forward_times(const void* y, const void* w, const void* lambda, const void* times, int d, int64_t T,
                               int64_t B, void* z, whit_ws* ws) {
  return whit_forward_times_bands(y, w, lambda, times, d, T, B, 1, z, ws);
}

whit_status whit_forward_mse(const void* y, const void* w, const void* lambda, const void* loss_w, int d, int64_t T,
                             int64_t B, void* z, void* grad_z, void* loss, whit_ws* ws) {
  WHIT_NVTX("whit_forward_mse");
  if (!ws) return fail(WHIT_ERR_ARG, "factor_ws is NULL");
  if (!y || !w || !lambda || !loss_w || !z || !grad_z || !loss) return fail(WHIT_ERR_ARG, "NULL data pointer");
  if (ws->nb != 1 || ws->irr) return fail(WHIT_ERR_SHAPE, "the fused loss needs a single-band daily-grid workspace");
  if (d != ws->d || T != ws->T || B != ws->B)
    return fail(WHIT_ERR_SHAPE, "(d,T,B) = (%d,%lld,%lld) != workspace (%d,%lld,%lld)", d, (long long)T,
                (long long)B, ws->d, (long long)ws->T, (long long)ws->B);
  if (!aligned16(y) || !aligned16(w) || !aligned16(lambda) || !aligned16(loss_w) || !aligned16(z) ||
      !aligned16(grad_z) || !aligned16(loss))
    return fail(WHIT_ERR_ALIGN, "data pointers must be 16-B aligned");
  for (const void* o : {(const void*)z, (const void*)grad_z, (const void*)loss})
    if (o == y || o == w || o == lambda || o == loss_w) return fail(WHIT_ERR_ARG, "an output aliases an input");
  if (z == grad_z || z == loss || grad_z == loss) return fail(WHIT_ERR_ARG, "outputs alias each other");
  DeviceGuard guard(ws->device);
  if (!guard.ok) return fail(WHIT_ERR_CUDA, "cudaSetDevice(%d) failed", ws->device);
  Params p;
  whit_status st = fill_params(ws, &p, y, w, lambda);
  if (st != WHIT_OK) return st;
  const int kK = ws->kk;
  if ((st = wmap(ws, &p.tm_out0, z, ws->dt, B, T, kK, 1)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_out1, ws->buf + ws->L.off_dz, ws->dt, B, T - d, kK, 1)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_lw, loss_w, ws->dt, B, T, kK)) != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_out2, grad_z, ws->dt, B, T, kK, 1)) != WHIT_OK) return st;
  p.loss = loss;
  p.out2 = grad_z;
  const bool wdet = wdet_enabled();  // binary-W detection as in whit_forward: the backward reads bits
  if (wdet) {
    p.wbits_out = reinterpret_cast<uint32_t*>(ws->buf + ws->L.off_wbits);
    p.wbits = p.wbits_out;
    p.wflag = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_wflag);
  }
  ws->have_fwd = false;
  const bool pd = ws->lm == WHIT_LAMBDA_PER_DATE;
  if (ws->dt == WHIT_F32)
    st = pd ? dispatch_loss_d<float, true>(d, p, ws->stream) : dispatch_loss_d<float, false>(d, p, ws->stream);
  else
    st = pd ? dispatch_loss_d<double, true>(d, p, ws->stream) : dispatch_loss_d<double, false>(d, p, ws->stream);
  if (st != WHIT_OK) return st;
  mark_forward(ws, w, lambda, z, nullptr, nullptr, wdet);
  return WHIT_OK;
}

whit_status whit_forward(const void* y, const void* w, const void* lambda, int d, int64_t T, int64_t B, void* z,
                         whit_ws* ws) {
  if (ws && ws->nb != 1) return fail(WHIT_ERR_SHAPE, "workspace has %d bands: use whit_forward_bands", ws->nb);
  return whit_forward_bands(y, w, lambda, d, T, B, 1, z, ws);
}

whit_status whit_backward(const void* grad_z, whit_ws* ws, const void* z, void* grad_y, void* grad_lambda) {
  WHIT_NVTX("whit_backward");
  if (!ws) return fail(WHIT_ERR_ARG, "factor_ws is NULL");
  if (!ws->have_fwd) return fail(WHIT_ERR_STATE, "whit_backward without a preceding whit_forward on this workspace");
  if (!grad_z || !grad_y || !grad_lambda) return fail(WHIT_ERR_ARG, "NULL data pointer");
  if (z && z != ws->z) return fail(WHIT_ERR_STATE, "z is not the output of the matching whit_forward");
  if (!aligned16(grad_z) || !aligned16(grad_y) || !aligned16(grad_lambda))
    return fail(WHIT_ERR_ALIGN, "data pointers must be 16-B aligned");
  if (grad_y == grad_z || grad_lambda == grad_z || grad_y == grad_lambda)
    return fail(WHIT_ERR_ARG, "outputs alias inputs");
  DeviceGuard guard(ws->device);
  if (!guard.ok) return fail(WHIT_ERR_CUDA, "cudaSetDevice(%d) failed", ws->device);
  Params p;
  whit_status st = fill_params(ws, &p, grad_z, ws->w, ws->lam);
  if (st != WHIT_OK) return st;
  const int kK = ws->kk;
  if ((st = wmap(ws, &p.tm_dz, ws->buf + ws->L.off_dz, ws->dt, ws->B, ws->T - ws->d, kK, ws->nb)) != WHIT_OK)
    return st;
  if ((st = wmap(ws, &p.tm_out0, grad_y, ws->dt, ws->B, ws->T, kK, ws->nb)) != WHIT_OK) return st;
  if (ws->lm == WHIT_LAMBDA_PER_DATE) {
    if ((st = wmap(ws, &p.tm_out1, grad_lambda, ws->dt, ws->B, ws->T - ws->d, kK)) != WHIT_OK) return st;
  }
  p.out0 = grad_y;
  p.out1 = grad_lambda;
  p.dz_cache = ws->buf + ws->L.off_dz;
  if (ws->irr) {
    if ((st = wmap(ws, &p.tm_lw, ws->times, ws->dt, ws->B, ws->T, kK + 2 * ws->d)) != WHIT_OK) return st;
    return dispatch_irr<true>(ws, p);
  }
  if (ws->wbits) {
    p.wbits = ws->wbits;
    return dispatch_wb<true>(ws, p);
  }
  if (ws->tw && ws->hyb_g1 > 0) {
    // hybrid forward: the backward is ONE sequential launch (its bit-packed body where the forward's sequential
    // part found W binary); the groups the forward solved twisted rebuild the sequential factor checkpoints in
    // their up sweep (bwd_fac_from), which that launch's down sweep then reads (measured: the twisted backward
    // is slower than the sequential one at this size)
    p.bwd_fac_from = ws->hyb_g1;
    if (ws->wdet) {
      p.wbits = reinterpret_cast<const uint32_t*>(ws->buf + ws->L.off_wbits);
      p.wflag = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_wflag);
    }
    return dispatch<true>(ws, p);
  }
  if (ws->tw) {  // twisted backward, then whit_kernel for the groups the forward handed back
    Params pt;
    if ((st = tw_fill(ws, &pt, grad_z, ws->w, ws->lam, grad_y, grad_lambda, ws->buf + ws->L.off_dz, true)) != WHIT_OK)
      return st;
    if ((st = dispatch_tw<true>(ws, pt)) != WHIT_OK) return st;
    p.twflag = pt.twflag;
    p.tw_filter = 1;
    return dispatch<true>(ws, p);
  }
  if (ws->wdet) {  // the forward's binary-W bit plane and per-warp flags (the float plane is read otherwise)
    p.wbits = reinterpret_cast<const uint32_t*>(ws->buf + ws->L.off_wbits);
    p.wflag = reinterpret_cast<int32_t*>(ws->buf + ws->L.off_wflag);
  }
  return dispatch<true>(ws, p);
}

whit_status whit_backward_bands(const void* grad_z, whit_ws* ws, const void* z, void* grad_y, void* grad_lambda) {
  return whit_backward(grad_z, ws, z, grad_y, grad_lambda);
}

whit_status whit_grad_w(whit_ws* ws, const void* y, const void* z, const void* grad_y, void* grad_w) {
  WHIT_NVTX("whit_grad_w");
  if (!ws) return fail(WHIT_ERR_ARG, "factor_ws is NULL");
  if (!ws->have_fwd) return fail(WHIT_ERR_STATE, "whit_grad_w without a preceding forward on this workspace");
  if (ws->wbits || !ws->w) return fail(WHIT_ERR_STATE, "whit_grad_w needs the float weight plane (not bit-packed W)");
  if (!y || !z || !grad_y || !grad_w) return fail(WHIT_ERR_ARG, "NULL data pointer");
  if (z != ws->z) return fail(WHIT_ERR_STATE, "z is not the output of the matching forward");
  if (grad_w == y || grad_w == z || grad_w == grad_y || grad_w == ws->w)
    return fail(WHIT_ERR_ARG, "grad_w aliases an input");
  DeviceGuard guard(ws->device);
  if (!guard.ok) return fail(WHIT_ERR_CUDA, "cudaSetDevice(%d) failed", ws->device);
  const int32_t* info = reinterpret_cast<const int32_t*>(ws->buf + ws->L.off_info);
  const dim3 grid((unsigned)((ws->B + 255) / 256), (unsigned)std::min<int64_t>(ws->T, 1024));
  if (ws->dt == WHIT_F32)
    whit::grad_w_kernel<float><<<grid, 256, 0, ws->stream>>>(
        static_cast<const float*>(ws->w), static_cast<const float*>(y), static_cast<const float*>(z),
        static_cast<const float*>(grad_y), info, static_cast<float*>(grad_w), ws->T, ws->B, ws->nb);
  else
    whit::grad_w_kernel<double><<<grid, 256, 0, ws->stream>>>(
        static_cast<const double*>(ws->w), static_cast<const double*>(y), static_cast<const double*>(z),
        static_cast<const double*>(grad_y), info, static_cast<double*>(grad_w), ws->T, ws->B, ws->nb);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return WHIT_OK;
}

whit_status whit_posterior_variance(const void* w, const void* lambda, int d, int64_t T, int64_t B, void* var,
                                    whit_ws* ws) {
  WHIT_NVTX("whit_posterior_variance");
  if (!ws) return fail(WHIT_ERR_ARG, "factor_ws is NULL");
  if (!w || !lambda || !var) return fail(WHIT_ERR_ARG, "NULL data pointer");
  if (ws->nb != 1 || ws->irr) return fail(WHIT_ERR_SHAPE, "posterior variance needs a single-band daily-grid workspace");
  if (d != ws->d || T != ws->T || B != ws->B)
    return fail(WHIT_ERR_SHAPE, "(d,T,B) = (%d,%lld,%lld) != workspace (%d,%lld,%lld)", d, (long long)T,
                (long long)B, ws->d, (long long)ws->T, (long long)ws->B);
  if (!aligned16(w) || !aligned16(lambda) || !aligned16(var))
    return fail(WHIT_ERR_ALIGN, "data pointers must be 16-B aligned");
  if (var == w || var == lambda) return fail(WHIT_ERR_ARG, "var aliases an input");
  DeviceGuard guard(ws->device);
  if (!guard.ok) return fail(WHIT_ERR_CUDA, "cudaSetDevice(%d) failed", ws->device);
  Params p;
  whit_status st = fill_params(ws, &p, w /* unused rhs slot */, w, lambda);
  if (st != WHIT_OK) return st;
  if ((st = wmap(ws, &p.tm_out0, var, ws->dt, B, T, ws->kk, 1)) != WHIT_OK) return st;
  // the factor checkpoints are shared with the forward: a different (w, lambda) invalidates its backward, and
  // so does any forward whose checkpoints are not the sequential layout this kernel rewrites (twisted / hybrid)
  if (w != ws->w || lambda != ws->lam || ws->tw) ws->have_fwd = false;
  ws->have_info = true;  // (set at enqueue: info is written by this launch)
  const bool pd = ws->lm == WHIT_LAMBDA_PER_DATE;
  if (ws->dt == WHIT_F32)
    return pd ? dispatch_var_d<float, true>(d, p, ws->stream) : dispatch_var_d<float, false>(d, p, ws->stream);
  return pd ? dispatch_var_d<double, true>(d, p, ws->stream) : dispatch_var_d<double, false>(d, p, ws->stream);
}

whit_status whit_failures(whit_ws* ws, int64_t* n_failed, int32_t* host_info) {
  if (!ws || !n_failed) return fail(WHIT_ERR_ARG, "NULL argument");
  if (!ws->have_info) return fail(WHIT_ERR_STATE, "no forward or posterior variance has run on this workspace");
  DeviceGuard guard(ws->device);
  auto* cnt = reinterpret_cast<unsigned long long*>(ws->buf + ws->L.off_cnt);
  const int32_t* info = reinterpret_cast<const int32_t*>(ws->buf + ws->L.off_info);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof *cnt, ws->stream);
  if (e == cudaSuccess) {
    const long long blocks = std::min<long long>((ws->B + 255) / 256, 4096);
    whit::count_failures<<<(unsigned)blocks, 256, 0, ws->stream>>>(info, ws->B, cnt);
    e = cudaGetLastError();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, ws->stream);
  if (e == cudaSuccess && host_info)
    e = cudaMemcpyAsync(host_info, info, size_t(ws->B) * 4, cudaMemcpyDeviceToHost, ws->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ws->stream);
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "whit_failures: %s", cudaGetErrorString(e));
  *n_failed = (int64_t)h;
  return WHIT_OK;
}

whit_status whit_ws_set_twist(whit_ws* ws, int mode) {
  if (!ws) return fail(WHIT_ERR_ARG, "ws is NULL");
  if (mode < -1 || mode > 2) return fail(WHIT_ERR_ARG, "twist mode %d not in {-1, 0, 1, 2}", mode);
  ws->tw_mode = mode;
  return WHIT_OK;
}

whit_status whit_twist_groups(whit_ws* ws, int64_t* n_twisted, int64_t* n_groups) {
  if (!ws || !n_twisted || !n_groups) return fail(WHIT_ERR_ARG, "NULL argument");
  if (!ws->have_fwd) return fail(WHIT_ERR_STATE, "no forward has run on this workspace");
  const long long ng = (ws->B + 31) / 32;
  *n_groups = ng;
  *n_twisted = 0;
  if (!ws->tw) return WHIT_OK;
  DeviceGuard guard(ws->device);
  auto* cnt = reinterpret_cast<unsigned long long*>(ws->buf + ws->L.off_cnt);
  const int32_t* flags = reinterpret_cast<const int32_t*>(ws->buf + ws->L.off_twflag);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof *cnt, ws->stream);
  if (e == cudaSuccess) {
    whit::count_failures<<<(unsigned)std::min<long long>((ng + 255) / 256, 4096), 256, 0, ws->stream>>>(flags, ng, cnt);
    e = cudaGetLastError();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, ws->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ws->stream);
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "whit_twist_groups: %s", cudaGetErrorString(e));
  *n_twisted = (int64_t)h - ws->hyb_g1;  // (hybrid: groups [0, g1) are marked solved for the fallback's filter)
  return WHIT_OK;
}

whit_status whit_wbits_detected(whit_ws* ws, int64_t* n_binary, int64_t* n_warps) {
  if (!ws || !n_binary || !n_warps) return fail(WHIT_ERR_ARG, "NULL argument");
  if (!ws->have_info) return fail(WHIT_ERR_STATE, "no forward has run on this workspace");
  const long long nw = (ws->B + 31) / 32;
  *n_warps = nw;
  *n_binary = 0;
  if (!ws->wdet) return WHIT_OK;
  DeviceGuard guard(ws->device);
  auto* cnt = reinterpret_cast<unsigned long long*>(ws->buf + ws->L.off_cnt);
  const int32_t* flags = reinterpret_cast<const int32_t*>(ws->buf + ws->L.off_wflag);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof *cnt, ws->stream);
  if (e == cudaSuccess) {
    whit::count_failures<<<(unsigned)std::min<long long>((nw + 255) / 256, 4096), 256, 0, ws->stream>>>(flags, nw, cnt);
    e = cudaGetLastError();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, ws->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ws->stream);
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "whit_wbits_detected: %s", cudaGetErrorString(e));
  *n_binary = (int64_t)h;
  return WHIT_OK;
}

const int32_t* whit_info_device(const whit_ws* ws) {
  return ws ? reinterpret_cast<const int32_t*>(ws->buf + ws->L.off_info) : nullptr;
}

}  // extern "C"
