/*
 * libwhit -- B200 (sm_100a) hot path of the differentiable heteroscedastic
 * Whittaker layer, arXiv 2604.00048 ("the paper"; PAPER.md line n = P:n).
 *
 * For B independent series of length T (the paper's pixel time series)
 * the library solves, per series,
 *
 *     Omega z = W y,   Omega = W + D^T diag(lambda) D             Eq. (3)
 *
 * where W = diag(w) holds observation weights (1 observed, 0 cloud / gap /
 * padding), D is the order-d difference operator (the paper's order
 * k+1; on the daily grid its rows are the binomial stencil
 * c_j = (-1)^(d-j) C(d,j)), and lambda holds one penalty weight per
 * difference row -- or one scalar per series, the homoscedastic
 * Eq. (2).  Omega is symmetric positive definite with bandwidth d
 * and is factored by banded LDL^T with forward and back substitution
 * (Algorithm 1 P:127-142 is the LL^T analogue) -- never materialised:
 * each row of the band is assembled in registers from w, lambda and D.
 *
 * The backward pass takes the upstream cotangent g = dL/dz, solves
 * ONE adjoint system u = Omega^{-1} g with the same factor, and returns
 *     dL/dy         = w * u                        Eq. (5), P:77 (as a VJP)
 *     dL/dlambda_r  = -(D u)_r (D z)_r             Eq. (4), contracted with g
 *     (scalar lambda: the sum over r).
 *
 * ---------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ---------------------------------------------------------------------------
 * Pointers.  Every data pointer is a CUDA DEVICE pointer (cudaMalloc'd or a
 *   torch CUDA tensor's data_ptr), 16-byte aligned.  The library never
 *   allocates, frees, or copies through the host except where stated.
 * Layout.  Time-outer, series-contiguous ("[T][B]"): element (t, b) of a
 *   series-length plane lives at index t*B + b.  Planes: y, w, z, grad_z,
 *   grad_y are [T][B]; per-date lambda and its gradient are [T-d][B]
 *   (lambda_r weights difference row r, whose stencil covers dates r..r+d);
 *   scalar lambda and its gradient are [B].
 * Element type.  Either all planes are float32 (WHIT_F32) or all are float64
 *   (WHIT_F64), fixed at workspace creation.  All arithmetic is fp64 in
 *   registers either way; float32 outputs are rounded once at the store.
 * Sizes.  1 <= d <= 3;  T >= d + 1;  1 <= B;  B % 4 == 0 (F32) or B % 2 == 0
 *   (F64) so every time row is 16-byte aligned (the TMA row-stride rule);
 *   T * B < 2^31 per plane row index range is NOT required (64-bit indexing).
 * Inputs.  y finite where w > 0 (values where w == 0 are never read into the
 *   arithmetic: (W y)_t := 0 there, so NaN padding is allowed); w >= 0 and
 *   finite; lambda >= 0 and finite.  Inputs are never modified; outputs must
 *   not alias inputs.
 * Streams.  Every call is asynchronous on the stream bound to the workspace
 *   (whit_ws_create / whit_ws_set_stream); nothing synchronises except
 *   whit_failures.
 * Errors.  Argument problems are detected on the host before any launch and
 *   returned as a whit_status (nothing is launched); a launch failure returns
 *   WHIT_ERR_CUDA.  whit_last_error() gives a one-line reason for the calling
 *   thread's last non-OK status.  No C++ exception crosses this ABI.
 * Numerical failure.  A series whose Omega is not SPD is NOT a call error:
 *   the call returns WHIT_OK, that series' outputs (z, and in the backward
 *   grad_y, grad_lambda) are NaN, and its status is recorded LAPACK-style
 *   (xPBTRF "info") in the workspace: info[b] = 0 success; T-d+1 if fewer
 *   than d days have w > 0 (Omega = W + D^T Lambda D is then singular for
 *   lambda > 0: a nonzero polynomial of degree < d vanishing on every
 *   observed day has zero objective) -- unless an earlier pivot already
 *   failed; otherwise t+1 for the first pivot row t whose D_t is not a
 *   positive normal double below 2^1022 (D_t <= 0, NaN, Inf, or a subnormal /
 *   huge pivot whose reciprocal is not a normal double: DESIGN.md R-8).  This
 *   holds for every kernel family (single series, multi-band, irregular grid,
 *   posterior variance).  Read it with whit_failures().
 */
#ifndef LIBWHIT_H
#define LIBWHIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LIBWHIT_VERSION 100 /* 1.0.0 */

typedef enum {
  WHIT_OK = 0,
  WHIT_ERR_ARG = 1,    /* null pointer, bad enum, d out of range            */
  WHIT_ERR_SHAPE = 2,  /* T, B inconsistent with the workspace or rules     */
  WHIT_ERR_ALIGN = 3,  /* pointer not 16-B aligned or B % 4 (F32) / 2 (F64) */
  WHIT_ERR_WS = 4,     /* workspace buffer missing or too small             */
  WHIT_ERR_CUDA = 5,   /* CUDA runtime / driver error (see whit_last_error) */
  WHIT_ERR_STATE = 6   /* backward without a matching forward, z mismatch   */
} whit_status;

typedef enum { WHIT_F32 = 0, WHIT_F64 = 1 } whit_dtype;

typedef enum {
  WHIT_LAMBDA_SCALAR = 0,   /* lambda is [B]: Eq. (2)           */
  WHIT_LAMBDA_PER_DATE = 1  /* lambda is [T-d][B]: Eq. (3)  */
} whit_lambda_mode;

/* Opaque HOST handle describing one (d, T, B, dtype, lambda mode) problem and
 * binding a caller-owned device buffer ("factor_ws").  It owns no device
 * memory.  It carries the state a forward leaves for its backward: the
 * factor checkpoints, the cached D z plane, the per-series info, and the
 * w / lambda pointers of that forward. */
typedef struct whit_ws whit_ws;

/* Library version (LIBWHIT_VERSION). */
int whit_version(void);

/* Human-readable name of a status code (static string). */
const char* whit_status_string(whit_status s);

/* One-line reason for the calling thread's most recent non-OK status, or ""
 * (thread-local static string, valid until the next call on that thread). */
const char* whit_last_error(void);

/* Bytes of device memory whit_ws_create needs for this problem; 0 if the
 * arguments are invalid.  Host-only, no CUDA call.  Contents: the D z cache
 * ([T-d][B] of the I/O dtype), fp64 factor checkpoints every K time steps
 * (the forward's factor + RHS state, the backward's RHS state), and int32
 * info[B]. */
size_t whit_ws_bytes(int d, int64_t T, int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode);

/* Create a workspace handle over dev_buf (device memory of at least
 * whit_ws_bytes(...) bytes, 256-B aligned, owned by the caller and kept alive
 * until whit_ws_destroy).  cuda_stream is a cudaStream_t (NULL = legacy
 * default stream).  On success *out receives the handle. */
whit_status whit_ws_create(whit_ws** out, int d, int64_t T, int64_t B, whit_dtype dtype,
                           whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes,
                           void* cuda_stream);

/* Rebind the stream later calls launch on (cudaStream_t). */
whit_status whit_ws_set_stream(whit_ws* ws, void* cuda_stream);

/* Destroy the host handle (does not touch device memory).  NULL is a no-op. */
void whit_ws_destroy(whit_ws* ws);

/* Forward, Eq. (3) or Eq. (2):  z = (W + D^T diag(lambda) D)^{-1} W y.
 *   y       [T][B]            observations (paper's x)
 *   w       [T][B]            weights, diag of W
 *   lambda  [T-d][B] or [B]   per the workspace's lambda mode
 *   d, T, B                   must equal the workspace's
 *   z       [T][B]            output
 *   factor_ws                 receives the state the backward reuses; w and
 *                             lambda must stay valid and unmodified until the
 *                             matching whit_backward has run.
 * Binary W: the forward checks every weight; for each warp of 32
 * series whose weights are all exactly 0 or 1 it writes W as a bit plane
 * (1 bit per date) into factor_ws, and its own back substitution and the
 * matching whit_backward read those bits instead of the float w rows (fewer
 * HBM bytes; results bitwise identical).  Soft weights keep the float path.
 * WHIT_WDET=0 in the environment turns the detection off (A/B runs).
 * One kernel launch. */
whit_status whit_forward(const void* y, const void* w, const void* lambda, int d, int64_t T,
                         int64_t B, void* z, whit_ws* factor_ws);

/* Backward: one adjoint solve u = Omega^{-1} grad_z reusing the
 * forward's factor (checkpointed in factor_ws, recomputed per chunk), then
 *   grad_y      [T][B]             = w * u                       Eq. (5)
 *   grad_lambda [T-d][B] or [B]    = -(D u)_r (D z)_r (or sum_r)   Eq. (4)
 * z may be NULL; if non-NULL it must be the z pointer of the matching
 * whit_forward (the cached fp64-derived D z is used, not z itself).
 * Returns WHIT_ERR_STATE if no forward ran on factor_ws.  One kernel launch. */
whit_status whit_backward(const void* grad_z, whit_ws* factor_ws, const void* z, void* grad_y,
                          void* grad_lambda);

/* Gradient with respect to the observation weights (the optional output of
 * NEXT-3; the paper keeps W fixed).  Differentiating Eq. (3)
 * in w_t gives Omega dz = e_t (y_t - z_t) dw_t, so with u = Omega^{-1} g:
 *   grad_w[t][b] = sum_c u_{c,t} (y_{c,t} - z_{c,t}),   u = grad_y / w,
 * summed over the bands of a multi-band workspace (C = 1 otherwise).  Reading
 * R-19: grad_w = 0 where w_t = 0 (y_t carries no value there, R-4); NaN for a
 * failed series.  Call after whit_backward (or whit_backward_bands, or the
 * irregular-grid backward) on the same workspace: y is the forward's input, z
 * the forward's output (checked against the workspace), grad_y the backward's
 * output; grad_w has w's shape [T][B] and dtype.  The float weight plane of the
 * last forward is used (WHIT_ERR_STATE after whit_forward_wbits).  One
 * element-wise kernel launch on the workspace stream. */
whit_status whit_grad_w(whit_ws* factor_ws, const void* y, const void* z, const void* grad_y, void* grad_w);

/* ---------------------------------------------------------------------------
 * Multi-band pixels (NEXT-1; the paper's "batched multivariate vectors", P:28,
 * C = 10 bands per pixel in its benchmark).  The C bands of a pixel
 * share w and lambda, hence Omega and its factor; each band is its own
 * right-hand side.  B counts PIXELS:
 *   y, z, grad_z, grad_y   [C][T][B]       (band planes stacked)
 *   w                      [T][B]           (shared)
 *   lambda, grad_lambda    [T-d][B] or [B]  (shared; grad_lambda is summed over
 *                                             bands, in a fixed order, in fp64:
 *                                             dL/dlambda_r = -sum_c (D u_c)_r (D z_c)_r)
 * 1 <= C <= 10 (one CTA's shared memory holds the C band pipelines).  The
 * factor is formed once per pixel per sweep by one factor warp and handed to
 * the band warps through shared memory (two bands per band warp), so w,
 * lambda and factor-checkpoint bytes and the factor's fp64 work are amortised
 * over C bands; every band's z and grad_y equal the single-band results bit
 * for bit.  info (one per pixel): the status rule of "Numerical failure"
 * (first failing pivot row of the shared factor, T-d+1 for < d observed
 * days).  The
 * single-band entry points above are the C = 1 case (whit_forward on a C > 1
 * workspace is WHIT_ERR_SHAPE; whit_backward works for any C). */
size_t whit_ws_bytes_bands(int d, int64_t T, int64_t B, int C, whit_dtype dtype, whit_lambda_mode lambda_mode);

whit_status whit_ws_create_bands(whit_ws** out, int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                                 whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes,
                                 void* cuda_stream);

whit_status whit_forward_bands(const void* y, const void* w, const void* lambda, int d, int64_t T,
                               int64_t B, int C, void* z, whit_ws* factor_ws);

whit_status whit_backward_bands(const void* grad_z, whit_ws* factor_ws, const void* z, void* grad_y,
                                void* grad_lambda);

/* ---------------------------------------------------------------------------
 * Irregular acquisition grid (NEXT-2; the paper's formulation on uneven dates,
 * P:26-28): D is the order-d dspline divided-difference operator on per-series
 * times, row r: c_{r,j} = (d-1)! (t_{r+d} - t_r) / prod_{i != j} (t_{r+j} - t_{r+i})
 * (plain differences for d = 1; the daily stencil on unit-spaced times).
 *   times [T][B] (I/O dtype), strictly increasing per series (e.g. days; pad
 *   unaligned series with w = 0 at increasing dummy dates).
 * Workspace from whit_ws_create_times (checkpoint interval 8); the matching
 * backward is whit_backward (the workspace remembers times, which must stay
 * valid and unmodified until it has run).  info: T-d+1 (< d observed days),
 * -1 (other non-positive pivot).  One launch each.
 * The _bands variants take C <= 10 bands per pixel sharing w, lambda and
 * times (the paper's Table 1 workload: C = 10 on uneven dates),
 * with the multi-band layout above (y, z, grad_z, grad_y [C][T][B]); one
 * factor per pixel (the shared-factor kernel with the per-row dates stencils);
 * every band's z and grad_y equal the single-band irregular results bit for
 * bit, grad_lambda is summed over bands.  whit_forward_times is C = 1. */
size_t whit_ws_bytes_times(int d, int64_t T, int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode);

whit_status whit_ws_create_times(whit_ws** out, int d, int64_t T, int64_t B, whit_dtype dtype,
                                 whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes,
                                 void* cuda_stream);

whit_status whit_forward_times(const void* y, const void* w, const void* lambda, const void* times, int d,
                               int64_t T, int64_t B, void* z, whit_ws* factor_ws);

size_t whit_ws_bytes_times_bands(int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                                 whit_lambda_mode lambda_mode);

whit_status whit_ws_create_times_bands(whit_ws** out, int d, int64_t T, int64_t B, int C, whit_dtype dtype,
                                       whit_lambda_mode lambda_mode, void* dev_buf, size_t dev_bytes,
                                       void* cuda_stream);

whit_status whit_forward_times_bands(const void* y, const void* w, const void* lambda, const void* times, int d,
                                     int64_t T, int64_t B, int C, void* z, whit_ws* factor_ws);

/* ---------------------------------------------------------------------------
 * Bit-packed W.  The paper's W is binary (w_ii is 1 if the date was
 * observed and not cloud-flagged, else 0); storing it as 1 bit per date
 * instead of a float plane removes ~4 of the ~19 bytes per series-date each
 * sweep reads.  Layout: uint32 [ceil(T/32)][B], bit j of word r of series b is
 * (w[32r + j][b] != 0); bits past T are 0.  Results are bitwise identical to
 * whit_forward / whit_backward with the 0/1 float plane.
 *   whit_pack_mask   packs a [T][B] plane (any nonzero -> 1) on `cuda_stream`.
 *   whit_forward_wbits  forward from the bits; the matching backward is
 *                    whit_backward (the workspace remembers wbits, which must
 *                    stay valid and unmodified until it has run).
 * Single-band daily-grid workspaces (whit_ws_create). */
whit_status whit_pack_mask(const void* w, int64_t T, int64_t B, whit_dtype dtype, uint32_t* bits, void* cuda_stream);

whit_status whit_forward_wbits(const void* y, const uint32_t* wbits, const void* lambda, int d, int64_t T, int64_t B,
                               void* z, whit_ws* factor_ws);

/* Forward fused with the training loss (NEXT-3): the paper trains with a
 * masking strategy and an MSE loss, the MSE of P:222:
 *     loss[b]   = T^{-1} sum_t loss_w[t][b] (z[t][b] - y[t][b])^2
 *     grad_z    = dL/dz with L = sum_b loss[b]:  2 T^{-1} loss_w (z - y)
 * y is both the smoother input (through W y: held-out dates have w = 0) and
 * the reference (the caller may pre-fill y at cloud/edge gaps with the
 * nearest valid value, P:197 -- w = 0 there, so the solve never reads it).
 * loss_w [T][B] selects / weights the scored dates (0 = not scored; y may be
 * NaN there).  Same z and factor_ws state as whit_forward: feed grad_z to
 * whit_backward.  Saves the separate loss/gradient pass over z (and the
 * round trip of g).  Binary-W detection as in whit_forward (the matching
 * whit_backward reads W as bits where it is binary).  Single-band workspaces.
 * One launch. */
whit_status whit_forward_mse(const void* y, const void* w, const void* lambda, const void* loss_w, int d, int64_t T,
                             int64_t B, void* z, void* grad_z, void* loss, whit_ws* factor_ws);

/* Posterior variance (NEXT-4): var[t][b] = (Omega^{-1})_{tt}, the pointwise
 * variance of z up to the noise-variance factor sigma^2 (the credibility band
 * of Fig. 4: under y ~ N(z, sigma^2 W^{-1}) with prior precision
 * D^T Lambda D / sigma^2, Cov(z | y) = sigma^2 Omega^{-1}).  Computed by
 * Takahashi's selected inversion on the same deviation-form banded factor
 * (one up sweep, one down sweep; only the d x d window of Omega^{-1} next to
 * the diagonal is ever formed).  w, lambda, d, T, B as in whit_forward; var
 * [T][B] output.  Uses factor_ws's checkpoint area and info[] (the status
 * rule of "Numerical failure" above: first failing pivot row, var NaN);
 * if (w, lambda) differ from the last forward's, that forward's backward is
 * invalidated (WHIT_ERR_STATE).  Single-band workspaces only.  One launch. */
whit_status whit_posterior_variance(const void* w, const void* lambda, int d, int64_t T, int64_t B, void* var,
                                    whit_ws* factor_ws);

/* SYNCHRONISES the workspace stream, then reports how many series of the
 * last forward (or posterior variance) failed (non-SPD, see "Numerical failure") in *n_failed and,
 * if host_info is non-NULL, copies info[0..B) (int32) to host_info. */
whit_status whit_failures(whit_ws* ws, int64_t* n_failed, int32_t* host_info);

/* Device pointer to the workspace's info[B] (int32), for callers that want to
 * consume it on the device without a synchronisation. */
const int32_t* whit_info_device(const whit_ws* ws);

/* Execution path of whit_forward / whit_backward on a single-band daily-grid
 * workspace: the same solve of Eq. (3) and the same backward
 * by a different elimination order of the banded SPD system (
 * DESIGN.md R-21) -- results agree to rounding.  Small batches take the TWISTED path (two warps per group of 32
 * series: one factors the first half of the dates forward, the other the
 * second half in reversed time; they meet in a d x d block -- half the
 * per-series latency, twice the warps in flight); a group whose halves are
 * not safely SPD on their own falls back to the sequential kernel inside the
 * same call (results and status as the sequential path).  Batches just past
 * one wave of the sequential kernel (1,776 < ceil(B/32) <= 2,400 groups, e.g.
 * B = 65,536) take a HYBRID launch: the first g1 groups sequential (g1 =
 * 1,728 with scalar lambda, 1,504 per date), the
 * rest twisted on a second stream (forked and joined with events on the
 * workspace stream).  mode: -1 auto (the default: WHIT_TWIST=0/1 in the
 * environment, else twisted for B <= 28,416 with scalar lambda, B <= 24,864
 * per date -- its warps fit one wave -- and
 * hybrid as above; WHIT_HYBRID=0 turns the hybrid off), 0 never, 1 twisted
 * whenever T allows (T >= about 4K + 2d), 2 hybrid whenever B > g1 * 32. */
whit_status whit_ws_set_twist(whit_ws* ws, int mode);

/* SYNCHRONISES the workspace stream, then reports how many groups of 32
 * series the last whit_forward solved on the twisted path (*n_twisted) out of
 * *n_groups = ceil(B/32) (0 if the path was not taken).  Diagnostic. */
whit_status whit_twist_groups(whit_ws* ws, int64_t* n_twisted, int64_t* n_groups);

/* SYNCHRONISES the workspace stream, then reports how many of the last plain
 * whit_forward's warps (groups of 32 consecutive series) found a binary W (the
 * paper's W is 0/1) and
 * read it as bits (*n_binary) out of *n_warps = ceil(B/32).  *n_binary = 0 if
 * the last forward was not the plain float-W forward or the detection is off.
 * Diagnostic (tests, bench); WHIT_ERR_STATE if no forward ran. */
whit_status whit_wbits_detected(whit_ws* ws, int64_t* n_binary, int64_t* n_warps);

/* ---------------------------------------------------------------------------
 * Streaming executor for data in HOST memory.
 *
 * Runs the forward (and, if grad_z != NULL, the backward) over B series whose
 * planes live in HOST memory in the same [T][B] layout, streaming them through
 * the GPU in series chunks of `chunk` columns on `nbuf` device slots with one
 * stream each: pitched 2-D host->device copies of the chunk, whit_forward /
 * whit_backward, pitched 2-D device->host copies of z, grad_y, grad_lambda and
 * (if info != NULL) the chunk's info.  Slots overlap, so copies in both
 * directions run concurrently with the kernels.  Same arithmetic and results
 * as the device entry points (each chunk is an independent batch).
 *
 *   y, w, lambda, grad_z   HOST inputs ([T][B], [T][B], [T-d][B] or [B], [T][B])
 *   z, grad_y, grad_lambda HOST outputs (grad_* ignored when grad_z == NULL)
 *   info                   optional HOST int32[B] (LAPACK-style status, see above)
 *   chunk, nbuf            series per chunk (multiple of 4 for F32, 2 for F64),
 *                          device slots in flight (1..8; 3 recommended)
 *   dev_buf, dev_bytes     caller-owned device scratch, >= whit_host_ws_bytes(),
 *                          256-B aligned
 *   cuda_stream            the call is ordered after prior work on this stream
 *                          and later work on it waits for completion; the host
 *                          call itself returns after enqueueing.
 * Host buffers should be page-locked (cudaHostAlloc / torch pin_memory) for the
 * copies to be asynchronous and overlap; pageable memory works but serialises.
 * The host buffers must stay valid until the stream has completed. */
size_t whit_host_ws_bytes(int d, int64_t T, int64_t chunk, whit_dtype dtype, whit_lambda_mode lambda_mode,
                          int nbuf);

whit_status whit_run_host(const void* y, const void* w, const void* lambda, const void* grad_z, int d, int64_t T,
                          int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode, void* z, void* grad_y,
                          void* grad_lambda, int32_t* info, int64_t chunk, int nbuf, void* dev_buf,
                          size_t dev_bytes, void* cuda_stream);

/* The same with the binary W as bits (HOST uint32 [ceil(T/32)][B], the layout
 * of whit_pack_mask): 1/32 of the weight plane's PCIe bytes; each chunk runs
 * whit_forward_wbits (+ whit_backward).  Results equal whit_run_host with the
 * 0/1 float plane bit for bit.  Same device scratch size. */
whit_status whit_run_host_wbits(const void* y, const uint32_t* wbits, const void* lambda, const void* grad_z, int d,
                                int64_t T, int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode, void* z,
                                void* grad_y, void* grad_lambda, int32_t* info, int64_t chunk, int nbuf,
                                void* dev_buf, size_t dev_bytes, void* cuda_stream);

/* Multi-band pixels from HOST memory (a Sentinel-2 tile streamed through the
 * shared-factor kernels): y, grad_z, z, grad_y are HOST [C][T][B] (band planes
 * stacked), w [T][B] and lambda shared, info per pixel; each chunk of `chunk`
 * pixels runs whit_forward_bands (+ whit_backward_bands).  Device scratch:
 * whit_host_ws_bytes_bands (C = 1 gives whit_host_ws_bytes). */
size_t whit_host_ws_bytes_bands(int d, int64_t T, int64_t chunk, int C, whit_dtype dtype,
                                whit_lambda_mode lambda_mode, int nbuf);

whit_status whit_run_host_bands(const void* y, const void* w, const void* lambda, const void* grad_z, int d,
                                int64_t T, int64_t B, int C, whit_dtype dtype, whit_lambda_mode lambda_mode,
                                void* z, void* grad_y, void* grad_lambda, int32_t* info, int64_t chunk, int nbuf,
                                void* dev_buf, size_t dev_bytes, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* LIBWHIT_H */
