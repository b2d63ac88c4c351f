// libwhit streaming executor for data in HOST memory (whit_run_host).
//
// The batch of B series lives in host [T][B] planes; the executor walks it in
// series chunks of `chunk` columns, cycling through `nbuf` device slots, each
// with its own stream: 2-D copies (cudaMemcpy2DAsync, pitched host source) of
// the chunk's input columns host->device, whit_forward (+ whit_backward), and
// 2-D copies of the outputs device->host.  Slots run concurrently, so the
// H2D of chunk j+1, the kernels of chunk j and the D2H of chunk j-1 overlap
// (B200 has separate copy engines per direction; PCIe is full duplex).
//
// Built only on the public entry points (whit_ws_create / whit_forward /
// whit_backward / whit_info_device): it is a runtime around the kernels, no
// arithmetic of the method happens here.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "libwhit.h"
#include "whit_internal.h"

using whit_detail::fail;

namespace {

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

struct SlotLayout {
  size_t y, w, lam, g, z, gy, gl, ws, total;
};

// One device slot: the chunk's planes (y, g, z, grad_y: C band planes each) and its workspace.
bool slot_layout(int d, int64_t T, int64_t chunk, int C, whit_dtype dt, whit_lambda_mode lm, SlotLayout* L) {
  const size_t esz = dt == WHIT_F32 ? 4 : 8;
  const size_t plane = size_t(T) * size_t(chunk) * esz;
  const size_t lamb = lm == WHIT_LAMBDA_PER_DATE ? size_t(T - d) * size_t(chunk) * esz : size_t(chunk) * esz;
  const size_t wsb = whit_ws_bytes_bands(d, T, chunk, C, dt, lm);
  if (wsb == 0) return false;
  size_t o = 0;
  L->y = o;   o = a256(o + size_t(C) * plane);
  L->w = o;   o = a256(o + plane);
  L->lam = o; o = a256(o + lamb);
  L->g = o;   o = a256(o + size_t(C) * plane);
  L->z = o;   o = a256(o + size_t(C) * plane);
  L->gy = o;  o = a256(o + size_t(C) * plane);
  L->gl = o;  o = a256(o + lamb);
  L->ws = o;  o = a256(o + wsb);
  L->total = o;
  return true;
}

}  // namespace

extern "C" {

size_t whit_host_ws_bytes_bands(int d, int64_t T, int64_t chunk, int C, whit_dtype dtype,
                                whit_lambda_mode lambda_mode, int nbuf) {
  if (nbuf < 1 || nbuf > 8 || chunk < 1) return 0;
  if (lambda_mode != WHIT_LAMBDA_SCALAR && lambda_mode != WHIT_LAMBDA_PER_DATE) return 0;
  SlotLayout L;
  if (!slot_layout(d, T, chunk, C, dtype, lambda_mode, &L)) return 0;
  return size_t(nbuf) * L.total;
}

size_t whit_host_ws_bytes(int d, int64_t T, int64_t chunk, whit_dtype dtype, whit_lambda_mode lambda_mode,
                          int nbuf) {
  return whit_host_ws_bytes_bands(d, T, chunk, 1, dtype, lambda_mode, nbuf);
}

}  // extern "C"

namespace {

// w (a [T][B] weight plane) or wbits (the bit-packed binary W, [ceil(T/32)][B] uint32) -- exactly one.
whit_status run_host(const void* y, const void* w, const uint32_t* wbits, const void* lambda, const void* grad_z,
                     int d, int64_t T, int64_t B, int C, whit_dtype dtype, whit_lambda_mode lambda_mode, void* z,
                     void* grad_y, void* grad_lambda, int32_t* info, int64_t chunk, int nbuf, void* dev_buf,
                     size_t dev_bytes, void* cuda_stream) {
  if (!y || !(w || wbits) || !lambda || !z) return fail(WHIT_ERR_ARG, "NULL host pointer");
  if (grad_z && (!grad_y || !grad_lambda)) return fail(WHIT_ERR_ARG, "grad_z given without grad_y / grad_lambda");
  if (dtype != WHIT_F32 && dtype != WHIT_F64) return fail(WHIT_ERR_ARG, "bad dtype");
  if (lambda_mode != WHIT_LAMBDA_SCALAR && lambda_mode != WHIT_LAMBDA_PER_DATE) return fail(WHIT_ERR_ARG, "bad lambda mode");
  if (d < 1 || d > 3) return fail(WHIT_ERR_ARG, "d = %d not in {1,2,3}", d);
  if (T < d + 1 || B < 1) return fail(WHIT_ERR_SHAPE, "bad T = %lld / B = %lld", (long long)T, (long long)B);
  const int q = dtype == WHIT_F32 ? 4 : 2;
  if (chunk < 1 || chunk % q || B % q)
    return fail(WHIT_ERR_ALIGN, "B and chunk must be multiples of %d", q);
  if (nbuf < 1 || nbuf > 8) return fail(WHIT_ERR_ARG, "nbuf = %d not in [1, 8]", nbuf);
  if (C < 1 || (C > 1 && wbits)) return fail(WHIT_ERR_ARG, "bands C = %d (bit-packed W is single-band)", C);
  chunk = std::min(chunk, B);
  SlotLayout L;
  if (!slot_layout(d, T, chunk, C, dtype, lambda_mode, &L)) return fail(WHIT_ERR_SHAPE, "bad chunk shape / bands");
  if (!dev_buf || (reinterpret_cast<uintptr_t>(dev_buf) & 255u)) return fail(WHIT_ERR_WS, "device buffer NULL or not 256-B aligned");
  if (dev_bytes < size_t(nbuf) * L.total)
    return fail(WHIT_ERR_WS, "device buffer %zu bytes < required %zu", dev_bytes, size_t(nbuf) * L.total);

  const size_t esz = dtype == WHIT_F32 ? 4 : 8;
  const bool pd = lambda_mode == WHIT_LAMBDA_PER_DATE;
  const int64_t TL = pd ? T - d : 1;  // rows of the lambda plane
  cudaStream_t user = static_cast<cudaStream_t>(cuda_stream);
  char* base = static_cast<char*>(dev_buf);

  std::vector<cudaStream_t> st(nbuf, nullptr);
  std::vector<cudaEvent_t> done(nbuf, nullptr);
  cudaEvent_t start = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  for (int s = 0; s < nbuf && e == cudaSuccess; ++s) {
    e = cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventRecord(start, user);
  for (int s = 0; s < nbuf && e == cudaSuccess; ++s) e = cudaStreamWaitEvent(st[s], start, 0);

  whit_status status = WHIT_OK;
  const int64_t nch = (B + chunk - 1) / chunk;
  for (int64_t j = 0; j < nch && e == cudaSuccess && status == WHIT_OK; ++j) {
    const int s = int(j % nbuf);
    const int64_t b0 = j * chunk, bc = std::min(chunk, B - b0);
    char* sb = base + size_t(s) * L.total;
    const size_t hp = size_t(B) * esz, dp = size_t(bc) * esz, off = size_t(b0) * esz;
    // one [T][bc] plane (band c of a [C][T][B] host array: rows c*T .. c*T+T-1 of the [C*T][B] view)
    auto h2d = [&](size_t dst, const void* src, int64_t rows, int c = 0) {
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(sb + dst + size_t(c) * size_t(rows) * dp, dp,
                              static_cast<const char*>(src) + size_t(c) * size_t(rows) * hp + off, hp, dp,
                              size_t(rows), cudaMemcpyHostToDevice, st[s]);
    };
    auto d2h = [&](void* dst, size_t src, int64_t rows, int c = 0) {
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(static_cast<char*>(dst) + size_t(c) * size_t(rows) * hp + off, hp,
                              sb + src + size_t(c) * size_t(rows) * dp, dp, dp, size_t(rows), cudaMemcpyDeviceToHost,
                              st[s]);
    };
    for (int c = 0; c < C; ++c) h2d(L.y, y, T, c);
    if (w) {
      h2d(L.w, w, T);
    } else if (e == cudaSuccess) {  // bits: ceil(T/32) rows of bc uint32 words
      e = cudaMemcpy2DAsync(sb + L.w, size_t(bc) * 4, reinterpret_cast<const char*>(wbits) + size_t(b0) * 4,
                            size_t(B) * 4, size_t(bc) * 4, size_t((T + 31) / 32), cudaMemcpyHostToDevice, st[s]);
    }
    h2d(L.lam, lambda, TL);
    if (grad_z)
      for (int c = 0; c < C; ++c) h2d(L.g, grad_z, T, c);
    if (e != cudaSuccess) break;
    whit_ws* ws = nullptr;
    status = whit_ws_create_bands(&ws, d, T, bc, C, dtype, lambda_mode, sb + L.ws, L.total - L.ws, st[s]);
    if (status != WHIT_OK) break;
    if (!w)
      status = whit_forward_wbits(sb + L.y, reinterpret_cast<const uint32_t*>(sb + L.w), sb + L.lam, d, T, bc,
                                  sb + L.z, ws);
    else if (C > 1)
      status = whit_forward_bands(sb + L.y, sb + L.w, sb + L.lam, d, T, bc, C, sb + L.z, ws);
    else
      status = whit_forward(sb + L.y, sb + L.w, sb + L.lam, d, T, bc, sb + L.z, ws);
    if (status == WHIT_OK && grad_z) status = whit_backward(sb + L.g, ws, sb + L.z, sb + L.gy, sb + L.gl);
    const int32_t* dinfo = whit_info_device(ws);
    whit_ws_destroy(ws);  // host handle only; the enqueued work does not reference it
    if (status != WHIT_OK) break;
    for (int c = 0; c < C; ++c) d2h(z, L.z, T, c);
    if (grad_z) {
      for (int c = 0; c < C; ++c) d2h(grad_y, L.gy, T, c);
      d2h(grad_lambda, L.gl, TL);
    }
    if (info && e == cudaSuccess)
      e = cudaMemcpyAsync(info + b0, dinfo, size_t(bc) * 4, cudaMemcpyDeviceToHost, st[s]);
  }
  for (int s = 0; s < nbuf; ++s) {
    if (st[s] && done[s]) {
      cudaError_t e2 = cudaEventRecord(done[s], st[s]);
      if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(user, done[s], 0);
      if (e == cudaSuccess) e = e2;
    }
  }
  for (int s = 0; s < nbuf; ++s) {
    if (done[s]) cudaEventDestroy(done[s]);
    if (st[s]) cudaStreamDestroy(st[s]);  // deferred until its work completes
  }
  if (start) cudaEventDestroy(start);
  if (status != WHIT_OK) return status;
  if (e != cudaSuccess) return fail(WHIT_ERR_CUDA, "whit_run_host: %s", cudaGetErrorString(e));
  return WHIT_OK;
}

}  // namespace

extern "C" {

whit_status whit_run_host(const void* y, const void* w, const void* lambda, const void* grad_z, int d, int64_t T,
                          int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode, void* z, void* grad_y,
                          void* grad_lambda, int32_t* info, int64_t chunk, int nbuf, void* dev_buf,
                          size_t dev_bytes, void* cuda_stream) {
  if (!w) return fail(WHIT_ERR_ARG, "NULL host pointer");
  return run_host(y, w, nullptr, lambda, grad_z, d, T, B, 1, dtype, lambda_mode, z, grad_y, grad_lambda, info,
                  chunk, nbuf, dev_buf, dev_bytes, cuda_stream);
}

whit_status whit_run_host_wbits(const void* y, const uint32_t* wbits, const void* lambda, const void* grad_z, int d,
                                int64_t T, int64_t B, whit_dtype dtype, whit_lambda_mode lambda_mode, void* z,
                                void* grad_y, void* grad_lambda, int32_t* info, int64_t chunk, int nbuf,
                                void* dev_buf, size_t dev_bytes, void* cuda_stream) {
  if (!wbits) return fail(WHIT_ERR_ARG, "NULL host pointer");
  return run_host(y, nullptr, wbits, lambda, grad_z, d, T, B, 1, dtype, lambda_mode, z, grad_y, grad_lambda, info,
                  chunk, nbuf, dev_buf, dev_bytes, cuda_stream);
}

whit_status whit_run_host_bands(const void* y, const void* w, const void* lambda, const void* grad_z, int d,
                                int64_t T, int64_t B, int C, whit_dtype dtype, whit_lambda_mode lambda_mode,
                                void* z, void* grad_y, void* grad_lambda, int32_t* info, int64_t chunk, int nbuf,
                                void* dev_buf, size_t dev_bytes, void* cuda_stream) {
  if (!w) return fail(WHIT_ERR_ARG, "NULL host pointer");
  return run_host(y, w, nullptr, lambda, grad_z, d, T, B, C, dtype, lambda_mode, z, grad_y, grad_lambda, info,
                  chunk, nbuf, dev_buf, dev_bytes, cuda_stream);
}

}  // extern "C"
