"""ctypes binding of libwhit (include/libwhit.h): argument marshalling only.

Every compute step runs in the CUDA kernels inside ``libwhit.so``; this module
converts torch tensors to device pointers, checks shapes, and raises
``WhitError`` on a non-OK status.  There is no CPU fallback: if the shared
library is missing, importing the package raises ``ImportError``.

Function names mirror the C-ABI: ``whit_ws_bytes``, ``whit_ws_create``,
``whit_forward``, ``whit_backward``, ``whit_failures`` ...
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WHIT_LIB_PATH") or os.path.join(_HERE, "libwhit.so")  # override: dev A/B builds

WHIT_F32, WHIT_F64 = 0, 1
WHIT_LAMBDA_SCALAR, WHIT_LAMBDA_PER_DATE = 0, 1
STATUS = {0: "WHIT_OK", 1: "WHIT_ERR_ARG", 2: "WHIT_ERR_SHAPE", 3: "WHIT_ERR_ALIGN",
          4: "WHIT_ERR_WS", 5: "WHIT_ERR_CUDA", 6: "WHIT_ERR_STATE"}

# (name, restype, argtypes) for every function in include/libwhit.h
_VP, _I64, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
SIGNATURES = [
    ("whit_version", ctypes.c_int, []),
    ("whit_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("whit_last_error", ctypes.c_char_p, []),
    ("whit_ws_bytes", _SZ, [ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int]),
    ("whit_ws_create", ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int,
                                      _VP, _SZ, _VP]),
    ("whit_ws_set_stream", ctypes.c_int, [_VP, _VP]),
    ("whit_ws_destroy", None, [_VP]),
    ("whit_forward", ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int, _I64, _I64, _VP, _VP]),
    ("whit_backward", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("whit_grad_w", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("whit_failures", ctypes.c_int, [_VP, ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_int32)]),
    ("whit_info_device", _VP, [_VP]),
    ("whit_wbits_detected", ctypes.c_int, [_VP, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("whit_ws_set_twist", ctypes.c_int, [_VP, ctypes.c_int]),
    ("whit_twist_groups", ctypes.c_int, [_VP, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("whit_ws_bytes_bands", _SZ, [ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("whit_ws_create_bands", ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, _VP, _SZ, _VP]),
    ("whit_forward_bands", ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int, _I64, _I64, ctypes.c_int, _VP, _VP]),
    ("whit_backward_bands", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("whit_ws_bytes_times", _SZ, [ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int]),
    ("whit_ws_create_times", ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int,
                                            _VP, _SZ, _VP]),
    ("whit_forward_times", ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int, _I64, _I64, _VP, _VP]),
    ("whit_ws_bytes_times_bands", _SZ, [ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("whit_ws_create_times_bands", ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_int, _I64, _I64, ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_int, _VP, _SZ, _VP]),
    ("whit_forward_times_bands", ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int, _I64, _I64, ctypes.c_int, _VP,
                                                _VP]),
    ("whit_pack_mask", ctypes.c_int, [_VP, _I64, _I64, ctypes.c_int, _VP, _VP]),
    ("whit_forward_wbits", ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int, _I64, _I64, _VP, _VP]),
    ("whit_forward_mse", ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int, _I64, _I64, _VP, _VP, _VP, _VP]),
    ("whit_posterior_variance", ctypes.c_int, [_VP, _VP, ctypes.c_int, _I64, _I64, _VP, _VP]),
    ("whit_host_ws_bytes", _SZ, [ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("whit_run_host", ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int,
                                     _VP, _VP, _VP, _VP, _I64, ctypes.c_int, _VP, _SZ, _VP]),
    ("whit_run_host_wbits", ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int,
                                           _VP, _VP, _VP, _VP, _I64, ctypes.c_int, _VP, _SZ, _VP]),
    ("whit_host_ws_bytes_bands", _SZ, [ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int]),
    ("whit_run_host_bands", ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int, _I64, _I64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _VP, _VP, _VP, _VP, _I64, ctypes.c_int, _VP, _SZ, _VP]),
]


class WhitError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.whit_last_error().decode() if _lib is not None else ""
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libwhit.so not found at {LIB_PATH}: build it with `make -C paper_2604_00048_b200` "
                          "or __graft_entry__.build() (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def lib():
    return _lib


def _check(status: int, where: str):
    if status != 0:
        raise WhitError(status, where)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return WHIT_F32
    if dt == torch.float64:
        return WHIT_F64
    raise TypeError(f"libwhit supports float32 / float64 planes, got {dt}")


def _stream_handle(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def whit_ws_bytes(d: int, T: int, B: int, dtype: torch.dtype, per_date: bool) -> int:
    return int(_lib.whit_ws_bytes(d, T, B, _dtype_code(dtype), int(per_date)))


def whit_ws_bytes_bands(d: int, T: int, B: int, C: int, dtype: torch.dtype, per_date: bool) -> int:
    return int(_lib.whit_ws_bytes_bands(d, T, B, C, _dtype_code(dtype), int(per_date)))


class Workspace:
    """Host handle (``whit_ws*``) plus the torch-owned device buffer it binds (C bands per pixel,
    or an irregular-grid workspace with ``times=True``)."""

    def __init__(self, d: int, T: int, B: int, dtype: torch.dtype, per_date: bool, device=None, stream=None,
                 C: int = 1, times: bool = False, buf: torch.Tensor | None = None):
        if times:
            nbytes = int(_lib.whit_ws_bytes_times_bands(d, T, B, C, _dtype_code(dtype), int(per_date)))
        else:
            nbytes = whit_ws_bytes_bands(d, T, B, C, dtype, per_date)
        if nbytes == 0:
            raise WhitError(1, f"workspace bytes(d={d}, T={T}, B={B}, C={C}, times={times})")
        self.d, self.T, self.B, self.C, self.dtype, self.per_date = d, T, B, C, dtype, per_date
        if buf is not None:  # caller-provided device buffer (uint8, >= nbytes, 256-B aligned)
            if buf.dtype != torch.uint8 or not buf.is_cuda or buf.numel() < nbytes:
                raise ValueError(f"workspace buffer must be a CUDA uint8 tensor of >= {nbytes} bytes")
            self.buf = buf
        else:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device or "cuda")
        self.nbytes = nbytes
        h = ctypes.c_void_p()
        if times:
            _check(_lib.whit_ws_create_times_bands(ctypes.byref(h), d, T, B, C, _dtype_code(dtype), int(per_date),
                                                   ctypes.c_void_p(self.buf.data_ptr()), nbytes,
                                                   _stream_handle(stream)),
                   "whit_ws_create_times_bands")
        else:
            _check(_lib.whit_ws_create_bands(ctypes.byref(h), d, T, B, C, _dtype_code(dtype), int(per_date),
                                             ctypes.c_void_p(self.buf.data_ptr()), nbytes, _stream_handle(stream)),
                   "whit_ws_create_bands")
        self.handle = h

    def set_twist(self, mode: int):
        """-1 auto, 0 never, 1 whenever the shape allows (whit_ws_set_twist)."""
        _check(_lib.whit_ws_set_twist(self.handle, int(mode)), "whit_ws_set_twist")

    def set_stream(self, stream=None):
        _check(_lib.whit_ws_set_stream(self.handle, _stream_handle(stream)), "whit_ws_set_stream")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.whit_ws_destroy(h)
            self.handle = None


def _shapes(ws: "Workspace", where: str, lam, *planes, C: int = 1):
    """Tensor-shape checks the pointer ABI cannot make: lambda's mode must match the workspace
    ((T-d, B) per date, (B,) scalar) and the [T][B] / [C][T][B] planes must have the workspace's shape."""
    T, B, d = ws.T, ws.B, ws.d
    for name, t in [("lambda", lam)] + [(n, t) for n, t, _ in planes]:
        if not t.is_contiguous():
            raise ValueError(f"{where}: {name} must be contiguous (the ABI reads a dense [T][B] plane)")
        if t.dtype != ws.dtype:
            raise TypeError(f"{where}: {name} dtype {t.dtype} != workspace dtype {ws.dtype}")
        if getattr(ws, "device_check", True) and not t.is_cuda:
            raise ValueError(f"{where}: {name} must be a CUDA tensor (no CPU fallback)")
    want = (T - d, B) if ws.per_date else (B,)
    if tuple(lam.shape) != want:
        raise ValueError(f"{where}: lambda shape {tuple(lam.shape)} != {want} "
                         f"({'per-date' if ws.per_date else 'scalar'} workspace)")
    for name, t, shp in planes:
        exp = {"TB": (T, B), "CTB": (C, T, B) if C > 1 else None}[shp]
        if exp is None:
            ok = tuple(t.shape) in ((T, B), (1, T, B))
        else:
            ok = tuple(t.shape) == exp
        if not ok:
            raise ValueError(f"{where}: {name} shape {tuple(t.shape)} does not match the workspace (T={T}, B={B}, C={C})")


def whit_forward(y, w, lam, d: int, T: int, B: int, z, ws: Workspace):
    _shapes(ws, "whit_forward", lam, ("y", y, "TB"), ("w", w, "TB"), ("z", z, "TB"))
    _check(_lib.whit_forward(_ptr(y), _ptr(w), _ptr(lam), d, T, B, _ptr(z), ws.handle), "whit_forward")


def whit_forward_bands(y, w, lam, d: int, T: int, B: int, C: int, z, ws: Workspace):
    _shapes(ws, "whit_forward_bands", lam, ("y", y, "CTB"), ("w", w, "TB"), ("z", z, "CTB"), C=C)
    _check(_lib.whit_forward_bands(_ptr(y), _ptr(w), _ptr(lam), d, T, B, C, _ptr(z), ws.handle), "whit_forward_bands")


def whit_backward_bands(grad_z, ws: Workspace, z, grad_y, grad_lambda):
    _shapes(ws, "whit_backward_bands", grad_lambda, ("grad_z", grad_z, "CTB"), ("grad_y", grad_y, "CTB"), C=ws.C)
    _check(_lib.whit_backward_bands(_ptr(grad_z), ws.handle, _ptr(z), _ptr(grad_y), _ptr(grad_lambda)),
           "whit_backward_bands")


def whit_backward(grad_z, ws: Workspace, z, grad_y, grad_lambda):
    _shapes(ws, "whit_backward", grad_lambda, ("grad_z", grad_z, "CTB"), ("grad_y", grad_y, "CTB"), C=ws.C)
    _check(_lib.whit_backward(_ptr(grad_z), ws.handle, _ptr(z), _ptr(grad_y), _ptr(grad_lambda)), "whit_backward")


def whit_grad_w(ws: Workspace, y, z, grad_y, grad_w):
    """dL/dw = sum over bands of (grad_y / w) (y - z), 0 where w = 0 (after whit_backward)."""
    _check(_lib.whit_grad_w(ws.handle, _ptr(y), _ptr(z), _ptr(grad_y), _ptr(grad_w)), "whit_grad_w")


def whit_forward_times(y, w, lam, times, d: int, T: int, B: int, z, ws: Workspace):
    _shapes(ws, "whit_forward_times", lam, ("y", y, "TB"), ("w", w, "TB"), ("times", times, "TB"), ("z", z, "TB"))
    _check(_lib.whit_forward_times(_ptr(y), _ptr(w), _ptr(lam), _ptr(times), d, T, B, _ptr(z), ws.handle),
           "whit_forward_times")


def whit_forward_times_bands(y, w, lam, times, d: int, T: int, B: int, C: int, z, ws: Workspace):
    """C bands per pixel on uneven dates (y, z: [C][T][B]; w, lam, times shared)."""
    _shapes(ws, "whit_forward_times_bands", lam, ("y", y, "CTB"), ("w", w, "TB"), ("times", times, "TB"),
            ("z", z, "CTB"), C=C)
    _check(_lib.whit_forward_times_bands(_ptr(y), _ptr(w), _ptr(lam), _ptr(times), d, T, B, C, _ptr(z), ws.handle),
           "whit_forward_times_bands")


def whit_pack_mask(w, bits=None, stream=None):
    """Pack a 0/1 [T][B] weight plane into uint32 bits [ceil(T/32)][B] (as int32 tensor storage)."""
    T, B = w.shape
    if bits is None:
        bits = torch.empty(((T + 31) // 32, B), dtype=torch.int32, device=w.device)
    _check(_lib.whit_pack_mask(_ptr(w), T, B, _dtype_code(w.dtype), _ptr(bits), _stream_handle(stream)), "whit_pack_mask")
    return bits


def whit_forward_wbits(y, wbits, lam, d: int, T: int, B: int, z, ws: Workspace):
    _shapes(ws, "whit_forward_wbits", lam, ("y", y, "TB"), ("z", z, "TB"))
    _check(_lib.whit_forward_wbits(_ptr(y), _ptr(wbits), _ptr(lam), d, T, B, _ptr(z), ws.handle), "whit_forward_wbits")


def whit_forward_mse(y, w, lam, loss_w, d: int, T: int, B: int, z, grad_z, loss, ws: Workspace):
    _shapes(ws, "whit_forward_mse", lam, ("y", y, "TB"), ("w", w, "TB"), ("loss_w", loss_w, "TB"), ("z", z, "TB"),
            ("grad_z", grad_z, "TB"))
    _check(_lib.whit_forward_mse(_ptr(y), _ptr(w), _ptr(lam), _ptr(loss_w), d, T, B, _ptr(z), _ptr(grad_z), _ptr(loss),
                                 ws.handle), "whit_forward_mse")


def whit_posterior_variance(w, lam, d: int, T: int, B: int, var, ws: Workspace):
    _shapes(ws, "whit_posterior_variance", lam, ("w", w, "TB"), ("var", var, "TB"))
    _check(_lib.whit_posterior_variance(_ptr(w), _ptr(lam), d, T, B, _ptr(var), ws.handle), "whit_posterior_variance")


def whit_failures(ws: Workspace, with_info: bool = False):
    n = ctypes.c_int64(0)
    if with_info:
        info = (ctypes.c_int32 * ws.B)()
        _check(_lib.whit_failures(ws.handle, ctypes.byref(n), info), "whit_failures")
        import numpy as np
        return int(n.value), np.frombuffer(info, dtype=np.int32).copy()
    _check(_lib.whit_failures(ws.handle, ctypes.byref(n), None), "whit_failures")
    return int(n.value)


def whit_wbits_detected(ws: Workspace):
    """(warps that read W as bits, warps) of the last plain whit_forward on ws (synchronises)."""
    nb, nw = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(_lib.whit_wbits_detected(ws.handle, ctypes.byref(nb), ctypes.byref(nw)), "whit_wbits_detected")
    return int(nb.value), int(nw.value)


def whit_twist_groups(ws: Workspace):
    """(groups of 32 series solved on the twisted path, groups) of the last whit_forward (synchronises)."""
    nt, ng = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(_lib.whit_twist_groups(ws.handle, ctypes.byref(nt), ctypes.byref(ng)), "whit_twist_groups")
    return int(nt.value), int(ng.value)


def whit_host_ws_bytes(d: int, T: int, chunk: int, dtype, per_date: bool, nbuf: int) -> int:
    return int(_lib.whit_host_ws_bytes(d, T, chunk, _dtype_code(dtype), int(per_date), nbuf))


def whit_run_host_bands(y, w, lam, grad_z, d: int, z, grad_y=None, grad_lambda=None, info=None, *,
                        chunk: int = 8192, nbuf: int = 3, dev_buf=None, stream=None):
    """Streaming executor for C bands per pixel in HOST memory: y, grad_z, z, grad_y (C, T, B); w (T, B);
    lam (T-d, B) or (B,).  Returns the device buffer (reuse it across calls)."""
    C, T, B = y.shape
    per_date = lam.dim() == 2
    need = int(_lib.whit_host_ws_bytes_bands(d, T, min(chunk, B), C, _dtype_code(y.dtype), int(per_date), nbuf))
    if need == 0:
        raise WhitError(1, "whit_host_ws_bytes_bands")
    if dev_buf is None or dev_buf.numel() < need:
        dev_buf = torch.empty(need, dtype=torch.uint8, device="cuda")
    for t in (y, w, lam, z) + ((grad_z, grad_y, grad_lambda) if grad_z is not None else ()):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("whit_run_host_bands takes contiguous HOST tensors")
    _check(_lib.whit_run_host_bands(_ptr(y), _ptr(w), _ptr(lam), _ptr(grad_z), d, T, B, C, _dtype_code(y.dtype),
                                    int(per_date), _ptr(z), _ptr(grad_y), _ptr(grad_lambda), _ptr(info),
                                    min(chunk, B), nbuf, ctypes.c_void_p(dev_buf.data_ptr()), dev_buf.numel(),
                                    _stream_handle(stream)), "whit_run_host_bands")
    return dev_buf


def whit_run_host(y, w, lam, grad_z, d: int, z, grad_y=None, grad_lambda=None, info=None, *, chunk: int = 16384,
                  nbuf: int = 3, dev_buf=None, stream=None, wbits=None):
    """Streaming executor over HOST (CPU, ideally pinned) tensors in [T][B] layout.

    ``dev_buf`` (uint8 CUDA tensor of >= whit_host_ws_bytes bytes) is allocated if not given.
    Returns the device buffer (reuse it across calls).  Asynchronous on ``stream``.  With ``wbits`` (HOST
    int32/uint32 [ceil(T/32)][B], the bit-packed binary W) ``w`` is ignored and whit_run_host_wbits runs.
    """
    T, B = y.shape
    per_date = lam.dim() == 2
    need = whit_host_ws_bytes(d, T, min(chunk, B), y.dtype, per_date, nbuf)
    if dev_buf is None or dev_buf.numel() < need:
        dev_buf = torch.empty(need, dtype=torch.uint8, device="cuda")
    wt = wbits if wbits is not None else w
    for t in (y, wt, lam, z) + ((grad_z, grad_y, grad_lambda) if grad_z is not None else ()):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("whit_run_host takes contiguous HOST tensors")
    fn = _lib.whit_run_host_wbits if wbits is not None else _lib.whit_run_host
    _check(fn(_ptr(y), _ptr(wt), _ptr(lam), _ptr(grad_z), d, T, B, _dtype_code(y.dtype), int(per_date),
                              _ptr(z), _ptr(grad_y), _ptr(grad_lambda), _ptr(info), min(chunk, B), nbuf,
                              ctypes.c_void_p(dev_buf.data_ptr()), dev_buf.numel(), _stream_handle(stream)),
           "whit_run_host")
    return dev_buf
