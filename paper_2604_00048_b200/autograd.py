"""Thin ``torch.autograd.Function`` over libwhit (the paper's custom autograd op).

``smooth(y, w, lam, d)`` is the layer ``z = f_Lambda(x | W, D)`` of P:74:
forward = ``whit_forward`` (Eq. (3)), backward = ``whit_backward``
(Eq. (4)-(5)).  Torch is used for device memory and the current
stream only; all arithmetic runs in the library's kernels.

Tensors are time-outer ``(T, B)`` (``lam``: ``(T-d, B)`` per date or ``(B,)``
scalar per series), CUDA, contiguous, float32 or float64.  Variants:

* ``y`` of shape ``(C, T, B)``: C bands per pixel sharing ``w`` and ``lam``
  (``whit_forward_bands``, NEXT-1); ``lam``'s gradient is summed over bands;
* ``times=(T, B)``: uneven acquisition dates (``whit_forward_times``, NEXT-2; with bands:
  ``whit_forward_times_bands``).

``w`` gets a gradient when it requires one: ``dL/dw_t = sum_c u_t (y_t - z_t)`` (``whit_grad_w``; 0 at
``w_t = 0``, reading R-19).
"""
from __future__ import annotations

import torch

from . import _lib as L


def _pad_cols(x: torch.Tensor, Bp: int, value: float) -> torch.Tensor:
    if x.shape[-1] == Bp:
        return x.contiguous()
    pad = torch.full(x.shape[:-1] + (Bp - x.shape[-1],), value, dtype=x.dtype, device=x.device)
    return torch.cat([x, pad], dim=-1).contiguous()


class WhittakerFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, y, w, lam, d, times=None):
        if not (y.is_cuda and w.is_cuda and lam.is_cuda):
            raise ValueError("libwhit runs on CUDA tensors only (no CPU fallback)")
        bands = y.dim() == 3
        C = y.shape[0] if bands else 1
        T, B = y.shape[-2:]
        if w.shape != (T, B):
            raise ValueError(f"w must be (T, B) = {(T, B)}, got {tuple(w.shape)}")
        per_date = lam.dim() == 2
        if per_date and lam.shape != (T - d, B):
            raise ValueError(f"per-date lambda must be (T-d, B) = {(T - d, B)}, got {tuple(lam.shape)}")
        if not per_date and lam.shape != (B,):
            raise ValueError(f"scalar lambda must be (B,), got {tuple(lam.shape)}")
        if not (y.dtype == w.dtype == lam.dtype):
            raise TypeError("y, w, lambda must share a dtype")
        if times is not None and (times.shape != (T, B) or times.dtype != y.dtype):
            raise ValueError("times must be (T, B) of y's dtype")
        if T < d + 1:
            raise ValueError(f"T = {T} < d + 1 = {d + 1}: Omega needs at least d + 1 dates (P:87)")
        ctx.empty = B == 0
        if ctx.empty:  # an empty batch: nothing to solve (the C-ABI requires B >= 1)
            ctx.shapes = (w.shape, lam.shape)
            return torch.empty_like(y)
        q = 4 if y.dtype == torch.float32 else 2
        Bp = (B + q - 1) // q * q  # 16-byte row stride; padded series: w = 1, lam = 1, y = 0
        yp = _pad_cols(y, Bp, 0.0)
        wp = _pad_cols(w, Bp, 1.0)
        lp = _pad_cols(lam, Bp, 1.0)
        z = torch.empty_like(yp)
        if times is not None:
            tp = times if Bp == B else torch.cat(
                [times, torch.arange(T, dtype=times.dtype, device=times.device)[:, None].expand(T, Bp - B)], dim=1)
            tp = tp.contiguous()
            ws = L.Workspace(d, T, Bp, y.dtype, per_date, device=y.device, C=C, times=True)
            if bands:
                L.whit_forward_times_bands(yp, wp, lp, tp, d, T, Bp, C, z, ws)
            else:
                L.whit_forward_times(yp, wp, lp, tp, d, T, Bp, z, ws)
            keep = (wp, lp, z, tp)
        elif bands:
            ws = L.Workspace(d, T, Bp, y.dtype, per_date, device=y.device, C=C)
            L.whit_forward_bands(yp, wp, lp, d, T, Bp, C, z, ws)
            keep = (wp, lp, z)
        else:
            ws = L.Workspace(d, T, Bp, y.dtype, per_date, device=y.device)
            L.whit_forward(yp, wp, lp, d, T, Bp, z, ws)
            keep = (wp, lp, z)
        # tensors go through save_for_backward (no z -> grad_fn -> ctx -> z reference cycle keeping the
        # workspace alive, and autograd's version check guards w, lambda and z against in-place edits
        # before the backward the ABI requires them for); only the host handle is a ctx attribute
        need_w = ctx.needs_input_grad[1]
        ctx.save_for_backward(*keep, yp if need_w else None)
        ctx.ws, ctx.B, ctx.Bp, ctx.need_w = ws, B, Bp, need_w
        return z[..., :B] if Bp != B else z

    @staticmethod
    def backward(ctx, gz):
        if ctx.empty:
            new = lambda shape: gz.new_empty(shape)  # noqa: E731
            gw = new(ctx.shapes[0]) if ctx.needs_input_grad[1] else None
            return new(gz.shape), gw, new(ctx.shapes[1]), None, None
        ws = ctx.ws
        saved = ctx.saved_tensors
        wp, lp, z = saved[0], saved[1], saved[2]
        yp = saved[-1]
        gzp = _pad_cols(gz, ctx.Bp, 0.0)
        gy = torch.empty_like(gzp)
        gl = torch.empty_like(lp)
        ws.set_stream()
        L.whit_backward(gzp, ws, z, gy, gl)
        gw = None
        if ctx.need_w:
            gw = torch.empty_like(wp)
            L.whit_grad_w(ws, yp, z, gy, gw)
        B = ctx.B
        if ctx.Bp != B:
            gy, gl = gy[..., :B], gl[..., :B]
            gw = gw[..., :B] if gw is not None else None
        return gy, gw, gl, None, None


def smooth(y: torch.Tensor, w: torch.Tensor, lam: torch.Tensor, d: int = 2, times: torch.Tensor | None = None):
    """Differentiable Whittaker smoother (heteroscedastic if ``lam`` is (T-d, B)); see module doc."""
    return WhittakerFn.apply(y, w, lam, d, times)
