"""Seeded synthetic Sentinel-2-shaped inputs for the Whittaker hot path.

This module holds NONE of the method's arithmetic: it only draws inputs
(``y``, ``w``, ``lambda``, upstream cotangent ``g``).  Both the CUDA path's
tests/bench and the CPU oracle consume its output; the oracle is always fed
the very tensors (copied to host) that the GPU saw, so no RNG bit-matching
between devices is needed.  It is nevertheless device-independent for the
integer parts (a counter-based hash keyed on (seed, stream, global series id,
date)), so the mask and the per-series parameters of series ``b`` are the same
whatever rank, shard or device generates them.

Layout: time-outer ``[T][B]`` (element (t, b) at ``t*B + b``), the layout the
library consumes.  Per-date lambda is ``[T-d][B]``; scalar lambda is ``[B]``.

Recipe (DESIGN.md §4 states it with its sources):

* daily grid t = 0..T-1 <-> 2016-01-01.. (T = 3288 ends 2024-12-31);
* Sentinel-2 acquisitions: S2A every 10 days from a per-pixel orbit phase, S2B
  with a 5-day offset from t = 547 (2017-07-01), 30 % of pixels get a second
  overlapping orbit; no acquisitions from t = 3197 (2024-10-02, the paper's
  last date) -> a ~90-day trailing gap;
* clouds: an acquisition is cloudy with probability
  0.45 + 0.30 cos(2 pi (doy - 15) / 365) (cloudy winters); w = 1 on clear
  acquisitions, 0 elsewhere; at least d+1 clear days are forced;
* y: NDVI-like seasonal curve base + amp exp(-((doy-peak)/45)^2/2) + N(0, s^2),
  5 % of clear days get an undetected-cloud dip U[0.1, 0.4] (heteroscedastic
  outliers); masked days carry a bright cloud value;
* lambda: toy/homo scalar per series, log10 lam ~ U[0,4] / U[1,5]; per-date
  ``log10 lam_r = mu + 0.5 sin(2 pi doy_r/365 + phi) + 0.3 sin(2 pi r/P + psi)``,
  mu ~ U[2, 4.5], clipped to [1, 1e5] (the gated range, BASELINE.json);
* g ~ N(0, 1) iid (any cotangent exercises the backward identically).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

BASE_SEED = 260400048
T_DAILY = 3288          # 2016-01-01 .. 2024-12-31
T_LAST_ACQ = 3197       # 2024-10-02: no acquisitions from here on
T_S2B = 547             # 2017-07-01

_M32 = 0xFFFFFFFF


@dataclass(frozen=True)
class Config:
    name: str
    B: int
    T: int
    d: int
    lam_mode: str      # "scalar" | "per_date"
    mask: str          # "bernoulli" | "s2"
    backward: bool
    seed_offset: int


# BASELINE.json "configs" (the sweep/s2tile shapes are built by the bench on demand).
CONFIGS = {
    "toy": Config("toy", 1024, 365, 2, "scalar", "bernoulli", False, 0),
    "homo": Config("homo", 65536, T_DAILY, 2, "scalar", "s2", True, 1),
    "hetero": Config("hetero", 262144, T_DAILY, 2, "per_date", "s2", True, 2),
}


def _mix(x: torch.Tensor) -> torch.Tensor:
    """32-bit avalanche hash on int64 tensors holding values in [0, 2^32)."""
    x = x & _M32
    x = x ^ (x >> 16)
    x = (x * 0x45D9F3B) & _M32
    x = x ^ (x >> 16)
    x = (x * 0x45D9F3B) & _M32
    x = x ^ (x >> 16)
    return x


def _key(*parts) -> torch.Tensor:
    h = None
    for p in parts:
        p = p if isinstance(p, torch.Tensor) else torch.tensor(p, dtype=torch.int64)
        h = _mix(p & _M32) if h is None else _mix(h ^ _mix((p + 0x9E3779B9) & _M32))
    return h


def _uniform(h: torch.Tensor) -> torch.Tensor:
    """(0, 1) float64 from a 32-bit hash."""
    return (h.to(torch.float64) + 0.5) / 4294967296.0


class _Stream:
    def __init__(self, seed: int, series: torch.Tensor):
        self.seed = seed
        self.series = series  # (B,) int64 global series ids

    def per_series(self, stream: int) -> torch.Tensor:
        return _uniform(_key(self.seed, stream, self.series))

    def per_cell(self, stream: int, t: torch.Tensor) -> torch.Tensor:
        # t: (R, 1) int64 -> (R, B)
        k = _key(self.seed, stream)
        k = _mix(k ^ _mix((self.series[None, :] + 0x9E3779B9) & _M32))
        k = _mix(k ^ _mix((t * 0x632BE5AB + 0x7F4A7C15) & _M32))
        return _uniform(k)


def _normal(u1: torch.Tensor, u2: torch.Tensor) -> torch.Tensor:
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def make_inputs(cfg: Config | str, *, B: int | None = None, T: int | None = None,
                d: int | None = None, seed: int | None = None, series_offset: int = 0,
                device="cpu", dtype=torch.float32, with_g: bool = True,
                lam_mode: str | None = None, mask: str | None = None,
                lam_max: float = 1e5, row_chunk_elems: int = 1 << 24, series_ids=None,
                last_acq: int | None = None) -> dict:
    """Draw one shard ``[series_offset, series_offset + B)`` of a config (or the
    explicit global ``series_ids``, e.g. a sample spread over the batch).

    Returns ``{"y": (T,B), "w": (T,B), "lam": (T-d,B) or (B,), "g": (T,B)}`` on
    ``device`` in ``dtype`` (float32 or float64), plus the config echo.
    ``last_acq``: first date without acquisitions for the "s2" mask (default 3197, 2024-10-02, which
    gives T = 3288 its 90-day trailing gap; the sweep passes T - 91 to keep that gap at any T).
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    B = cfg.B if B is None else B
    T = cfg.T if T is None else T
    d = cfg.d if d is None else d
    lam_mode = cfg.lam_mode if lam_mode is None else lam_mode
    mask = cfg.mask if mask is None else mask
    seed = BASE_SEED + cfg.seed_offset if seed is None else seed
    dev = torch.device(device)
    if series_ids is not None:
        ser = torch.as_tensor(series_ids, dtype=torch.int64, device=dev)
        B = int(ser.numel())
    else:
        ser = torch.arange(series_offset, series_offset + B, dtype=torch.int64, device=dev)
    S = _Stream(seed, ser)

    # per-series parameters
    phase = torch.floor(S.per_series(1) * 10).to(torch.int64)
    phase2 = torch.floor(S.per_series(2) * 10).to(torch.int64)
    has2 = S.per_series(3) < 0.30
    base = 0.15 + 0.15 * S.per_series(4)
    amp = 0.30 + 0.30 * S.per_series(5)
    peak = 150.0 + 70.0 * S.per_series(6)
    sig = 0.01 + 0.04 * S.per_series(7)
    mu = 2.0 + 2.5 * S.per_series(8)
    phi = 2 * math.pi * S.per_series(9)
    per = 20.0 + 100.0 * S.per_series(10)
    psi = 2 * math.pi * S.per_series(11)

    y = torch.empty((T, B), dtype=dtype, device=dev)
    w = torch.empty((T, B), dtype=dtype, device=dev)
    g = torch.empty((T, B), dtype=dtype, device=dev) if with_g else None
    if lam_mode == "per_date":
        lam = torch.empty((T - d, B), dtype=dtype, device=dev)
    elif lam_mode == "scalar":
        lo, hi = (0.0, 4.0) if mask == "bernoulli" else (1.0, 5.0)
        lam = torch.pow(10.0, lo + (hi - lo) * S.per_series(12)).to(dtype)
    else:
        raise ValueError(lam_mode)

    # forced clear days (>= d+1 observations per series)
    if mask == "s2":
        forced = [phase + 10 * k + 1 for k in range(d + 1)]
    else:
        forced = [torch.full_like(phase, v) for v in (0, T // 2, T - 1)][: max(d + 1, 3)]

    R = max(1, row_chunk_elems // max(B, 1))
    for t0 in range(0, T, R):
        t1 = min(T, t0 + R)
        t = torch.arange(t0, t1, dtype=torch.int64, device=dev)[:, None]
        tf = t.to(torch.float64)
        doy = torch.remainder(tf, 365.25)
        if mask == "s2":
            acq = (torch.remainder(t - phase - 1, 10) == 0) & (t >= 1)
            acq |= (torch.remainder(t - phase - 6, 10) == 0) & (t >= T_S2B)
            acq |= has2 & (torch.remainder(t - phase2 - 3, 10) == 0) & (t >= 1)
            acq &= t < (T_LAST_ACQ if last_acq is None else last_acq)
            pc = 0.45 + 0.30 * torch.cos(2 * math.pi * (doy - 15.0) / 365.0)
            clear = acq & (S.per_cell(20, t) > pc)
        else:
            clear = S.per_cell(20, t) < 0.7
        for f in forced:
            clear |= (t == f[None, :]) & (t < T)
        dd = torch.remainder(doy - peak + 182.625, 365.25) - 182.625
        curve = base + amp * torch.exp(-0.5 * (dd / 45.0) ** 2)
        noise = sig * _normal(S.per_cell(21, t), S.per_cell(22, t))
        dip = torch.where(S.per_cell(23, t) < 0.05, 0.1 + 0.3 * S.per_cell(24, t),
                          torch.zeros((), dtype=torch.float64, device=dev))
        yy = curve + noise - dip
        cloud = 0.2 + 0.4 * S.per_cell(25, t)
        y[t0:t1] = torch.where(clear, yy, curve + cloud).to(dtype)
        w[t0:t1] = clear.to(dtype)
        if with_g:
            g[t0:t1] = _normal(S.per_cell(26, t), S.per_cell(27, t)).to(dtype)
        if lam_mode == "per_date":
            r1 = min(t1, T - d)
            if r1 > t0:
                tr = t[: r1 - t0]
                trf = tr.to(torch.float64)
                l10 = (mu + 0.5 * torch.sin(2 * math.pi * torch.remainder(trf, 365.25) / 365.0 + phi)
                       + 0.3 * torch.sin(2 * math.pi * trf / per + psi))
                l10 = torch.clamp(l10, 0.0, math.log10(lam_max))
                lam[t0:r1] = torch.pow(10.0, l10).to(dtype)
    return {"y": y, "w": w, "lam": lam, "g": g, "B": B, "T": T, "d": d,
            "lam_mode": lam_mode, "seed": seed, "series_offset": series_offset}


def series_major(x: torch.Tensor):
    """[T][B] -> [B][T] numpy float64 (for the oracle, which is series-major)."""
    import numpy as np
    a = x.detach().to("cpu", torch.float64).numpy()
    return np.ascontiguousarray(a.T) if a.ndim == 2 else a


def make_inputs_bands(cfg: Config | str, C: int, *, B: int | None = None, T: int | None = None,
                      d: int | None = None, seed: int | None = None, series_offset: int = 0, device="cpu",
                      dtype=torch.float32, lam_mode: str | None = None, mask: str | None = None,
                      row_chunk_elems: int = 1 << 24) -> dict:
    """C reflectance bands per pixel sharing the mask and lambda (BASELINE 's2tile' shape):
    band c = a_c (ndvi - 0.45) / 0.2 + b_c + 0.1 N(0, 1) (standardised-reflectance-like),
    a_c in [-1, 1], b_c in [-0.5, 0.5] fixed per band.  Returns y, g as [C][T][B]; w [T][B];
    lam [T-d][B] or [B]."""
    base = make_inputs(cfg, B=B, T=T, d=d, seed=seed, series_offset=series_offset, device=device,
                       dtype=torch.float64, lam_mode=lam_mode, mask=mask, row_chunk_elems=row_chunk_elems)
    T, B, d = base["T"], base["B"], base["d"]
    dev = torch.device(device)
    ser = torch.arange(series_offset, series_offset + B, dtype=torch.int64, device=dev)
    S = _Stream(base["seed"], ser)
    y = torch.empty((C, T, B), dtype=dtype, device=dev)
    g = torch.empty((C, T, B), dtype=dtype, device=dev)
    R = max(1, row_chunk_elems // max(B, 1))
    for c in range(C):
        kc = _uniform(_key(base["seed"], 900 + c)).item()
        a_c = -1.0 + 2.0 * kc
        b_c = -0.5 + _uniform(_key(base["seed"], 950 + c)).item()
        for t0 in range(0, T, R):
            t1 = min(T, t0 + R)
            t = torch.arange(t0, t1, dtype=torch.int64, device=dev)[:, None]
            nz = _normal(S.per_cell(100 + 4 * c, t), S.per_cell(101 + 4 * c, t))
            y[c, t0:t1] = (a_c * (base["y"][t0:t1] - 0.45) / 0.2 + b_c + 0.1 * nz).to(dtype)
            g[c, t0:t1] = _normal(S.per_cell(102 + 4 * c, t), S.per_cell(103 + 4 * c, t)).to(dtype)
    return {"y": y, "w": base["w"].to(dtype), "lam": base["lam"].to(dtype), "g": g, "B": B, "T": T, "d": d, "C": C,
            "lam_mode": base["lam_mode"], "seed": base["seed"], "series_offset": series_offset}


def make_times(B: int, T: int, *, seed: int = BASE_SEED + 7, series_offset: int = 0, device="cpu",
               dtype=torch.float32, max_gap: int = 12) -> torch.Tensor:
    """Per-series increasing acquisition days [T][B] for the irregular-grid path: cumulative
    gaps uniform in {1..max_gap} (Sentinel-2 revisits are 5-10 days; unaligned series,
    P:26), first date in [0, 10)."""
    dev = torch.device(device)
    ser = torch.arange(series_offset, series_offset + B, dtype=torch.int64, device=dev)
    S = _Stream(seed, ser)
    t = torch.arange(T, dtype=torch.int64, device=dev)[:, None]
    gaps = 1 + torch.floor(S.per_cell(60, t) * max_gap)
    gaps[0] = torch.floor(S.per_series(61) * 10)
    return torch.cumsum(gaps, dim=0).to(dtype)
