#!/usr/bin/env python
"""BASELINE.json configs[4] "sweep": d in {1,2,3}, T in {128..8192}; libwhit (banded,
fwd+bwd) vs the paper's dense comparison (Table 1 "Full"): torch.linalg.solve on the
assembled dense Omega with autograd backward.  Context numbers, not the headline metric
(bench.py).  One JSON line per (d, T, mask, impl, B); OOM is reported as null (the paper's ∅).

Timing: CUDA events around K steps after W warm-up steps; inputs resident in HBM.  Masks: "bernoulli"
(toy-like iid, no trailing gap) and "s2" (Sentinel-2 revisits + seasonal clouds with a 90-day trailing gap
at every T).

--accuracy: instead of timing, report (not gate -- SURVEY §8(c): d = 3 is reported, not gated) the
libwhit errors per (d, T, mask, I/O dtype) on a seeded subsample against O2 (Algorithm 1 in long double,
every sampled series) and O1 (dense + refinement, a few series, T <= 2048): max over series of
max|z - z_ref| / max|y_obs|, and the normwise relative errors of dL/dy and dL/dlambda.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def time_steps(fn, steps, warmup):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def banded(x, d, dtype, steps, warmup):
    import torch
    import paper_2604_00048_b200 as P
    y, w, lam, g = (x[k].to(dtype) for k in ("y", "w", "lam", "g"))
    T, B = y.shape
    ws = P.Workspace(d, T, B, dtype, True)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)

    def step():
        P.whit_forward(y, w, lam, d, T, B, z, ws)
        P.whit_backward(g, ws, z, gy, gl)
    return time_steps(step, steps, warmup)


def dense(x, d, dtype, steps, warmup):
    """Paper's "Full" solver: dense Omega (B, T, T), torch.linalg.solve, autograd backward."""
    import torch
    y, w, lam, g = (x[k].to(dtype).t().contiguous() for k in ("y", "w", "lam", "g"))  # (B, T), (B, T-d)
    B, T = y.shape
    Dm = torch.zeros(T - d, T, dtype=dtype, device=y.device)
    c = [(-1) ** (d - j) * __import__("math").comb(d, j) for j in range(d + 1)]
    for j, cj in enumerate(c):
        Dm[torch.arange(T - d), torch.arange(T - d) + j] = cj
    lam = lam.clone().requires_grad_(True)
    yy = y.clone().requires_grad_(True)

    def step():
        Om = torch.diag_embed(w) + Dm.t() @ (lam[:, :, None] * Dm)
        z = torch.linalg.solve(Om, (w * yy)[:, :, None])[:, :, 0]
        torch.autograd.grad(z, (yy, lam), grad_outputs=g)
    return time_steps(step, steps, warmup)


def accuracy(d, T, mask, dtype, B=64, n_o1=4):
    """Errors of one (d, T, mask, dtype) point vs O2 (all B series) and O1 (n_o1 series, T <= 2048)."""
    import numpy as np
    import torch
    import synth
    import paper_2604_00048_b200 as P
    from oracle import banded as O2
    from oracle import whittaker as O1
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=dtype, mask=mask, seed=700 + d,
                          last_acq=T - 91)
    y, w, lam, g = (x[k] for k in ("y", "w", "lam", "g"))
    ws = P.Workspace(d, T, B, dtype, True)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
    P.whit_forward(y, w, lam, d, T, B, z, ws)
    P.whit_backward(g, ws, z, gy, gl)
    nfail = P.whit_failures(ws)
    h = {k: v.double().cpu().numpy().T.copy() for k, v in (("y", y), ("w", w), ("lam", lam), ("g", g))}
    res = {"z": z.double().cpu().numpy().T, "ybar": gy.double().cpu().numpy().T, "lambar": gl.double().cpu().numpy().T}
    ymax = np.max(np.where(h["w"] > 0, np.abs(h["y"]), 0.0), axis=1)

    def errs(ref, idx):
        ez = np.max(np.abs(res["z"][idx] - ref["z"].astype(float)), axis=1) / ymax[idx]
        ey = np.max(np.abs(res["ybar"][idx] - ref["ybar"].astype(float)), axis=1) / np.max(np.abs(ref["ybar"].astype(float)), axis=1)
        el = np.max(np.abs(res["lambar"][idx] - ref["lambar"].astype(float)), axis=1) / np.max(np.abs(ref["lambar"].astype(float)), axis=1)
        return float(ez.max()), float(ey.max()), float(el.max())

    zr, _, info = O2.forward_banded(h["y"], h["w"], h["lam"], d)
    yb, lb = O2.backward_banded(h["g"], h["w"], h["lam"], d, zr)
    e2 = errs({"z": zr, "ybar": yb, "lambar": lb}, np.arange(B))
    rec = {"config": "sweep-accuracy", "d": d, "T": T, "mask": mask, "io": "f32" if dtype == torch.float32 else "f64",
           "B": B, "failed": nfail, "obs_per_series_min": int((h["w"] > 0).sum(axis=1).min()),
           "vs_O2": {"z": e2[0], "ybar": e2[1], "lambar": e2[2], "series": B}}
    if T <= 2048:
        idx = np.linspace(0, B - 1, n_o1).astype(int)
        o = [O1.forward_backward(h["y"][b], h["w"][b], h["lam"][b], d, h["g"][b]) for b in idx]
        ref = {k: np.stack([oo[k] for oo in o]) for k in ("z", "ybar", "lambar")}
        e1 = errs(ref, idx)
        rec["vs_O1"] = {"z": e1[0], "ybar": e1[1], "lambar": e1[2], "series": int(n_o1)}
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="1,2,3")
    ap.add_argument("--Ts", default="128,256,512,1024,2048,4096,8192")
    ap.add_argument("--B-dense", type=int, default=4096)
    ap.add_argument("--B-banded", type=int, default=262144)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--masks", default="bernoulli,s2")
    ap.add_argument("--accuracy", action="store_true")
    args = ap.parse_args()
    import torch
    import synth
    masks = args.masks.split(",")
    if args.accuracy:
        for d in [int(v) for v in args.orders.split(",")]:
            for T in [int(v) for v in args.Ts.split(",")]:
                for mask in masks:
                    for dt in (torch.float32, torch.float64):
                        print(json.dumps(accuracy(d, T, mask, dt)), flush=True)
        return
    for d in [int(v) for v in args.orders.split(",")]:
        for T in [int(v) for v in args.Ts.split(",")]:
            for mask in masks:
                for impl, B, dt in (("libwhit", args.B_banded, torch.float32), ("libwhit", args.B_dense, torch.float32),
                                    ("dense_torch_solve", args.B_dense, torch.float32),
                                    ("dense_torch_solve", args.B_dense, torch.float64)):
                    if impl == "dense_torch_solve" and mask != masks[0]:
                        continue  # the dense comparison (context only) once per (d, T)
                    rec = {"config": "sweep", "d": d, "T": T, "mask": mask, "B": B, "impl": impl,
                           "io": "f32" if dt == torch.float32 else "f64"}
                    try:
                        x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=dt,
                                              mask=mask, seed=300 + d, last_acq=T - 91)
                        ms = (banded if impl == "libwhit" else dense)(x, d, dt, args.steps, args.warmup)
                        rec.update(ms_per_step=ms, series_per_s=B / (ms / 1e3))
                    except torch.OutOfMemoryError:
                        rec.update(ms_per_step=None, series_per_s=None, oom=True)
                    finally:
                        x = None
                        torch.cuda.empty_cache()
                    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
