#!/usr/bin/env python
"""BASELINE.json configs[4] "sweep": d in {1,2,3}, T in {128..8192}; libwhit (banded,
fwd+bwd) vs the paper's dense comparison (Table 1 "Full"): torch.linalg.solve on the
assembled dense Omega with autograd backward.  Context numbers, not the headline metric
(bench.py).  One JSON line per (d, T, impl, B); OOM is reported as null (the paper's ∅).

Timing: CUDA events around K steps after W warm-up steps; inputs resident in HBM.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="1,2,3")
    ap.add_argument("--Ts", default="128,256,512,1024,2048,4096,8192")
    ap.add_argument("--B-dense", type=int, default=4096)
    ap.add_argument("--B-banded", type=int, default=262144)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import torch
    import synth
    for d in [int(v) for v in args.orders.split(",")]:
        for T in [int(v) for v in args.Ts.split(",")]:
            for impl, B, dt in (("libwhit", args.B_banded, torch.float32), ("libwhit", args.B_dense, torch.float32),
                                ("dense_torch_solve", args.B_dense, torch.float32),
                                ("dense_torch_solve", args.B_dense, torch.float64)):
                rec = {"config": "sweep", "d": d, "T": T, "B": B, "impl": impl,
                       "io": "f32" if dt == torch.float32 else "f64"}
                try:
                    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=dt,
                                          mask="bernoulli", seed=300 + d)
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
