"""Quick timing of the irregular-grid path (dev tool): python quick_irr.py d [T] [B]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_00048_b200 as P
import synth

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
T = int(sys.argv[2]) if len(sys.argv) > 2 else 350
B = int(sys.argv[3]) if len(sys.argv) > 3 else 262144
x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", mask="bernoulli")
tt = synth.make_times(B, T, device="cuda")
ws = P.Workspace(d, T, B, torch.float32, True, times=True)
z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
step = lambda: (P.whit_forward_times(x["y"], x["w"], x["lam"], tt, d, T, B, z, ws),
                P.whit_backward(x["g"], ws, z, gy, gl))
for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"irregular d={d} T={T} B={B}: {ms:.3f} ms/step -> {B / ms * 1e3 / 1e6:.1f} M series/s")
