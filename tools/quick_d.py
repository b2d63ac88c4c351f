"""Quick device timing of whit_forward + whit_backward for a given d (dev tool): python quick_d.py d [T] [B]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_00048_b200 as P
import synth

d = int(sys.argv[1]) if len(sys.argv) > 1 else 3
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3288
B = int(sys.argv[3]) if len(sys.argv) > 3 else 262144
x = synth.make_inputs(os.environ.get("QD_W", "hetero"), B=B, T=T, d=d, device="cuda")
y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
ws = P.Workspace(d, T, B, torch.float32, lam.dim() == 2)
if os.environ.get("QD_WBITS"):  # forward with the bit-packed W (the backward then reads the bits too)
    bits = P.whit_pack_mask(w)
    P.whit_forward = lambda y, w, *a: P.whit_forward_wbits(y, bits, *a)
z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
for _ in range(3):
    P.whit_forward(y, w, lam, d, T, B, z, ws)
    P.whit_backward(g, ws, z, gy, gl)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tf, tb = [], []
for _ in range(5):
    e[0].record()
    P.whit_forward(y, w, lam, d, T, B, z, ws)
    e[1].record()
    P.whit_backward(g, ws, z, gy, gl)
    e[2].record()
    torch.cuda.synchronize()
    tf.append(e[0].elapsed_time(e[1]))
    tb.append(e[1].elapsed_time(e[2]))
print(f"d={d} T={T} B={B}: fwd {min(tf):.3f} bwd {min(tb):.3f} ms -> {B / (min(tf) + min(tb)) * 1e3 / 1e6:.2f} M series/s;"
      f" failures {P.whit_failures(ws)}")
