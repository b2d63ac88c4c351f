"""Quick device timing of the multi-band (shared factor) path vs independent band-series (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_00048_b200 as P
import synth

C = int(sys.argv[1]) if len(sys.argv) > 1 else 10
B = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
d = int(os.environ.get("QB_D", "2"))
x = synth.make_inputs_bands("hetero", C, B=B, d=d, device="cuda")
x.pop("lam_mode", None)
y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
_, T, _ = y.shape
ws = P.Workspace(d, T, B, torch.float32, True, C=C)
z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
def step():
    P.whit_forward_bands(y, w, lam, d, T, B, C, z, ws); P.whit_backward_bands(g, ws, z, gy, gl)
for _ in range(3): step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tf, tb = [], []
for _ in range(5):
    ev[0].record(); P.whit_forward_bands(y, w, lam, d, T, B, C, z, ws); ev[1].record(); P.whit_backward_bands(g, ws, z, gy, gl); ev[2].record()
    torch.cuda.synchronize(); tf.append(ev[0].elapsed_time(ev[1])); tb.append(ev[1].elapsed_time(ev[2]))
ms = min(tf) + min(tb)
print(f"bands C={C} pixels={B} T={T}: fwd {min(tf):.3f} bwd {min(tb):.3f} ms -> {B*C/ms*1e3/1e6:.2f} M band-series/s "
      f"({B/ms*1e3/1e6:.2f} M pixels/s)")
if os.environ.get("QB_ONLY"):
    sys.exit(0)
# independent-series baseline on the same band-series (w, lambda replicated per band)
del ws, z, gy, gl
x.clear()
torch.cuda.empty_cache()
ys = y.permute(1, 0, 2).reshape(T, C * B).contiguous(); gs = g.permute(1, 0, 2).reshape(T, C * B).contiguous()
ws_ = w.repeat(1, C).contiguous(); ls = lam.repeat(1, C).contiguous()
del y, g, w, lam
torch.cuda.empty_cache()
W = P.Workspace(d, T, C * B, torch.float32, True)
z1, gy1, gl1 = torch.empty_like(ys), torch.empty_like(ys), torch.empty_like(ls)
def step1():
    P.whit_forward(ys, ws_, ls, d, T, C * B, z1, W); P.whit_backward(gs, W, z1, gy1, gl1)
for _ in range(2): step1()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): step1()
e1.record(); torch.cuda.synchronize()
ms1 = e0.elapsed_time(e1) / 3
print(f"independent band-series C*B={C*B}: {ms1:.3f} ms -> {C*B/ms1*1e3/1e6:.2f} M band-series/s; shared-factor speedup {ms1/ms:.2f}x")
