import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_00048_b200 as P
import synth
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T, B = 40, 64
x = synth.make_inputs("toy", B=B, T=T, d=d, lam_mode="per_date", device="cuda", seed=1)
tt = synth.make_times(B, T, device="cuda")
ws = P.Workspace(d, T, B, torch.float32, True, times=True)
z = torch.empty_like(x["y"])
t0 = time.time()
P.whit_forward_times(x["y"], x["w"], x["lam"], tt, d, T, B, z, ws)
torch.cuda.synchronize()
print("fwd ok", time.time() - t0, z[:5, 0])
gy, gl = torch.empty_like(z), torch.empty_like(x["lam"])
P.whit_backward(x["g"], ws, z, gy, gl)
torch.cuda.synchronize()
print("bwd ok", time.time() - t0, gy[:5, 0])
