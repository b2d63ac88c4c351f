"""dev: run one tiny twisted forward (+ backward) and report the CUDA status (stage-bisection builds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_00048_b200 as P
import synth
d, T, B = int(os.environ.get("D", "1")), 128, 64
x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda")
ws = P.Workspace(d, T, B, torch.float32, True)
ws.set_twist(1)
z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
try:
    P.whit_forward(x["y"], x["w"], x["lam"], d, T, B, z, ws)
    torch.cuda.synchronize()
    print(os.environ.get("WHIT_LIB_PATH", "main"), "forward ok", P.whit_twist_groups(ws))
    P.whit_backward(x["g"], ws, z, gy, gl)
    torch.cuda.synchronize()
    print("backward ok")
except Exception as e:
    print(os.environ.get("WHIT_LIB_PATH", "main"), "ERROR", e)
