"""Small end-to-end exercise of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_00048_b200 as P
import synth

def fb(d, T, B, dtype, pd):
    x = synth.make_inputs("hetero", B=B, T=T, d=d, lam_mode="per_date" if pd else "scalar", device="cuda", dtype=dtype)
    # a non-binary weight in warp 1 (float path there, bit path elsewhere), a failing pivot in series 3
    # (cold exact-row replay) and an unobserved series 5 (count rule)
    x["w"][7, 40] = 0.5
    if pd:
        x["lam"][11, 3] = -1e6
    x["w"][:, 5] = 0
    ws = P.Workspace(d, T, B, dtype, pd)
    z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
    P.whit_forward(x["y"], x["w"], x["lam"], d, T, B, z, ws); P.whit_backward(x["g"], ws, z, gy, gl)
    var = torch.empty_like(x["y"])
    P.whit_posterior_variance(x["w"], x["lam"], d, T, B, var, ws)
    if d == 2:
        lw = (x["w"] == 0).to(dtype)
        gz, loss = torch.empty_like(z), torch.empty(B, dtype=dtype, device="cuda")
        P.whit_forward_mse(x["y"], x["w"], x["lam"], lw, d, T, B, z, gz, loss, ws)
    tt = synth.make_times(B, T, device="cuda", dtype=dtype)
    wt = P.Workspace(d, T, B, dtype, pd, times=True)
    P.whit_forward_times(x["y"], x["w"], x["lam"], tt, d, T, B, z, wt); P.whit_backward(x["g"], wt, z, gy, gl)
    P.whit_failures(ws)
    wb = (x["w"] != 0).to(dtype)
    bits = P.whit_pack_mask(wb)
    P.whit_forward_wbits(x["y"], bits, x["lam"], d, T, B, z, ws); P.whit_backward(x["g"], ws, z, gy, gl)
    gw = torch.empty_like(x["w"])
    P.whit_forward(x["y"], x["w"], x["lam"], d, T, B, z, ws); P.whit_backward(x["g"], ws, z, gy, gl)
    P.whit_grad_w(ws, x["y"], z, gy, gw)
    P.whit_wbits_detected(ws)

def bands(d, T, B, C, dtype, pd, times=False):
    x = synth.make_inputs_bands("hetero", C, B=B, T=T, d=d, lam_mode="per_date" if pd else "scalar", device="cuda", dtype=dtype)
    x["w"][:, 5] = 0
    ws = P.Workspace(d, T, B, dtype, pd, C=C, times=times)
    z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
    if times:
        tt = synth.make_times(B, T, device="cuda", dtype=dtype)
        P.whit_forward_times_bands(x["y"], x["w"], x["lam"], tt, d, T, B, C, z, ws)
    else:
        P.whit_forward_bands(x["y"], x["w"], x["lam"], d, T, B, C, z, ws)
    P.whit_backward_bands(x["g"], ws, z, gy, gl)

for d in (1, 2, 3):
    for dt in (torch.float32, torch.float64):
        for pd in (True, False):
            fb(d, 45, 136, dt, pd)
bands(2, 45, 72, 3, torch.float32, True)
bands(2, 45, 72, 10, torch.float32, False)
bands(3, 45, 72, 2, torch.float64, True)
bands(2, 45, 72, 10, torch.float32, True, times=True)
bands(1, 45, 72, 3, torch.float64, False, times=True)
h = {k: v.cpu().pin_memory() for k, v in synth.make_inputs("hetero", B=200, T=40, device="cuda").items() if k in ("y", "w", "lam", "g")}
oz, oy, ol = torch.empty_like(h["y"]).pin_memory(), torch.empty_like(h["y"]).pin_memory(), torch.empty_like(h["lam"]).pin_memory()
P.whit_run_host(h["y"], h["w"], h["lam"], h["g"], 2, oz, oy, ol, chunk=64, nbuf=3)
torch.cuda.synchronize()
print("sanitize workload done")
