"""Quick device timing of whit_forward / whit_backward at a config (dev tool, not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_00048_b200 as P
import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "hetero"
dtype = torch.float64 if (len(sys.argv) > 2 and sys.argv[2] == "f64") else torch.float32
QB = int(os.environ.get("QT_B", "0")) or None  # override the batch (tail-effect experiments)
x = synth.make_inputs(cfg, device="cuda", dtype=dtype, **({"B": QB} if QB else {}))
y, w, lam, g = x["y"], x["w"], x["lam"], x["g"]
T, B = y.shape
d = 2
ws = P.Workspace(d, T, B, dtype, lam.dim() == 2)
z = torch.empty_like(y); gy = torch.empty_like(y); gl = torch.empty_like(lam)
WB = os.environ.get("WHIT_WBITS") == "1"
if WB:
    wbits = P.whit_pack_mask(w)
    fwd = lambda: P.whit_forward_wbits(y, wbits, lam, d, T, B, z, ws)
else:
    fwd = lambda: P.whit_forward(y, w, lam, d, T, B, z, ws)
for _ in range(3):
    fwd(); P.whit_backward(g, ws, z, gy, gl)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tf, tb = [], []
for _ in range(5):
    ev[0].record(); fwd(); ev[1].record(); P.whit_backward(g, ws, z, gy, gl); ev[2].record()
    torch.cuda.synchronize()
    tf.append(ev[0].elapsed_time(ev[1])); tb.append(ev[1].elapsed_time(ev[2]))
esz = 4 if dtype == torch.float32 else 8
pd = lam.dim() == 2
steps = T * B
# algorithmic (R-mode) bytes: fwd: 2x(y,w,lam) + z + dz + ckpt w/r ; bwd: 2x(g,w,lam) + dz + ybar + lambar + ckpts
C = (T + 15) // 16
fwd_b = steps * esz * (2 * (3 if pd else 2) + 2) + C * B * 5 * 8 * 2 + (0 if pd else 2 * B * esz)
bwd_b = steps * esz * (2 * (3 if pd else 2) + 1 + 1 + (1 if pd else 0)) + C * B * (3 + 2) * 8 + C * B * 2 * 8
tfm, tbm = min(tf), min(tb)
print(f"{cfg} {dtype} wbits={WB} T={T} B={B}: fwd {tfm:.3f} ms ({fwd_b/tfm/1e6:.0f} GB/s)  bwd {tbm:.3f} ms ({bwd_b/tbm/1e6:.0f} GB/s)  "
      f"fwd+bwd {(tfm+tbm):.3f} ms -> {B/((tfm+tbm)/1e3)/1e6:.2f} M series/s  all: {[round(a,3) for a in tf]} {[round(a,3) for a in tb]}")
print("nfail", P.whit_failures(ws), flush=True)
