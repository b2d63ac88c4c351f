"""dev: would a hybrid launch help the 1.15-wave homo batch?  The first full wave of warp groups on the
sequential kernel and the tail groups on the twisted kernel, on two streams, vs everything sequential."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_00048_b200 as P
import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "homo"
B = int(os.environ.get("HB_B", "65536"))
B1 = int(os.environ.get("HB_B1", str(148 * 12 * 32)))
x = synth.make_inputs(cfg, B=B, device="cuda")
d, T = 2, x["y"].shape[0]
pd = x["lam"].dim() == 2


def part(lo, hi, twist):
    sl = lambda t: (t[:, lo:hi] if t.dim() == 2 else t[lo:hi]).contiguous()
    y, w, lam, g = (sl(x[k]) for k in ("y", "w", "lam", "g"))
    ws = P.Workspace(d, T, hi - lo, torch.float32, pd)
    ws.set_twist(twist)
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
    return (y, w, lam, g, ws, z, gy, gl, hi - lo)


def run(pt, stream):
    y, w, lam, g, ws, z, gy, gl, n = pt
    ws.set_stream(stream)
    P.whit_forward(y, w, lam, d, T, n, z, ws)
    P.whit_backward(g, ws, z, gy, gl)


full = part(0, B, 0)
a, b = part(0, B1, 0), part(B1, B, 1)
s0 = torch.cuda.current_stream()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def time(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    for _ in range(n): fn()
    e1.record(s0)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
def hybrid():
    ev = torch.cuda.Event(); ev.record(s0)
    s1.wait_event(ev); s2.wait_event(ev)
    run(a, s1)
    run(b, s2)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1); e2.record(s2)
    s0.wait_event(e1); s0.wait_event(e2)
t_full = time(lambda: run(full, s0))
t_hyb = time(hybrid)
t_tw = time(lambda: run(part(0, B, 1), s0)) if B <= 131072 else float("nan")
print(f"{cfg} B={B} B1={B1}: sequential {t_full:.3f} ms ({B / t_full / 1e3:.2f} M/s)  hybrid {t_hyb:.3f} ms "
      f"({B / t_hyb / 1e3:.2f} M/s)  all-twisted {t_tw:.3f} ms")
