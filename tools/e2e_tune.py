"""Try whit_run_host chunk / stream counts at the hetero shape (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_00048_b200 as P
import synth
x = synth.make_inputs("hetero", device="cuda")
h = {k: torch.empty(x[k].shape, dtype=torch.float32, pin_memory=True) for k in ("y", "w", "lam", "g")}
for k in h: h[k].copy_(x[k])
del x; torch.cuda.empty_cache()
oz = torch.empty(h["y"].shape, pin_memory=True); oy = torch.empty(h["y"].shape, pin_memory=True); ol = torch.empty(h["lam"].shape, pin_memory=True)
B = h["y"].shape[1]
for chunk, nbuf in ((16384, 3), (32768, 3), (65536, 2), (65536, 3), (16384, 4), (8192, 6)):
    buf = P.whit_run_host(h["y"], h["w"], h["lam"], h["g"], 2, oz, oy, ol, chunk=chunk, nbuf=nbuf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        P.whit_run_host(h["y"], h["w"], h["lam"], h["g"], 2, oz, oy, ol, chunk=chunk, nbuf=nbuf, dev_buf=buf)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(f"chunk {chunk} nbuf {nbuf}: {ms:.1f} ms/step -> {B/ms*1e3/1e6:.3f} M series/s", flush=True)
    del buf; torch.cuda.empty_cache()
