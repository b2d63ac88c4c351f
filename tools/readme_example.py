"""The README usage example (run from the repo root: PYTHONPATH=. python tools/readme_example.py)."""
import torch, paper_2604_00048_b200 as whit
T, B, d = 3288, 8192, 2
y   = torch.randn(T, B, device="cuda")
w   = (torch.rand(T, B, device="cuda") > 0.9).float()
lam = torch.full((T - d, B), 1e3, device="cuda", requires_grad=True)
z = whit.smooth(y, w, lam, d)
z.square().mean().backward()
print("ok", z.shape, lam.grad.shape, torch.isfinite(z).all().item(), torch.isfinite(lam.grad).all().item())
