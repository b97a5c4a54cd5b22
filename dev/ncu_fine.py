import os, sys, torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L, kernels, noise
L.load()
N, S, P = 64, 100, 100000
xi = kernels.noise_buffer(N, S, P)
keys = noise.step_keys(0, False, 0, 0, N, S)
noise.fill_normals(keys, P, xi, xi.stride(1))
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
x = torch.randn((N, P), dtype=torch.float64, device='cuda')
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device='cuda')
t0 = torch.zeros(N, dtype=torch.float64, device='cuda')
for _ in range(2):
    kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad)
torch.cuda.synchronize()
print('ok')
