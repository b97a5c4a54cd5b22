"""One launch of each hot kernel on config-4 shapes, for ncu (development aid)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels, noise

N, S, P = 64, 100, 100000
xi = kernels.noise_buffer(N, S, P)
keys = noise.step_keys(0, False, 0, 0, N, S)
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
x = torch.randn((N, P), dtype=torch.float64, device='cuda')
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device='cuda')
t0 = torch.zeros(N, dtype=torch.float64, device='cuda')
part = mm.SINGLE_REGION.descriptor()
stats = torch.empty((N, 3), dtype=torch.float64, device='cuda')
counts = torch.empty((N, 1), dtype=torch.int64, device='cuda')
st = torch.empty(N, dtype=torch.int32, device='cuda')
for _ in range(2):
    noise.fill_normals(keys, P, xi, xi.stride(1))
    kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad)
    kernels.restrict(part, out, stats, counts)
    kernels.match(part, stats, stats, counts, out, x, 0, st)
torch.cuda.synchronize()
print('ok')
