"""One config-4-shaped fine sweep (64 slices x 1e5 particles x 100 steps)
with counter-based increments, for an ncu capture (launch 2 of the kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels, noise

N, P, S, DT = int(os.environ.get("NP_N", "64")), 100_000, 100, 1e-3
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
ens = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), mm.NoisePlan(0), P)
x = ens.device_positions.reshape(1, P).repeat(N, 1).contiguous()
out = torch.empty_like(x)
t0 = torch.zeros(N, dtype=torch.float64, device="cuda")
bad = torch.empty(N, dtype=torch.int32, device="cuda")
stats = torch.empty((N, 3), dtype=torch.float64, device="cuda")
cnts = torch.empty((N, 1), dtype=torch.int64, device="cuda")
c = noise.counter_noise(0, False)
for _ in range(3):
    kernels.fine_sweep(model.descriptor, x, out, t0, S, DT, None, bad, stats=stats, counts=cnts, counter=c)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
kernels.fine_sweep(model.descriptor, x, out, t0, S, DT, None, bad, stats=stats, counts=cnts, counter=c)
b.record()
torch.cuda.synchronize()
print(f"philox fine sweep {a.elapsed_time(b):.3f} ms")
