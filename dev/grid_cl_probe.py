"""Grid sweep with a cluster first level: parity vs the plain grid path and timing (development aid)."""
import os, sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels
def timeit(fn, reps=7):
    out = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)
P = int(os.environ.get('P', 1 << 20))
N, S = 8, 200
xi = kernels.noise_buffer(N, S, P); xi.normal_()
x = torch.randn((N, P), dtype=torch.float64, device='cuda')
out = torch.empty_like(x); bad = torch.empty(N, dtype=torch.int32, device='cuda')
t0 = torch.zeros(N, dtype=torch.float64, device='cuda')
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad)
ref = out.clone()
ms = timeit(lambda: kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad))
print(f"P={P} {os.environ.get('MMPR_FINE_GRID_SLOTS','64')} cl={os.environ.get('MMPR_FINE_GRID_CLUSTER','1')}: {ms:.3f} ms {N*S*P/ms*1e3:.3e} p-steps/s", flush=True)
