"""coarse_row timing at config-4 shape (development aid)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels
from paper_2310_11365_b200.moments import device_ode
from paper_2310_11365_b200.rk54 import integrator_descriptor

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
model = mm.make_perturbed_ou(spec)
ode_d, om_d = device_ode(mm.unimodal_rhs(model))
integ = integrator_descriptor(mm.EulerConfig(1e-2))
dev = torch.device('cuda')
times = torch.tensor([0.1 * n for n in range(N + 1)], dtype=torch.float64, device=dev)
rho0 = torch.tensor([[1.0, 0.01, 1.0]], dtype=torch.float64, device=dev)
fine = torch.rand((N, 3), dtype=torch.float64, device=dev)
cache = torch.rand((N, 3), dtype=torch.float64, device=dev)
macro = torch.empty((N + 1, 3), dtype=torch.float64, device=dev)
cout = torch.empty((N, 3), dtype=torch.float64, device=dev)
raw = torch.empty((N, 3), dtype=torch.float64, device=dev)
st = torch.empty(N, dtype=torch.int32, device=dev)
for k in (0, 1, 3):
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        kernels.coarse_row(ode_d, om_d, integ, times, k, rho0, fine, cache, macro, cout, raw, st, skip_until=k)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f'N={N} k={k}: coarse_row {min(ts)*1e3:.1f} us {[round(t*1e3,1) for t in ts]}')
