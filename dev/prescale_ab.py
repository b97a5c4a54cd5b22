"""A/B: fine sweep with increments pre-multiplied by b*sqrt(dt)
(MMPR_NOISE_PRESCALED) vs the plain sweep, config-4 shape (development aid)."""
import ctypes, math, sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L, kernels

N, S, P, dt = 64, 100, 100_000, 1e-3
dev = torch.device('cuda')
xi = kernels.noise_buffer(N, S, P); xi.normal_()
x = torch.randn((N, P), dtype=torch.float64, device=dev) * 0.1 + 1.0
t0 = torch.zeros(N, dtype=torch.float64, device=dev)
bad = torch.empty(N, dtype=torch.int32, device=dev)
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
pre = L.Model.from_buffer_copy(model)
pre.stat_kind |= 0x100
bsd = model.p[2] * math.sqrt(dt)
xi_pre = xi * bsd

def run(md, noise, out):
    L.call('mmpr_fine_sweep', ctypes.byref(md), N, P, S, dt, math.sqrt(dt), t0.data_ptr(), x.data_ptr(), P,
           out.data_ptr(), P, noise.data_ptr(), noise.stride(0), noise.stride(1), bad.data_ptr(), None, None)

o1, o2 = torch.empty_like(x), torch.empty_like(x)
run(model, xi, o1); run(pre, xi_pre, o2); torch.cuda.synchronize()
print('bitwise equal:', torch.equal(o1.view(torch.int64), o2.view(torch.int64)))
for rep in range(3):
    for name, md, nz, o in (('plain', model, xi, o1), ('prescaled', pre, xi_pre, o2)):
        ts = []
        for _ in range(7):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); run(md, nz, o); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f'{name}: min {ts[0]:.4f} med {ts[3]:.4f} ms', flush=True)
