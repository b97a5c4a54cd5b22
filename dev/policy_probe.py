import os, sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels
def timeit(fn, reps=5):
    out = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)
N, S, P = 64, 100, 100_000
xi = kernels.noise_buffer(N, S, P); xi.normal_()
x = torch.randn((N, P), dtype=torch.float64, device='cuda')
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device='cuda')
t0 = torch.zeros(N, dtype=torch.float64, device='cuda')
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
for pol in (None, '0', '1', '2'):
    if pol is None: os.environ.pop('MMPR_FINE_CLUSTER_POLICY', None)
    else: os.environ['MMPR_FINE_CLUSTER_POLICY'] = pol
    for spc in ('64', '128'):
        os.environ['MMPR_FINE_SLOTS_PER_CTA'] = spc
        for n in (64, 8):
            print(f'policy {pol} spc {spc} slices {n}: {timeit(lambda: kernels.fine_sweep(model, x[:n], out[:n], t0[:n], S, 1e-3, xi[:n], bad[:n])):.3f} ms', flush=True)
