"""Fine sweep tail-wave geometry experiment (development aid)."""
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
dev = torch.device('cuda')
xi = kernels.noise_buffer(N, S, P); xi.normal_()
x = torch.randn((N, P), dtype=torch.float64, device=dev)
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device=dev)
t0 = torch.zeros(N, dtype=torch.float64, device=dev)
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
def sweep(a, b):
    kernels.fine_sweep(model, x[a:b], out[a:b], t0[a:b], S, 1e-3, xi[a:b], bad[a:b])
print('64 default', timeit(lambda: sweep(0, 64)))
print('56 default', timeit(lambda: sweep(0, 56)))
print('8 default', timeit(lambda: sweep(56, 64)))
for env in ({'MMPR_FINE_STAGES': '4'}, {'MMPR_FINE_SLOTS_PER_CTA': '128'}, {'MMPR_FINE_SLOTS_PER_CTA': '128', 'MMPR_FINE_STAGES': '1'}):
    os.environ.update(env)
    try:
        print('8', env, timeit(lambda: sweep(56, 64)))
    except Exception as e:
        print('8', env, e)
    for k in env: os.environ.pop(k)
