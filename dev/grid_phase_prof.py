"""Phase cycle breakdown of the grid fine sweep (dev build, MMPR_FINE_PROFILE)."""
import ctypes, os, sys
import numpy as np, torch
os.environ['MMPR_LIB'] = '/root/repo/dev/libmmpr_gprof.so'
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L, kernels
lib = L.load()
lib.mmpr_dev_grid_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
N, S, P = 8, 200, 1 << 20
xi = kernels.noise_buffer(N, S, P); xi.normal_()
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
x = torch.randn((N, P), dtype=torch.float64, device='cuda')
out = torch.empty_like(x); bad = torch.empty(N, dtype=torch.int32, device='cuda')
t0 = torch.zeros(N, dtype=torch.float64, device='cuda')
kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad)
lib.mmpr_dev_grid_prof(None, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad); e1.record(); torch.cuda.synchronize()
buf = np.zeros((2048, 8), dtype=np.int64)
lib.mmpr_dev_grid_prof(buf.ctypes.data, 1)
ctas = 256
steps = N // 2 * S  # per team (2 teams)
per = buf[:ctas].sum(axis=0) / ctas / steps
names = ['update', 'B1', 'publish(red)', '-', 'B1->B2 (fold/spin, thread0)', 'B2', 'reduce total']
print(f'{e0.elapsed_time(e1):.3f} ms; cycles per CTA-step:', dict(zip(names, per[:7].round(0))))
