"""Phase cycle breakdown of the fine sweep (dev build with MMPR_FINE_PROFILE)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
os.environ['MMPR_LIB'] = '/root/repo/dev/libmmpr_prof.so'
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L, kernels, noise
lib = L.load()
lib.mmpr_dev_fine_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
N, S, P = 64, 100, 100000
xi = kernels.noise_buffer(N, S, P)
keys = noise.step_keys(0, False, 0, 0, N, S)
noise.fill_normals(keys, P, xi, xi.stride(1))
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
x = torch.randn((N, P), dtype=torch.float64, device='cuda')
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device='cuda')
t0 = torch.zeros(N, dtype=torch.float64, device='cuda')
buf = np.zeros((4096, 10), dtype=np.int64)
names = ['wait_stage', 'update', 'B1', 'cluster_wait', '-', 'leaf+warp', '-', 'fold+send', 'reduce_total']
for grp, spc in (('1', '64'),):
    os.environ['MMPR_FINE_GROUPS'] = grp
    os.environ['MMPR_FINE_SLOTS_PER_CTA'] = spc
    os.environ['MMPR_FINE_STAGES'] = '2'
    kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad)
    lib.mmpr_dev_fine_prof(None, 1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad); e1.record(); torch.cuda.synchronize()
    lib.mmpr_dev_fine_prof(buf.ctypes.data, 1)
    ctas = 64 * (8 if spc == '128' else 16)
    per_step = buf[:ctas, :9].sum(axis=0) / ctas / S
    print(f'groups {grp} spc {spc}: {e0.elapsed_time(e1):.3f} ms; cycles per CTA-step:', dict(zip(names, per_step.round(0))))
