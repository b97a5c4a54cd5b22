"""Cluster fine-sweep geometry sweep at config-4 shape (development aid)."""
import ctypes, os, sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L, kernels

def timeit(fn, reps=5):
    out = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), out

N, S, P = 64, 100, 100_000
dev = torch.device('cuda')
xi = kernels.noise_buffer(N, S, P); xi.normal_()
x = torch.randn((N, P), dtype=torch.float64, device=dev)
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device=dev)
t0 = torch.zeros(N, dtype=torch.float64, device=dev)
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
dwm = mm.make_double_well_multiplicative(mm.DoubleWellSpec(alpha=0.25, gamma=0.5, beta=0.2, J=0.0), 0.3).descriptor
configs = [dict(), dict(MMPR_FINE_SLOTS_PER_CTA='64', MMPR_FINE_STAGES='2'),
           dict(MMPR_FINE_SLOTS_PER_CTA='64', MMPR_FINE_STAGES='3'),
           dict(MMPR_FINE_SLOTS_PER_CTA='32', MMPR_FINE_STAGES='2'),
           dict(MMPR_FINE_FORCE_GRID='1', MMPR_FINE_GRID_SLOTS='64'),
           dict(MMPR_FINE_FORCE_GRID='1', MMPR_FINE_GRID_SLOTS='32')]
for env in configs + [dict(c, **{'X': 'dwm'}) for c in configs[:2]]:
    for k in ('MMPR_FINE_SLOTS_PER_CTA', 'MMPR_FINE_STAGES', 'MMPR_FINE_FORCE_GRID', 'MMPR_FINE_GRID_SLOTS'):
        os.environ.pop(k, None)
    os.environ.update({k: v for k, v in env.items() if k != 'X'})
    md = dwm if env.get('X') else model
    c, k = ctypes.c_int32(0), ctypes.c_int32(0)
    try:
        L.call('mmpr_fine_sweep_occupancy', P, ctypes.byref(c), ctypes.byref(k))
        ms, all_ = timeit(lambda: kernels.fine_sweep(md, x, out, t0, S, 1e-3, xi, bad))
    except L.MmprError as e:
        print(env, e); continue
    print(f'{env}: clusters={c.value} ctas={k.value} {ms:.3f} ms {N*S*P/ms*1e3:.3e} p-steps/s '
          f'{N*S*P*8/ms/1e6:.0f} GB/s {[round(a, 3) for a in all_]}', flush=True)
