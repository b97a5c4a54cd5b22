"""Fine-sweep timings of the grid variant at config-5 shape (development aid)."""
import ctypes, os, sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L, kernels

def timeit(fn, reps=3):
    out = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), out

dev = torch.device('cuda')
models = {'ou': mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor,
          'dw_mult': mm.make_double_well_multiplicative(mm.DoubleWellSpec(alpha=0.25, gamma=0.5, beta=0.2, J=0.0),
                                                        0.3).descriptor}
cases = [(1 << 20, 8, 200, {}), (1 << 20, 8, 200, {'MMPR_FINE_GRID_SLOTS': '64'}),
         (1 << 20, 8, 200, {'MMPR_FINE_GRID_SLOTS': '32'}),
         (100_000, 64, 100, {}), (100_000, 64, 100, {'MMPR_FINE_FORCE_GRID': '1'}),
         (100_000, 64, 100, {'MMPR_FINE_FORCE_GRID': '1', 'MMPR_FINE_GRID_SLOTS': '64'})]
for P, N, S, env in cases:
    for k in ('MMPR_FINE_GRID_SLOTS', 'MMPR_FINE_FORCE_GRID', 'MMPR_FINE_GRID_CHUNKS'):
        os.environ.pop(k, None)
    os.environ.update(env)
    xi = kernels.noise_buffer(N, S, P)
    xi.normal_()
    x = torch.randn((N, P), dtype=torch.float64, device=dev)
    out = torch.empty_like(x)
    bad = torch.empty(N, dtype=torch.int32, device=dev)
    t0 = torch.zeros(N, dtype=torch.float64, device=dev)
    c, k = ctypes.c_int32(0), ctypes.c_int32(0)
    L.call('mmpr_fine_sweep_occupancy', P, ctypes.byref(c), ctypes.byref(k))
    for name, model in models.items():
        ms, all_ = timeit(lambda: kernels.fine_sweep(model, x, out, t0, S, 5e-4, xi, bad))
        byts = N * S * P * 8 + 2 * N * P * 8
        print(f'P={P} N={N} S={S} {env} {name}: teams/clusters={c.value} ctas={k.value} {ms:.3f} ms '
              f'{N*S*P/ms*1e3:.3e} p-steps/s {byts/ms/1e6:.0f} GB/s {[round(a, 3) for a in all_]}', flush=True)
    del xi
