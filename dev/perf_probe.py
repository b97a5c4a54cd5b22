"""Per-kernel timings for the config-4 workload (development aid)."""
import ctypes, math, os, sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L, kernels, noise

def timeit(fn, reps=3):
    out = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), out

N, S, P = 64, 100, 100000
dev = torch.device('cuda')
xi = kernels.noise_buffer(N, S, P)
keys = noise.step_keys(0, False, 0, 0, N, S)
ms, _ = timeit(lambda: noise.fill_normals(keys, P, xi, xi.stride(1)))
print(f'noise fill: {ms:.3f} ms  {N*S*P/ms/1e6:.3f} Gnormals/s')
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
x = torch.randn((N, P), dtype=torch.float64, device=dev)
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device=dev)
t0 = torch.zeros(N, dtype=torch.float64, device=dev)
for grp, spc, ns, l2 in (('1', '128', '2', '0'), ('0', '128', '2', '0'), ('1', '128', '2', '3'), ('1', '64', '4', '0')):
    os.environ['MMPR_FINE_DIRECT'] = grp
    os.environ['MMPR_FINE_SLOTS_PER_CTA'] = spc
    os.environ['MMPR_FINE_STAGES'] = ns
    os.environ['MMPR_FINE_L2_AHEAD'] = l2
    c, k = ctypes.c_int32(0), ctypes.c_int32(0)
    try:
        L.call('mmpr_fine_sweep_occupancy', P, ctypes.byref(c), ctypes.byref(k))
    except L.MmprError as e:
        print('spc', spc, e); continue
    ms, all_ = timeit(lambda: kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad))
    byts = N*S*P*8 + 2*N*P*8
    print(f'fine sweep direct={grp} l2={l2} ns={ns} spc={spc} ctas/slice={k.value} clusters={c.value}: {ms:.3f} ms {N*S*P/ms/1e9*1e3:.3e} p-steps/s {byts/ms/1e6:.0f} GB/s  {all_}')
[os.environ.pop(k) for k in ('MMPR_FINE_DIRECT', 'MMPR_FINE_SLOTS_PER_CTA', 'MMPR_FINE_STAGES', 'MMPR_FINE_L2_AHEAD')]
part = mm.SINGLE_REGION.descriptor()
stats = torch.empty((N, 3), dtype=torch.float64, device=dev); counts = torch.empty((N, 1), dtype=torch.int64, device=dev)
ms, _ = timeit(lambda: kernels.restrict(part, x, stats, counts))
print(f'restrict 64x1e5: {ms:.3f} ms ({2*N*P*8/ms/1e6:.0f} GB/s algorithmic)')
st = torch.empty(N, dtype=torch.int32, device=dev)
tg = stats.clone(); tg[:, 0] += 0.1
ms, _ = timeit(lambda: kernels.match(part, tg, stats, counts, x, out, 0, st))
print(f'match 64x1e5: {ms:.3f} ms ({2*N*P*8/ms/1e6:.0f} GB/s)')
spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
m = mm.make_perturbed_ou(spec)
cfg = mm.PararealConfig(n_slices=N, iterations=5, slice_length=0.1, particles=P, step=mm.StepConfig(1e-3, S),
                        integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
plan = mm.NoisePlan(0)
ens0 = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), plan, P)
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    tr = mm.run_micro_macro(m, mm.unimodal_rhs(m), ens0, cfg, plan)
    torch.cuda.synchronize(); el = time.perf_counter() - t
    tm = {k: round(sum(v)*1e3, 3) for k, v in tr.timings.items()}
    print(f'run_micro_macro C4: {el*1e3:.2f} ms wall; stage ms {tm}')
