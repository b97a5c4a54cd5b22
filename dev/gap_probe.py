"""Kernel timeline of back-to-back config-4 runs (torch.profiler / CUPTI): where the time between
the sum of the kernels and the measured run goes (development aid)."""
import sys, json
sys.path.insert(0, '/root/repo')
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2310_11365_b200 as mm
ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
cfg = mm.PararealConfig(n_slices=64, iterations=5, slice_length=0.1, particles=100_000, step=mm.StepConfig(1e-3, 100),
                        integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
init = mm.InitialDistribution.normal(1.0, 0.01)
ens = mm.sample_initial(init, mm.NoisePlan(0), 100_000)
def run():
    return mm.run_micro_macro(ou, mm.unimodal_rhs(ou), ens if ens is not None else init, cfg, mm.NoisePlan(0))
for _ in range(4):
    run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(4):
        run()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = None
for e in evs:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = (e.time_range.start - prev_end) if prev_end is not None else 0
    if d > 20 or gap > 20:
        print(f"{s/1e3:9.3f} ms  dur {d:8.1f} us  gap-before {gap:7.1f} us  {e.name[:60]}")
    prev_end = max(prev_end or 0, e.time_range.end)

import cProfile, pstats, time
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(30):
    run()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats('tottime').print_stats(18)
