"""Stage breakdown of BASELINE config 3 (bimodal, two regions) per run (development aid)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_11365_b200 as mm

dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
model = mm.make_double_well(dw)
part = dw.default_partition()
ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
cfg = mm.PararealConfig(n_slices=32, iterations=10, slice_length=0.0625, particles=100_000,
                        step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6),
                        retain_snapshots=False)
init = mm.bimodal_initial(-1.0, 1.0, 0.2)
plan = mm.NoisePlan(0)
for _ in range(2):
    tr = mm.run_micro_macro(model, ode, init, cfg, plan, record_timings=True)
t = {k: round(1e3 * sum(v), 3) for k, v in tr.stage_timings.items() if isinstance(v, list) and v}
n = {k: len(v) for k, v in tr.stage_timings.items() if isinstance(v, list) and v}
print(t, n, round(sum(t.values()), 3))
