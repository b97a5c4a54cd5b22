"""Per-stage device times (record_timings) for BASELINE configs 3 and 5 (development aid)."""
import math, sys
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
mdw = mm.make_double_well(dw)
part = dw.default_partition()
c3 = mm.PararealConfig(n_slices=32, iterations=10, slice_length=0.0625, particles=100_000,
                       step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6),
                       retain_snapshots=False)
for _ in range(2):
    tr = mm.run_micro_macro(mdw, mm.multimodal_rhs(mdw, part, dw.potential, dw.sigma), mm.bimodal_initial(-1.0, 1.0, 0.2),
                            c3, mm.NoisePlan(0), record_timings=True)
print('config 3 stage ms:', {k: round(1e3 * sum(v), 3) for k, v in tr.timings.items() if isinstance(v, list)})
dw5 = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.3 * math.sqrt(1.8))
m5 = mm.make_double_well_multiplicative(dw5, 0.3)
part5 = dw5.default_partition()
c5 = mm.PararealConfig(n_slices=32, iterations=10, slice_length=0.1, particles=1 << 20,
                       step=mm.StepConfig(5e-4, 200), partition=part5, integrator=mm.EulerConfig(1e-2),
                       retain_snapshots=False)
for _ in range(2):
    tr = mm.run_micro_macro(m5, mm.multimodal_rhs(m5, part5, dw5.potential, dw5.sigma), mm.bimodal_initial(-1.0, 1.0, 0.2),
                            c5, mm.NoisePlan(0), record_timings=True)
print('config 5 stage ms:', {k: round(1e3 * sum(v), 3) for k, v in tr.timings.items() if isinstance(v, list)})
