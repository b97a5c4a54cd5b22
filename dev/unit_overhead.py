"""Per-unit overhead of the iteration pipeline: launch time for S = 25, 50,
100 steps per slice (config-4 otherwise); the intercept of time vs S is the
per-unit cost outside the step loop (development aid)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_11365_b200 as mm

model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
ode = mm.unimodal_rhs(model)
plan = mm.NoisePlan(0)
ens0 = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), plan, 100000)
res = []
for S in (25, 50, 100):
    cfg = mm.PararealConfig(n_slices=64, iterations=5, slice_length=S * 1e-3, particles=100000,
                            step=mm.StepConfig(1e-3, S), integrator=mm.EulerConfig(1e-3), retain_snapshots=False)
    for _ in range(2):
        mm.run_micro_macro(model, ode, ens0, cfg, plan)
    ms = min(1e3 * sum(mm.run_micro_macro(model, ode, ens0, cfg, plan, record_timings=True).timings["iterations"])
             for _ in range(3))
    res.append((S, ms))
    print(f"S={S}: pipeline {ms:.3f} ms", flush=True)
(s1, t1), (s2, t2) = res[0], res[-1]
slope = (t2 - t1) / (s2 - s1)
print(f"per step (all 320 units / 14 clusters): {1e3 * slope:.1f} us; intercept {t1 - slope * s1:.3f} ms "
      f"= {1e3 * (t1 - slope * s1) * 14 / 320:.1f} us per unit")
