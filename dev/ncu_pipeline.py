"""Two default config-4 runs (graph replay), for ncu captures of the
iteration pipeline kernel (development aid)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_11365_b200 as mm

model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
cfg = mm.PararealConfig(n_slices=64, iterations=5, slice_length=0.1, particles=100000,
                        step=mm.StepConfig(1e-3, 100), integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
for _ in range(2):
    mm.run_micro_macro(model, mm.unimodal_rhs(model), mm.InitialDistribution.normal(1.0, 0.01), cfg, mm.NoisePlan(0),
                       use_graph=False)
torch.cuda.synchronize()
print("ok", mm.engine.last_run_info)
