"""Config-4 run in NoiseMode.PHILOX (graph replay): ms per run (dev A/B; MMPR_LIB selects the library)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_11365_b200 as mm

N = int(os.environ.get("NP_N", "64"))
ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
c = mm.PararealConfig(n_slices=N, iterations=5, slice_length=0.1, particles=100_000, step=mm.StepConfig(1e-3, 100),
                      integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
ens = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), mm.NoisePlan(0), c.particles)
plan = mm.NoisePlan(0, mm.NoiseMode.PHILOX)
fn = lambda: mm.run_micro_macro(ou, mm.unimodal_rhs(ou), ens, c, plan)
fn(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    fn()
e1.record(); torch.cuda.synchronize()
print(f"philox config-4 run {e0.elapsed_time(e1) / 5:.3f} ms pipeline={mm.engine.last_run_info.get('pipeline')}")
