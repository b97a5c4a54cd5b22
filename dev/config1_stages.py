"""Per-stage device times (record_timings) and graph-replay time of BASELINE config 1 (development aid)."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2310_11365_b200 as mm
ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
c1 = mm.PararealConfig(n_slices=10, iterations=5, slice_length=0.1, particles=10_000, step=mm.StepConfig(1e-3, 100),
                       integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
init = mm.InitialDistribution.normal(1.0, 0.01)
for _ in range(3):
    tr = mm.run_micro_macro(ou, mm.unimodal_rhs(ou), init, c1, mm.NoisePlan(0), record_timings=True)
print('config 1 stage ms:', {k: round(1e3 * sum(v), 4) for k, v in tr.timings.items() if isinstance(v, list)})
print('fine per sweep ms:', [round(1e3 * v, 4) for v in tr.timings.get('fine', [])][:12])
for _ in range(5):
    mm.run_micro_macro(ou, mm.unimodal_rhs(ou), init, c1, mm.NoisePlan(0))
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    mm.run_micro_macro(ou, mm.unimodal_rhs(ou), init, c1, mm.NoisePlan(0))
e1.record(); torch.cuda.synchronize()
print('config 1 ms per run (20 runs):', round(e0.elapsed_time(e1) / 20, 4), mm.engine.last_run_info if hasattr(mm.engine, 'last_run_info') else '')
