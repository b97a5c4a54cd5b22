"""Config 3 (bimodal double well, two regions, N=32, P=1e5, S=64, K=10) ms per
run, graph-replayed (dev A/B; environment switches apply)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_11365_b200 as mm

dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
mdw = mm.make_double_well(dw)
part = dw.default_partition()
c = mm.PararealConfig(n_slices=32, iterations=10, slice_length=0.0625, particles=100_000,
                      step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6),
                      retain_snapshots=False)
ens = mm.sample_initial(mm.bimodal_initial(-1.0, 1.0, 0.2), mm.NoisePlan(0), c.particles)
ode = mm.multimodal_rhs(mdw, part, dw.potential, dw.sigma)
fn = lambda: mm.run_micro_macro(mdw, ode, ens, c, mm.NoisePlan(0))
tr = fn(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    fn()
e1.record(); torch.cuda.synchronize()
print(f"config3 {os.environ.get('TAG', '')}: {e0.elapsed_time(e1) / 5:.3f} ms per run, pipeline={mm.engine.last_run_info.get('pipeline')}")
if os.environ.get("STAGES"):
    mm.engine.clear_graph_cache()
    tr = mm.run_micro_macro(mdw, ode, ens, c, mm.NoisePlan(0), record_timings=True)
    print({k: round(sum(v) * 1e3, 3) for k, v in tr.stage_timings.items()})
