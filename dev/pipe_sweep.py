"""Per-run time of the config-4 run under pipeline tuning overrides
(MMPR_PIPELINE_CLUSTERS, MMPR_FINE_L2_AHEAD), development aid."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_11365_b200 as mm

model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
ode = mm.unimodal_rhs(model)
cfg = mm.PararealConfig(n_slices=64, iterations=5, slice_length=0.1, particles=100000,
                        step=mm.StepConfig(1e-3, 100), integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
plan = mm.NoisePlan(0)
ens0 = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), plan, 100000)
settings = [s.split(",") for s in sys.argv[1:]] or [["MMPR_PIPELINE_CLUSTERS=14"]]
for setting in settings:
    for kv in setting:
        k, v = kv.split("=")
        os.environ[k] = v
    mm.engine.clear_graph_cache()
    for _ in range(3):
        mm.run_micro_macro(model, ode, ens0, cfg, plan)
    ms = []
    for _ in range(3):
        tr = mm.run_micro_macro(model, ode, ens0, cfg, plan, record_timings=True)
        ms.append(1e3 * sum(tr.timings.get("iterations", [0.0])))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        mm.run_micro_macro(model, ode, ens0, cfg, plan)
    e1.record()
    torch.cuda.synchronize()
    print(f"{','.join(setting):50s} run {e0.elapsed_time(e1) / 10:.3f} ms  pipeline {min(ms):.3f} ms", flush=True)
