"""Config-3 run time (graph replay) with the one-pass cluster coupling
(MMPR_RESTRICT_CLUSTER=1) and the separate multi-kernel passes (=0)."""
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
for rep in range(2):
    for v in ("1", "0"):
        os.environ["MMPR_RESTRICT_CLUSTER"] = v
        mm.engine.clear_graph_cache()
        for _ in range(3):
            mm.run_micro_macro(model, ode, init, cfg, plan)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            mm.run_micro_macro(model, ode, init, cfg, plan)
        e1.record()
        torch.cuda.synchronize()
        print(f"MMPR_RESTRICT_CLUSTER={v}: {e0.elapsed_time(e1) / 10:.3f} ms per run", flush=True)
