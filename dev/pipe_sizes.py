"""Pipeline vs per-iteration kernels, ms per run over ensemble sizes (development aid)."""
import os, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2310_11365_b200 as mm
ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
init = mm.InitialDistribution.normal(1.0, 0.01)
SIZES = [(10_000, 10), (10_000, 64), (20_000, 64), (50_000, 64), (2 ** 14, 64), (2 ** 16, 64), (2 ** 17, 48), (100_000, 64),
         # the any-size form: 9, 11, 14, 15, 11, 14 elements per lane
         (4_608, 64), (9_999, 64), (12_345, 64), (30_000, 64), (60_000, 64), (70_000, 64), (90_000, 64), (99_999, 64),
         (120_001, 48)]
for P, N in SIZES:
    cfg = mm.PararealConfig(n_slices=N, iterations=5, slice_length=0.1, particles=P, step=mm.StepConfig(1e-3, 100),
                            integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
    res = {}
    for pipe in ("1", "0"):
        os.environ["MMPR_PIPELINE"] = pipe
        mm.engine.clear_graph_cache()
        for _ in range(3):
            mm.run_micro_macro(ou, mm.unimodal_rhs(ou), init, cfg, mm.NoisePlan(0))
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            mm.run_micro_macro(ou, mm.unimodal_rhs(ou), init, cfg, mm.NoisePlan(0))
        e1.record(); torch.cuda.synchronize()
        res[pipe] = (e0.elapsed_time(e1) / 10, mm.engine.last_run_info.get("pipeline"))
    print(f"P={P} N={N}: pipeline {res['1'][0]:.3f} ms ({res['1'][1]}), per-iteration {res['0'][0]:.3f} ms")
