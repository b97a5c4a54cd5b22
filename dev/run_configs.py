"""Wall time of run_micro_macro for BASELINE configs 1-5 on one B200 (config 5
with fewer slices than its 8-GPU N=256), graph-replayed, for DESIGN.md."""
import math, sys, time
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def report(name, cfg, fn):
    ms = timed(fn)
    ps = cfg.iterations * cfg.n_slices * cfg.particles * cfg.step.steps_per_slice
    print(f'{name}: N={cfg.n_slices} P={cfg.particles} S={cfg.step.steps_per_slice} K={cfg.iterations}: '
          f'{ms:.2f} ms per run, {ps / ms * 1e3:.3e} particle-steps/s', flush=True)


ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
init1 = mm.InitialDistribution.normal(1.0, 0.01)
c1 = mm.PararealConfig(n_slices=10, iterations=5, slice_length=0.1, particles=10_000,
                       step=mm.StepConfig(1e-3, 100), integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
report('config 1', c1, lambda: mm.run_micro_macro(ou, mm.unimodal_rhs(ou), init1, c1, mm.NoisePlan(0)))

cub = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
mc = mm.make_cubic_meanfield(cub)
c2 = mm.PararealConfig(n_slices=32, iterations=8, slice_length=0.0625, particles=100_000,
                       step=mm.StepConfig(2.0 ** -10, 64), integrator=mm.EulerConfig(2.0 ** -6), retain_snapshots=False)
report('config 2', c2, lambda: mm.run_micro_macro(mc, mm.gaussian_closure_rhs(cub), mm.InitialDistribution.normal(0.5, 0.04),
                                                  c2, mm.NoisePlan(0)))

dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
mdw = mm.make_double_well(dw)
part = dw.default_partition()
c3 = mm.PararealConfig(n_slices=32, iterations=10, slice_length=0.0625, particles=100_000,
                       step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6),
                       retain_snapshots=False)
report('config 3', c3, lambda: mm.run_micro_macro(mdw, mm.multimodal_rhs(mdw, part, dw.potential, dw.sigma),
                                                  mm.bimodal_initial(-1.0, 1.0, 0.2), c3, mm.NoisePlan(0)))

c4 = mm.PararealConfig(n_slices=64, iterations=5, slice_length=0.1, particles=100_000,
                       step=mm.StepConfig(1e-3, 100), integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
report('config 4 (G=1)', c4, lambda: mm.run_micro_macro(ou, mm.unimodal_rhs(ou), init1, c4, mm.NoisePlan(0)))

dw5 = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.3 * math.sqrt(1.8))
m5 = mm.make_double_well_multiplicative(dw5, 0.3)
part5 = dw5.default_partition()
N5 = int(sys.argv[1]) if len(sys.argv) > 1 else 32
c5 = mm.PararealConfig(n_slices=N5, iterations=10, slice_length=0.1, particles=1 << 20,
                       step=mm.StepConfig(5e-4, 200), partition=part5, integrator=mm.EulerConfig(1e-2),
                       retain_snapshots=False)
report(f'config 5 (one GPU, N={N5} of 256)', c5,
       lambda: mm.run_micro_macro(m5, mm.multimodal_rhs(m5, part5, dw5.potential, dw5.sigma),
                                  mm.bimodal_initial(-1.0, 1.0, 0.2), c5, mm.NoisePlan(0)))
