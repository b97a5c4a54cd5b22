"""Config 4 (N=64, P=1e5, S=100, K=5) per-run time: numpy-exact FROZEN vs
counter-based PHILOX, iteration pipeline and per-iteration kernels; plus
the fine sweep alone in both modes (CUDA events, graph-replayed runs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels, noise

N, P, S, K, DT = 64, 100_000, 100, 5, 1e-3
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
ode = mm.unimodal_rhs(model)
cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * DT, particles=P, step=mm.StepConfig(DT, S),
                        integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
init = mm.InitialDistribution.normal(1.0, 0.01)
ens = mm.sample_initial(init, mm.NoisePlan(0), P)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for pipe in ("1", "0"):
    os.environ["MMPR_PIPELINE"] = pipe
    for mode in (mm.NoiseMode.FROZEN, mm.NoiseMode.PHILOX):
        mm.engine.clear_graph_cache()
        plan = mm.NoisePlan(0, mode)
        ms = timed(lambda: mm.run_micro_macro(model, ode, ens, cfg, plan))
        tr = mm.run_micro_macro(model, ode, ens, cfg, plan, record_timings=True)
        st = {k: round(1e3 * sum(v), 3) for k, v in tr.timings.items() if isinstance(v, list) and v}
        print(f"pipeline={pipe} mode={mode.value:7s} run {ms:.3f} ms  "
              f"{K * N * P * S / ms / 1e-3:.3e} particle-steps/s  stages {st}", flush=True)

x = ens.device_positions.reshape(1, P).repeat(N, 1).contiguous()
out = torch.empty_like(x)
t0 = torch.zeros(N, dtype=torch.float64, device="cuda")
bad = torch.empty(N, dtype=torch.int32, device="cuda")
xi = noise.slice_noise(0, 0, N, S, P)
c = noise.counter_noise(0, False)
stats = torch.empty((N, 3), dtype=torch.float64, device="cuda")
cnts = torch.empty((N, 1), dtype=torch.int64, device="cuda")
for name, kw in (("hbm", dict(xi=xi)), ("philox", dict(xi=None, counter=c))):
    xi_ = kw.pop("xi")
    ms = timed(lambda: kernels.fine_sweep(model.descriptor, x, out, t0, S, DT, xi_, bad, stats=stats, counts=cnts, **kw))
    print(f"fine sweep {name:6s} {ms:.3f} ms  {N * P * S / ms / 1e-3:.3e} particle-steps/s", flush=True)
