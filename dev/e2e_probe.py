"""Wall-clock per run of the default graph-replayed config-4 run, device-resident
input vs pinned-host input, pipeline on/off (development aid)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_11365_b200 as mm

model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
ode = mm.unimodal_rhs(model)
cfg = mm.PararealConfig(n_slices=64, iterations=5, slice_length=0.1, particles=100000,
                        step=mm.StepConfig(1e-3, 100), integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
plan = mm.NoisePlan(0)
ens0 = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), plan, 100000)
host = ens0.device_positions.cpu().pin_memory()
for pipe in ("1", "0"):
    os.environ["MMPR_PIPELINE"] = pipe
    mm.engine.clear_graph_cache()
    for _ in range(3):
        mm.run_micro_macro(model, ode, ens0, cfg, plan)
    torch.cuda.synchronize()
    for label in ("device", "host", "device"):
        ts = []
        for _ in range(10):
            torch.cuda.synchronize()
            t = time.perf_counter()
            e = ens0 if label == "device" else mm.ParticleEnsemble(host.to("cuda", non_blocking=True))
            mm.run_micro_macro(model, ode, e, cfg, plan)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        print(f"pipeline={pipe} input={label}: {1e3 * sum(ts) / len(ts):.3f} ms/run (min {1e3 * min(ts):.3f})",
              flush=True)
    # with an eager timed run in between (as bench.py does)
    mm.run_micro_macro(model, ode, ens0, cfg, plan, record_timings=True)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t = time.perf_counter()
        mm.run_micro_macro(model, ode, mm.ParticleEnsemble(host.to("cuda", non_blocking=True)), cfg, plan)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"pipeline={pipe} after eager, host input: {1e3 * sum(ts) / len(ts):.3f} ms/run", flush=True)
