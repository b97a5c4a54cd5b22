"""Host-side cost of one graph-replayed config-4 run_micro_macro call from a
pinned host ensemble (the bench's e2e path), with cProfile (development aid)."""
import cProfile, os, pstats, sys, time
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
for _ in range(5):
    mm.run_micro_macro(model, ode, mm.ParticleEnsemble(host.to("cuda", non_blocking=True)), cfg, plan)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t = time.perf_counter()
    mm.run_micro_macro(model, ode, mm.ParticleEnsemble(host.to("cuda", non_blocking=True)), cfg, plan)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
print("e2e ms per run: mean %.3f min %.3f" % (1e3 * sum(ts) / len(ts), 1e3 * min(ts)))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    mm.run_micro_macro(model, ode, mm.ParticleEnsemble(host.to("cuda", non_blocking=True)), cfg, plan)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(25)
