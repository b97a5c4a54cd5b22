"""Host time of a run outside the device wait, by phase (development aid): monkeypatches perf_counter marks
around the engine's internals."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import engine
ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
cfg = mm.PararealConfig(n_slices=64, iterations=5, slice_length=0.1, particles=100_000, step=mm.StepConfig(1e-3, 100),
                        integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
ens = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), mm.NoisePlan(0), 100_000)
ode = mm.unimodal_rhs(ou)
marks = {}
def wrap(obj, name, key):
    f = getattr(obj, name)
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); marks[key] = marks.get(key, 0.0) + time.perf_counter() - t; return r
    setattr(obj, name, g)
wrap(engine, '_build_trace', 'build_trace'); wrap(engine, '_raise_first_error', 'error_scan'); wrap(engine, '_plan_key', 'plan_key')
wrap(engine, 'device_model', 'device_model'); wrap(engine, 'device_ode', 'device_ode'); wrap(engine, '_initial_ensemble', 'initial_ensemble')
wrap(engine._Workspace if hasattr(engine, '_Workspace') else engine, 'read_back', 'read_back') if hasattr(engine, '_Workspace') else None
wrap(engine._RunPlan, 'replay', 'replay'); wrap(engine._RunPlan, 'join', 'join')
for _ in range(5):
    tr = mm.run_micro_macro(ou, ode, ens, cfg, mm.NoisePlan(0))
marks.clear()
R = 50
t0 = time.perf_counter()
for _ in range(R):
    tr = mm.run_micro_macro(ou, ode, ens, cfg, mm.NoisePlan(0))
tot = (time.perf_counter() - t0) / R
print(f"wall per run {1e3*tot:.3f} ms")
for k, v in sorted(marks.items(), key=lambda x: -x[1]):
    print(f"  {k:18s} {1e6*v/R:8.1f} us")
