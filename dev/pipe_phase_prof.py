"""Phase cycles per unit of the iteration pipeline (dev build:
dev/build_variant.sh pprof "-DMMPR_PIPE_PROFILE" pipeline.cu) for config 3
(two regions) and config 2 (one region)."""
import ctypes, math, os, sys
import numpy as np, torch
os.environ.setdefault('MMPR_LIB', os.path.join(os.path.dirname(os.path.abspath(__file__)), 'ab', 'libmmpr_pprof.so'))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib as L
lib = L.load()
lib.mmpr_dev_pipe_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.mmpr_dev_rg_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
mdw = mm.make_double_well(dw)
part = dw.default_partition()
cub = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
mc = mm.make_cubic_meanfield(cub)
cases = {
    "config3": (mdw, mm.multimodal_rhs(mdw, part, dw.potential, dw.sigma), mm.bimodal_initial(-1.0, 1.0, 0.2), part, 10),
    "config2": (mc, mm.gaussian_closure_rhs(cub), mm.InitialDistribution.normal(0.5, 0.04), mm.SINGLE_REGION, 8),
}
names = ["wait F(k-1,n-1)", "chain+match+snap", "R(u)", "fine loop", "write+R(F)+publish"]
for name, (model, ode, init, pt, K) in cases.items():
    c = mm.PararealConfig(n_slices=32, iterations=K, slice_length=0.0625, particles=100_000,
                          step=mm.StepConfig(2.0 ** -10, 64), partition=pt, integrator=mm.EulerConfig(2.0 ** -6),
                          retain_snapshots=False)
    ens = mm.sample_initial(init, mm.NoisePlan(0), c.particles)
    mm.run_micro_macro(model, ode, ens, c, mm.NoisePlan(0)); torch.cuda.synchronize()
    lib.mmpr_dev_pipe_prof(None, 1)
    lib.mmpr_dev_rg_prof(None, 1)
    mm.run_micro_macro(model, ode, ens, c, mm.NoisePlan(0)); torch.cuda.synchronize()
    buf = np.zeros((1024, 8), dtype=np.uint64)
    lib.mmpr_dev_pipe_prof(buf.ctypes.data, 1)
    units = buf[:, 5].sum()
    tot = buf[:, :5].sum(axis=0).astype(float)
    rg = np.zeros((1024, 8), dtype=np.uint64)
    lib.mmpr_dev_rg_prof(rg.ctypes.data, 1)
    rgn = ["counts+prefix", "cluster sync 1", "totals+scatter", "cluster sync 2", "leaf sums (pass)", "syncthreads",
           "fold+send", "cluster sync (pass)"]
    if rg.sum():
        print(name, "rg_restrict cycles per fine unit (both calls):",
              {n: round(float(v) / max(units, 1)) for n, v in zip(rgn, rg.sum(axis=0))})
    print(name, "fine units (CTA-level):", int(units), "cycles per fine unit:",
          {n: round(v / max(units, 1)) for n, v in zip(names, tot)})
