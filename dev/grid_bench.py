"""Grid fine sweep (P = 2^20, config 5's geometry) timings: OU and the
config-5 multiplicative double well, N slices x 200 steps, for several
MMPR_FINE_GRID_* settings (dev A/B).  Prints ms, HBM GB/s of the increments."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels

N, S, P = int(os.environ.get("NG", "32")), 200, int(os.environ.get("PG", str(1 << 20)))
xi = kernels.noise_buffer(N, S, P)
xi.normal_()
dw5 = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.3 * math.sqrt(1.8))
models = {"ou": mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor,
          "dw_mult": mm.make_double_well_multiplicative(dw5, 0.3).descriptor}
x = torch.randn((N, P), dtype=torch.float64, device="cuda")
out = torch.empty_like(x)
bad = torch.empty(N, dtype=torch.int32, device="cuda")
t0 = torch.zeros(N, dtype=torch.float64, device="cuda")
settings = [s for s in os.environ.get("GRID_SETTINGS", "L2_AHEAD=0;L2_AHEAD=3;L2_AHEAD=6").split(";")]
for name, model in models.items():
    for st in settings:
        for kv in st.split(","):
            k, v = kv.split("=")
            os.environ["MMPR_FINE_GRID_" + k] = v
        dt = 5e-4
        for _ in range(2):
            kernels.fine_sweep(model, x, out, t0, S, dt, xi, bad)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            kernels.fine_sweep(model, x, out, t0, S, dt, xi, bad)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        gbs = N * S * P * 8 / (ms / 1e3) / 1e9
        print(f"{name:8s} {st:30s} {ms:8.3f} ms  {gbs:7.0f} GB/s  {N*S*P/(ms/1e3):.3e} particle-steps/s")
        for kv in st.split(","):
            os.environ.pop("MMPR_FINE_GRID_" + kv.split("=")[0], None)
