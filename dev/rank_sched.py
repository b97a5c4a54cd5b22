"""One-GPU emulation of the multi-GPU pipeline's scheduling: G virtual ranks,
each with its own clusters and ticket counter (MMPR_PIPELINE_RANK_TICKETS=1),
exchanging through each other's buffers.  Time of the iteration launch for
G = 1, 2, 4, 8 at a fixed total N (so per-rank work shrinks with G, as the
one GPU is shared): a rank that waits on its predecessor's coarse chain
shows up as extra time (development aid)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import sharded_pipeline as SP
from paper_2310_11365_b200.models import device_model
from paper_2310_11365_b200.moments import device_ode
from paper_2310_11365_b200.rk54 import integrator_descriptor

N, K, P, S = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 5, 100_000, 100
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
ode = mm.unimodal_rhs(model)
model_d = device_model(model)
ode_d, odm = device_ode(ode)
cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * 1e-3, particles=P, step=mm.StepConfig(1e-3, S),
                        integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
integ_d = integrator_descriptor(cfg.integrator)
plan = mm.NoisePlan(0)
times = torch.tensor([n * cfg.slice_length for n in range(N + 1)], dtype=torch.float64, device="cuda")
x0 = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.01), plan, P).device_positions
ref = None
for G in (1, 2, 4, 8):
    for mode in ("0", "1"):
        if G == 1 and mode == "1":
            continue
        os.environ["MMPR_PIPELINE_RANK_TICKETS"] = mode
        ranks = [SP.RankBuffers(r, G, N, K, P, S, False) for r in range(G)]
        for rb in ranks:
            rb.prologue(ode_d, odm, integ_d, times, x0, plan.master_seed)
        ios = [rb.io(times) for rb in ranks]
        ms = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            SP.launch(model_d, ode_d, odm, integ_d, 1e-3, S, True, ios, 0, G, 1, True, False, N, K, P)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        Ng = N // G
        macro = SP.merge_rows([rb.macro.cpu().numpy() for rb in ranks], Ng, G, N, "boundary")
        ref = macro if ref is None else ref
        print(f"G={G} rank_tickets={mode}: {min(ms):.3f} ms per launch; macro equal: {np.array_equal(macro, ref)}",
              flush=True)
        for rb in ranks:
            rb.free()
        del ranks
        torch.cuda.empty_cache()
