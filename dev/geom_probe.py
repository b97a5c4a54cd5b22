"""propagate_fine against the oracle over ensemble sizes and cluster geometries (development aid)."""
import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2310_11365_b200 as mm
from oracle import mm_oracle as O
ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
om = O.model_ou(-1.0, 0.5, 0.5)
S, dt = 8, 1e-3
for P in [int(a) for a in sys.argv[1:]] or [10_000, 20_000, 25_000, 40_000, 50_000, 30_000, 80_000, 100_000]:
    rng = np.random.default_rng(P)
    x0 = rng.normal(1.0, 0.1, P)
    inc = rng.standard_normal((S, P))
    ref = O.propagate_fine(om, x0, 0, 0.0, dt, S, inc)
    got = mm.propagate_fine(ou, mm.ParticleEnsemble(x0), 0, 0.0, mm.StepConfig(dt, S), mm.NoisePlan(0), increments=inc).positions
    print(P, os.environ.get('MMPR_FINE_SLOTS_PER_CTA', 'auto'), 'equal' if np.array_equal(ref, got) else f'DIFF max {np.abs(ref - got).max():.3e}')
