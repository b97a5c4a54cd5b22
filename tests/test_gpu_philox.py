"""GPU: the counter-based Philox mode (NoiseMode.PHILOX / PHILOX_FRESH),
increments generated in registers inside the fine kernels.

Two kinds of parity, as the north star asks:
* against its own restatement (oracle/npstream.c section 5), bit for bit:
  the generated increments, propagate_fine through the cluster sweep, the
  grid sweep and the iteration pipeline, and whole run_micro_macro traces
  with the oracle loop consuming the same counter increments;
* against the reference's numpy-stream noise, statistically: per-(k, n)
  means and variances within 3 combined Monte Carlo standard errors in
  >= 99% of cells (se_mean = sqrt(S/P), se_var = S*sqrt(2/(P-1)),
  pkg/tests/test_acceptance.py:99-100), and the Parareal error-vs-k curves
  reaching the floor at the same k +- 1 (metrics.py:73-130).
"""

import math

import numpy as np
import pytest

from oracle import mm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import paper_2310_11365_b200 as mm
    mm._lib.load()
    return mm


def _packed(trace, attr):
    return np.array([[s.packed() for s in row] for row in getattr(trace, attr)])


def _snap(trace):
    return np.array([[e.positions for e in row] for row in trace.snapshots])


@pytest.mark.parametrize("seed,n,j,P,p0,fresh,k", [(0, 0, 0, 100_000, 0, False, 0), (7, 63, 99, 5000, 0, False, 0),
                                                   (2 ** 40 + 3, 5, 17, 3000, 1_000_000, False, 0),
                                                   (11, 2, 3, 20_000, 0, True, 4)])
def test_counter_normals_equal_oracle(mm, seed, n, j, P, p0, fresh, k):
    from paper_2310_11365_b200 import noise
    got = noise.counter_normals(seed, fresh, n, j, P, k, rows=3, first_particle=p0).cpu().numpy()
    for r in range(3):
        ref = O.counter_normals(seed, n, j + r, P, k, fresh, first_particle=p0)
        assert np.array_equal(got[r], ref), (r, int((got[r] != ref).sum()))


def test_counter_normals_many_tail_draws(mm):
    """~1.3e7 draws (thousands of tail and wedge draws) equal the oracle."""
    from paper_2310_11365_b200 import noise
    P = 1_300_000
    got = noise.counter_normals(3, False, 1, 0, P, rows=10).cpu().numpy()
    tails = 0
    for r in range(10):
        ref = O.counter_normals(3, 1, r, P)
        assert np.array_equal(got[r], ref), r
        tails += int((np.abs(ref) > 3.6541528853610087).sum())
    assert tails > 2000


@pytest.mark.parametrize("P", [7, 1000, 12_345, 100_000, 2 ** 20])
@pytest.mark.parametrize("model_name", ["ou", "dw_mult"])
def test_propagate_fine_counter_equals_oracle(mm, P, model_name):
    """Cluster sweep (P <= 1e5) and grid sweep (P = 2^20) with in-register
    increments equal the oracle fed the same counter increments: bitwise
    for OU, 1e-12 for the cube drift (numpy pow vs exact cube)."""
    S, n, dt = 6 if P == 2 ** 20 else 20, 3, 1e-3
    if model_name == "ou":
        model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
        om = O.model_ou(-1.0, 0.5, 0.5)
    else:
        dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.4)
        model = mm.make_double_well_multiplicative(dw, 0.3)
        om = O.model_dw_mult(0.25, 0.4, 0.2, 0.0, 0.3)
    x0 = np.random.default_rng(P).normal(0.5, 0.7, P)
    plan = mm.NoisePlan(21, mm.NoiseMode.PHILOX)
    got = mm.propagate_fine(model, mm.ParticleEnsemble(x0), n, 0.3, mm.StepConfig(dt, S), plan).positions
    ref = O.propagate_fine(om, x0, n, 0.3, dt, S, O.counter_slice_noise(21, n, S, P))
    if model_name == "ou":
        assert np.array_equal(got, ref)
    else:
        assert np.max(np.abs(got - ref)) / max(1.0, np.max(np.abs(ref))) <= 1e-12


def test_counter_sweep_matches_materialised_counter_increments(mm):
    """The in-register sweep equals the HBM sweep fed the same counter
    increments written out (mmpr_counter_normals_fill), bit for bit, for
    several slices at once (slice offsets)."""
    from paper_2310_11365_b200 import kernels, noise
    N, P, S, dt = 5, 100_000, 12, 1e-3
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    import torch
    x = torch.as_tensor(np.random.default_rng(2).normal(1.0, 0.2, (N, P)), device="cuda")
    t0 = torch.arange(N, dtype=torch.float64, device="cuda") * S * dt
    a = torch.empty_like(x)
    b = torch.empty_like(x)
    bad = torch.empty(N, dtype=torch.int32, device="cuda")
    c = noise.counter_noise(9, False, 0, 40)
    kernels.fine_sweep(model.descriptor, x, a, t0, S, dt, None, bad, counter=c)
    xi = kernels.noise_buffer(N, S, P)
    for s in range(N):
        xi[s, :, :P] = noise.counter_normals(9, False, 40 + s, 0, P, rows=S)
    kernels.fine_sweep(model.descriptor, x, b, t0, S, dt, xi, bad)
    assert torch.equal(a, b)


def _ou_cfg(mm, N, K, S, P, **kw):
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * 1e-3, particles=P, step=mm.StepConfig(1e-3, S),
                            integrator=mm.EulerConfig(1e-2), **kw)
    return model, mm.unimodal_rhs(model), cfg


@pytest.mark.parametrize("pipeline", [True, False])
def test_run_philox_equals_oracle_with_counter_noise(mm, monkeypatch, pipeline):
    """A whole PHILOX-mode run (iteration pipeline, or per-iteration
    kernels) equals the oracle loop consuming the same counter increments,
    bit for bit."""
    N, K, S, P = 6, 4, 20, 100_000
    monkeypatch.setenv("MMPR_PIPELINE", "1" if pipeline else "0")
    mm.engine.clear_graph_cache()
    model, ode, cfg = _ou_cfg(mm, N, K, S, P)
    ens0 = O.sample_normal_initial(0, 1.0, 0.01, P)
    tr = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(0, mm.NoiseMode.PHILOX))
    assert mm.engine.last_run_info["pipeline"] is pipeline
    om = O.model_ou(-1.0, 0.5, 0.5)
    ref = O.run_micro_macro(om, O.ode_unimodal(om), ens0, N, K, S * 1e-3, 1e-3, S, 0, integ=O.Euler(1e-2),
                            noise=lambda n, k: O.counter_slice_noise(0, n, S, P))
    assert np.array_equal(_packed(tr, "macro"), ref.macro)
    assert np.array_equal(_packed(tr, "micro_stats"), ref.micro)
    assert np.array_equal(_snap(tr), np.array([[e for e in row] for row in ref.snapshots]))
    mm.engine.clear_graph_cache()


def test_philox_fresh_and_exactness(mm):
    """PHILOX_FRESH draws new increments per iteration (oracle, bitwise);
    PHILOX keeps the k >= n exactness property against sequential_fine."""
    N, K, S, P = 5, 3, 10, 20_000
    model, ode, cfg = _ou_cfg(mm, N, K, S, P)
    ens0 = O.sample_normal_initial(0, 1.0, 0.01, P)
    tr = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(5, mm.NoiseMode.PHILOX_FRESH))
    om = O.model_ou(-1.0, 0.5, 0.5)
    ref = O.run_micro_macro(om, O.ode_unimodal(om), ens0, N, K, S * 1e-3, 1e-3, S, 0, integ=O.Euler(1e-2),
                            noise=lambda n, k: O.counter_slice_noise(5, n, S, P, k, True))
    assert np.array_equal(_snap(tr), np.array([[e for e in row] for row in ref.snapshots]))
    plan = mm.NoisePlan(5, mm.NoiseMode.PHILOX)
    tr = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, plan)
    seq = mm.sequential_fine(model, mm.ParticleEnsemble(ens0), cfg, plan)
    for k in range(1, K + 1):
        for n in range(k + 1):
            assert np.array_equal(tr.snapshots[k][n].positions, seq[n].positions), (k, n)


def _cells_within(a, b, P):
    """Fraction of (k, n) cells whose means and variances agree within
    3 combined Monte Carlo standard errors."""
    ma, va = a[..., 0], a[..., 1]
    mb, vb = b[..., 0], b[..., 1]
    se_m = np.sqrt(va / P + vb / P)
    se_v = np.sqrt((va * math.sqrt(2 / (P - 1))) ** 2 + (vb * math.sqrt(2 / (P - 1))) ** 2)
    ok = (np.abs(ma - mb) <= 3 * se_m) & (np.abs(va - vb) <= 3 * se_v)
    return float(ok[:, 1:].mean())


def _kstar(errs, tol):
    return next((k for k, e in enumerate(errs) if e <= tol), len(errs))


@pytest.mark.parametrize("which", ["config4", "config2"])
def test_philox_statistical_parity_with_reference_noise(mm, which):
    """Philox-mode runs against the reference's numpy-stream runs (the
    FROZEN mode is bitwise the reference, test_gpu_fullsize_parity.py) at
    BASELINE sizes: >= 99% of (k, n) cells within 3 SE, and the same
    convergence k (+- 1) of the relative errors against each mode's own
    serial fine solution."""
    if which == "config4":
        N, K, S, P, dt = 64, 5, 100, 100_000, 1e-3
        model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
        ode, init, euler = mm.unimodal_rhs(model), mm.InitialDistribution.normal(1.0, 0.01), 1e-2
    else:
        N, K, S, P, dt = 32, 8, 64, 100_000, 2.0 ** -10
        spec = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
        model = mm.make_cubic_meanfield(spec)
        ode, init, euler = mm.gaussian_closure_rhs(spec), mm.InitialDistribution.normal(0.5, 0.04), 2.0 ** -6
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * dt, particles=P, step=mm.StepConfig(dt, S),
                            integrator=mm.EulerConfig(euler))
    runs, curves = {}, {}
    for mode in (mm.NoiseMode.FROZEN, mm.NoiseMode.PHILOX):
        plan = mm.NoisePlan(0, mode)
        tr = mm.run_micro_macro(model, ode, init, cfg, plan)
        runs[mode] = _packed(tr, "micro_stats")
        seq = mm.sequential_fine(model, init, cfg, plan)
        from types import SimpleNamespace
        both = SimpleNamespace(snapshots=[list(row) for row in tr.snapshots] + [seq], iterations=K + 1, n_slices=N)
        curves[mode] = np.array([_rel_errors(mm, both, k, K + 1) for k in range(K + 1)])
    frac = _cells_within(runs[mm.NoiseMode.FROZEN], runs[mm.NoiseMode.PHILOX], P)
    assert frac >= 0.99, frac
    for col in range(3):  # E_mean, E_var, E_W
        a, b = curves[mm.NoiseMode.FROZEN][:, col], curves[mm.NoiseMode.PHILOX][:, col]
        tol = 1e-2 * max(a[0], b[0])
        assert abs(_kstar(a, tol) - _kstar(b, tol)) <= 1, (col, a, b)


def _rel_errors(mm, trace, k, ref_k):
    rep = mm.relative_errors(trace, k, ref_k)
    return [rep.e_mean, rep.e_var, rep.e_wass]
