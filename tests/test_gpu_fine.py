"""GPU parity: fine propagator (fine.cu) against the oracle and the
reference's golden vectors.

Tolerance (north star): per-particle trajectories within 1e-12 relative
(max|x_gpu - x_ref| / max(1, max|x_ref|), the acceptance-1 metric).  For
models without a cube (OU, linear) and numpy-exact noise the result is
required to be bit-identical.
"""

import math

import numpy as np
import pytest

from oracle import mm_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel_dev(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / max(1.0, float(np.max(np.abs(b))))


GPU_MODELS = {
    "ou": lambda m: m.make_perturbed_ou(m.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)),
    "ou_default": lambda m: m.make_perturbed_ou(m.PerturbedOUSpec()),
    "linear": lambda m: m.make_linear(m.LinearMcKVSpec(A=-0.7, A_E=0.3, A_0=0.1, B=0.2, B_E=0.05, B_0=0.4)),
    "double_well": lambda m: m.make_double_well(m.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0,
                                                                 sigma=0.5)),
    "double_well_tilt": lambda m: m.make_double_well(m.DoubleWellSpec(alpha=0.25, gamma=0.5, beta=0.3, J=0.2,
                                                                      sigma=0.7)),
    "cubic": lambda m: m.make_cubic_meanfield(m.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)),
    "dw_mult": lambda m: m.make_double_well_multiplicative(m.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2,
                                                                            J=0.0), 0.3),
}
BITWISE = {"ou", "ou_default", "linear", "cubic"}


@pytest.fixture(scope="module")
def mm():
    import paper_2310_11365_b200 as mm
    mm._lib.load()
    return mm


@pytest.mark.parametrize("name", sorted(GPU_MODELS))
@pytest.mark.parametrize("P", [1, 5, 1000, 1001])
def test_propagate_fine_matches_reference_golden(mm, golden, name, P):
    g = golden("fine")
    key = f"{name}_P{P}"
    Pm, S, dt, n, t0, seed = g[key + "_meta"]
    model = GPU_MODELS[name](mm)
    ens = mm.ParticleEnsemble(g[key + "_x0"])
    out = mm.propagate_fine(model, ens, int(n), t0, mm.StepConfig(dt, int(S)), mm.NoisePlan(int(seed)))
    ref = g[key + "_x1"]
    assert rel_dev(out.positions, ref) <= TOL
    if name in BITWISE:
        tail = np.abs(O.slice_noise(int(seed), int(n), int(S), int(Pm))) > 3.6541528853610087
        if not tail.any():
            assert np.array_equal(out.positions, ref)


# (20_000 .. 50_000: one-slice launches spread a slice over 8 x 256-thread CTAs; 40_000 / 50_000 must not --
# 512 leaf slots at 32 per CTA would be 16 CTAs of 8 warps, more CTAs than the cluster fold has lanes with the total)
@pytest.mark.parametrize("P", [8, 100, 10_000, 12_345, 20_000, 25_000, 40_000, 50_000, 100_000, 131_072, 200_003])
def test_injected_mode_bitwise_ou(mm, P):
    """Same seeded increments on both sides: trajectories bit-identical."""
    rng = np.random.default_rng(P)
    S = 12
    x0 = rng.normal(1.0, 0.1, P)
    xi = rng.standard_normal((S, P))
    model = GPU_MODELS["ou"](mm)
    out = mm.propagate_fine(model, mm.ParticleEnsemble(x0), 0, 0.0, mm.StepConfig(1e-3, S), mm.NoisePlan(0),
                            increments=xi)
    ref = O.propagate_fine(O.model_ou(-1.0, 0.5, 0.5), x0, 0, 0.0, 1e-3, S, xi)
    assert np.array_equal(out.positions, ref)


@pytest.mark.parametrize("name", sorted(GPU_MODELS))
def test_injected_mode_all_models(mm, name):
    rng = np.random.default_rng(3)
    P, S = 100_000, 8
    x0 = np.concatenate([rng.normal(-1.0, 0.2, P // 2), rng.normal(1.0, 0.2, P - P // 2)])
    xi = rng.standard_normal((S, P))
    model = GPU_MODELS[name](mm)
    out = mm.propagate_fine(model, mm.ParticleEnsemble(x0), 0, 0.0, mm.StepConfig(2.0 ** -10, S),
                            mm.NoisePlan(0), increments=xi)
    oracle_models = {"ou": O.model_ou(-1.0, 0.5, 0.5), "ou_default": O.model_ou(-1.0, -0.5, 0.01),
                     "linear": O.model_linear(-0.7, 0.3, 0.1, 0.2, 0.05, 0.4),
                     "double_well": O.model_double_well(0.25, 0.4, 0.2, 0.0, 0.5),
                     "double_well_tilt": O.model_double_well(0.25, 0.5, 0.3, 0.2, 0.7),
                     "cubic": O.model_cubic(1.0, 1.0, 1.0, 0.4),
                     "dw_mult": O.model_dw_mult(0.25, 0.4, 0.2, 0.0, 0.3)}
    ref = O.propagate_fine(oracle_models[name], x0, 0, 0.0, 2.0 ** -10, S, xi)
    assert rel_dev(out.positions, ref) <= TOL
    if name in BITWISE:
        assert np.array_equal(out.positions, ref)


def test_em_step_known_answers(mm):
    out = mm.em_step(mm.make_perturbed_ou(mm.PerturbedOUSpec()), mm.ParticleEnsemble([100.0]), 0.0, 0.01,
                     np.zeros(1))
    assert out.positions[0] == pytest.approx(98.5)
    out = mm.em_step(mm.make_perturbed_ou(mm.PerturbedOUSpec(a=0.0, a_E=0.0, B=2.0)), mm.ParticleEnsemble([1.0]),
                     0.0, 0.25, np.array([3.0]))
    assert out.positions[0] == pytest.approx(4.0)


def test_em_step_validates_noise_and_finiteness(mm):
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec())
    ens = mm.ParticleEnsemble([1.0, 2.0])
    with pytest.raises(ValueError):
        mm.em_step(model, ens, 0.0, 0.01, np.zeros(3))
    with pytest.raises(mm.NumericalBlowup):
        mm.em_step(model, ens, 0.0, 0.01, np.array([np.inf, 0.0]))


def test_propagate_fine_replays_em_steps_exactly(mm):
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(B=1.0))
    plan = mm.NoisePlan(42)
    cfg = mm.StepConfig(dt=0.05, steps_per_slice=7)
    ens = mm.sample_initial(mm.InitialDistribution.normal(1.0, 0.5), plan, 64)
    manual = ens
    for j in range(cfg.steps_per_slice):
        manual = mm.em_step(model, manual, 3.0 + j * cfg.dt, cfg.dt, plan.normals(4, j, 64))
    out = mm.propagate_fine(model, ens, 4, 3.0, cfg, plan)
    assert np.array_equal(out.positions, manual.positions)


def test_frozen_vs_fresh(mm):
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(B=1.0))
    cfg = mm.StepConfig(dt=0.05, steps_per_slice=5)
    ens = mm.sample_initial(mm.InitialDistribution.normal(0.0, 1.0), mm.NoisePlan(42), 32)
    frozen = mm.NoisePlan(42)
    a = mm.propagate_fine(model, ens, 0, 0.0, cfg, frozen, iteration=0)
    b = mm.propagate_fine(model, ens, 0, 0.0, cfg, frozen, iteration=9)
    assert np.array_equal(a.positions, b.positions)
    fresh = mm.NoisePlan(42, mm.NoiseMode.FRESH)
    c = mm.propagate_fine(model, ens, 0, 0.0, cfg, fresh, iteration=0)
    d = mm.propagate_fine(model, ens, 0, 0.0, cfg, fresh, iteration=9)
    assert not np.array_equal(c.positions, d.positions)


def test_blowup_location(mm):
    model = mm.make_double_well(mm.DoubleWellSpec(sigma=0.0))
    cfg = mm.StepConfig(dt=0.5, steps_per_slice=50)
    with pytest.raises(mm.NumericalBlowup) as err:
        mm.propagate_fine(model, mm.ParticleEnsemble([3.0, 1.0]), 6, 0.0, cfg, mm.NoisePlan(1))
    assert err.value.slice_index == 6
    with np.errstate(over="ignore", invalid="ignore"):
        with pytest.raises(O.OracleBlowup) as ref:
            O.propagate_fine(O.model_double_well(0.25, 0.5, 0.3, 0.0, 0.0), np.array([3.0, 1.0]), 6, 0.0, 0.5, 50,
                             np.zeros((50, 2)))
    assert err.value.step_index == ref.value.step_index


def test_fine_sweep_many_slices_independent(mm):
    """One launch over 64 slices equals 64 single-slice launches (bitwise)."""
    from paper_2310_11365_b200 import kernels
    import torch
    P, S, N = 100_000, 10, 16
    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.normal(0.0, 1.0, (N, P))).cuda()
    xi = kernels.noise_buffer(N, S, P)
    xi[:, :, :P] = torch.from_numpy(rng.standard_normal((N, S, P))).cuda()
    model = GPU_MODELS["double_well"](mm).descriptor
    t0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    out = torch.empty_like(x)
    bad = torch.empty(N, dtype=torch.int32, device="cuda")
    kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad)
    for n in (0, 7, 15):
        one = torch.empty((1, P), dtype=torch.float64, device="cuda")
        kernels.fine_sweep(model, x[n:n + 1], one, t0[:1], S, 1e-3, xi[n:n + 1], bad[:1])
        assert torch.equal(one[0], out[n])


def test_occupancy_query(mm):
    import ctypes
    c, k = ctypes.c_int32(0), ctypes.c_int32(0)
    mm._lib.call("mmpr_fine_sweep_occupancy", 100_000, ctypes.byref(c), ctypes.byref(k))
    assert k.value in (8, 16) and c.value >= 1


# ---- grid variant (teams of co-resident CTAs, fine_grid.cu) ------------------
GRID_CASES = [
    # (P, slots per CTA, chunks per step, slices)
    (100_000, 128, 1, 40),     # C = 8, 18 teams looping over 40 slices
    (100_000, 128, 2, 5),      # half-step chunks
    (100_000, 32, 1, 3),       # C = 32
    (200_003, 64, 2, 3),       # tail, C = 32
    (5_000, 32, 1, 4),         # padded slot tree, C = 2
    (1 << 20, 128, 2, 3),      # config 5 shape: C = 64 (two partials per lane)
    (1 << 20, 64, 1, 2),       # C = 128
    (1 << 20, 32, 1, 2),       # C = 256 (eight partials per lane)
]


@pytest.mark.parametrize("P,spc,chunks,N", GRID_CASES)
def test_grid_variant_bitwise_ou(mm, monkeypatch, P, spc, chunks, N):
    """The grid-reduction kernel reproduces the oracle bit for bit (and so the
    cluster kernel) for every team size and chunking."""
    from paper_2310_11365_b200 import kernels
    import torch
    monkeypatch.setenv("MMPR_FINE_FORCE_GRID", "1")
    monkeypatch.setenv("MMPR_FINE_GRID_SLOTS", str(spc))
    monkeypatch.setenv("MMPR_FINE_GRID_CHUNKS", str(chunks))
    S = 6
    rng = np.random.default_rng(P + spc)
    x0 = rng.normal(1.0, 0.1, (N, P))
    xi_h = rng.standard_normal((N, S, P))
    xi = kernels.noise_buffer(N, S, P)
    xi[:, :, :P] = torch.from_numpy(xi_h).cuda()
    x = torch.from_numpy(x0).cuda()
    out = torch.empty_like(x)
    bad = torch.empty(N, dtype=torch.int32, device="cuda")
    fmean = torch.empty(N, dtype=torch.float64, device="cuda")
    t0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    model = GPU_MODELS["ou"](mm).descriptor
    kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad, final_mean=fmean)
    torch.cuda.synchronize()
    om = O.model_ou(-1.0, 0.5, 0.5)
    got = out.cpu().numpy()
    for n in sorted({0, N // 2, N - 1}):
        ref = O.propagate_fine(om, x0[n], 0, 0.0, 1e-3, S, xi_h[n])
        assert np.array_equal(got[n], ref), n
        assert fmean[n].item() == float(np.mean(ref))
    assert (bad.cpu().numpy() == -1).all()


def test_grid_variant_natural_dispatch_and_models(mm):
    """P = 2^20 exceeds one cluster: dispatched to the grid kernel without
    any override; every model family within the north-star tolerance."""
    import ctypes
    c, k = ctypes.c_int32(0), ctypes.c_int32(0)
    mm._lib.call("mmpr_fine_sweep_occupancy", 1 << 20, ctypes.byref(c), ctypes.byref(k))
    assert k.value > 16 and c.value >= 1
    rng = np.random.default_rng(7)
    P, S = 1 << 20, 3
    x0 = np.concatenate([rng.normal(-1.0, 0.2, P // 2), rng.normal(1.0, 0.2, P - P // 2)])
    xi = rng.standard_normal((S, P))
    for name, om in [("dw_mult", O.model_dw_mult(0.25, 0.4, 0.2, 0.0, 0.3)),
                     ("cubic", O.model_cubic(1.0, 1.0, 1.0, 0.4))]:
        out = mm.propagate_fine(GPU_MODELS[name](mm), mm.ParticleEnsemble(x0), 0, 0.0,
                                mm.StepConfig(5e-4, S), mm.NoisePlan(0), increments=xi)
        ref = O.propagate_fine(om, x0, 0, 0.0, 5e-4, S, xi)
        assert rel_dev(out.positions, ref) <= TOL
        if name == "cubic":
            assert np.array_equal(out.positions, ref)


def test_grid_variant_blowup(mm, monkeypatch):
    monkeypatch.setenv("MMPR_FINE_FORCE_GRID", "1")
    monkeypatch.setenv("MMPR_FINE_GRID_SLOTS", "32")
    model = mm.make_double_well(mm.DoubleWellSpec(sigma=0.0))
    cfg = mm.StepConfig(dt=0.5, steps_per_slice=50)
    x0 = np.full(20_000, 1.0)
    x0[12_345] = 3.0
    with pytest.raises(mm.NumericalBlowup) as err:
        mm.propagate_fine(model, mm.ParticleEnsemble(x0), 6, 0.0, cfg, mm.NoisePlan(1))
    with np.errstate(over="ignore", invalid="ignore"):
        with pytest.raises(O.OracleBlowup) as ref:
            O.propagate_fine(O.model_double_well(0.25, 0.5, 0.3, 0.0, 0.0), x0, 6, 0.0, 0.5, 50,
                             np.zeros((50, x0.size)))
    assert err.value.step_index == ref.value.step_index
    # the same launch configuration still works afterwards (barrier phases drained)
    out = mm.propagate_fine(mm.make_perturbed_ou(mm.PerturbedOUSpec()), mm.ParticleEnsemble(np.ones(20_000)), 0,
                            0.0, mm.StepConfig(1e-3, 4), mm.NoisePlan(0), increments=np.zeros((4, 20_000)))
    assert np.isfinite(out.positions).all()


@pytest.mark.parametrize("P,grid", [(1, False), (7, False), (1000, False), (1001, False), (100_000, False),
                                    (200_003, False), (100_000, True), (1 << 20, False)])
def test_fused_restriction_equals_restrict(mm, monkeypatch, P, grid):
    """mmpr_fine_sweep_restrict: the stats the sweep computes from registers
    equal restrict() of its output bit for bit (np.mean / np.var)."""
    from paper_2310_11365_b200 import kernels
    import torch
    if grid:
        monkeypatch.setenv("MMPR_FINE_FORCE_GRID", "1")
    N, S = 3, 5
    rng = np.random.default_rng(P)
    x = torch.from_numpy(rng.normal(0.5, 1.0, (N, P))).cuda()
    xi = kernels.noise_buffer(N, S, P)
    xi[:, :, :P] = torch.from_numpy(rng.standard_normal((N, S, P))).cuda()
    t0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    out = torch.empty_like(x)
    bad = torch.empty(N, dtype=torch.int32, device="cuda")
    stats = torch.empty((N, 3), dtype=torch.float64, device="cuda")
    counts = torch.empty((N, 1), dtype=torch.int64, device="cuda")
    model = GPU_MODELS["double_well"](mm).descriptor
    kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad, stats=stats, counts=counts)
    ref_stats = torch.empty_like(stats)
    ref_counts = torch.empty_like(counts)
    kernels.restrict(mm.SINGLE_REGION.descriptor(), out, ref_stats, ref_counts)
    assert torch.equal(stats, ref_stats)
    assert torch.equal(counts, ref_counts)
    plain = torch.empty_like(x)
    kernels.fine_sweep(model, x, plain, t0, S, 1e-3, xi, bad)
    assert torch.equal(plain, out)


def test_random_sizes_sweep_bitwise(mm):
    """Forty particle counts drawn over 1..3e5 (every geometry: single CTA,
    clusters of 2..16, padded slot trees, tails, the compile-time and the
    run-time accumulator bound): injected-mode OU bitwise against the oracle."""
    from paper_2310_11365_b200 import kernels
    import torch
    rng = np.random.default_rng(2024)
    sizes = sorted(set(int(v) for v in np.exp(rng.uniform(0, np.log(3e5), 40))))
    om = O.model_ou(-1.0, 0.5, 0.5)
    model = GPU_MODELS["ou"](mm).descriptor
    S = 3
    for P in sizes:
        x0 = rng.normal(0.0, 1.0, (2, P))
        xi_h = rng.standard_normal((2, S, P))
        xi = kernels.noise_buffer(2, S, P)
        xi[:, :, :P] = torch.from_numpy(xi_h).cuda()
        x = torch.from_numpy(x0).cuda()
        out = torch.empty_like(x)
        bad = torch.empty(2, dtype=torch.int32, device="cuda")
        stats = torch.empty((2, 3), dtype=torch.float64, device="cuda")
        t0 = torch.zeros(2, dtype=torch.float64, device="cuda")
        kernels.fine_sweep(model, x, out, t0, S, 1e-3, xi, bad, stats=stats)
        got = out.cpu().numpy()
        st = stats.cpu().numpy()
        for n in range(2):
            ref = O.propagate_fine(om, x0[n], 0, 0.0, 1e-3, S, xi_h[n])
            assert np.array_equal(got[n], ref), P
            assert np.array_equal(st[n], O.restrict(ref)[0]), P


@pytest.mark.parametrize("cl", ["1", "4", "8"])
def test_grid_cluster_levels_bitwise(mm, monkeypatch, cl):
    """The grid sweep's first reduction level in clusters of 1/4/8 CTAs (the
    default is 2) gives the same bits (P = 2^20, 128 CTAs per team)."""
    from paper_2310_11365_b200 import kernels
    import torch
    monkeypatch.setenv("MMPR_FINE_GRID_CLUSTER", cl)
    P, N, S = 1 << 20, 3, 4
    rng = np.random.default_rng(int(cl))
    x0 = rng.normal(0.0, 1.0, (N, P))
    xi_h = rng.standard_normal((N, S, P))
    xi = kernels.noise_buffer(N, S, P)
    xi[:, :, :P] = torch.from_numpy(xi_h).cuda()
    out = torch.empty((N, P), dtype=torch.float64, device="cuda")
    bad = torch.empty(N, dtype=torch.int32, device="cuda")
    kernels.fine_sweep(GPU_MODELS["ou"](mm).descriptor, torch.from_numpy(x0).cuda(), out,
                       torch.zeros(N, dtype=torch.float64, device="cuda"), S, 1e-3, xi, bad)
    got = out.cpu().numpy()
    om = O.model_ou(-1.0, 0.5, 0.5)
    for n in (0, N - 1):
        assert np.array_equal(got[n], O.propagate_fine(om, x0[n], 0, 0.0, 1e-3, S, xi_h[n]))
