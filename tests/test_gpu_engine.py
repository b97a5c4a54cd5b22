"""GPU parity: the full mM-Parareal run (fine + restrict + coarse + match on
the device) against the reference's golden traces and the oracle.

Tolerances (north star): trajectories 1e-12 relative (acceptance-1 metric),
per-iteration moments 1e-10 relative.  Within the GPU implementation the
k >= n exactness property is required bit for bit.
"""

import math

import numpy as np
import pytest

from oracle import mm_oracle as O

pytestmark = pytest.mark.gpu

TRAJ_TOL = 1e-12
MOM_TOL = 1e-10


@pytest.fixture(scope="module")
def mm():
    import paper_2310_11365_b200 as mm
    mm._lib.load()
    return mm


def _packed(trace, attr):
    return np.array([[s.packed() for s in row] for row in getattr(trace, attr)])


def _snap(trace):
    return np.array([[e.positions for e in row] for row in trace.snapshots])


def _rel(a, b):
    return float(np.max(np.abs(a - b))) / max(1.0, float(np.max(np.abs(b))))


def _check(trace, g, prefix, bitwise_macro=False):
    macro, micro = _packed(trace, "macro"), _packed(trace, "micro_stats")
    assert _rel(macro, g[prefix + "macro"]) <= MOM_TOL
    assert _rel(micro, g[prefix + "micro"]) <= MOM_TOL
    assert _rel(_snap(trace), g[prefix + "snap"]) <= TRAJ_TOL
    if bitwise_macro:
        assert np.array_equal(macro, g[prefix + "macro"])
        assert np.array_equal(micro, g[prefix + "micro"])
        assert np.array_equal(_snap(trace), g[prefix + "snap"])
    assert np.array_equal(np.array(trace.lift_collapses, dtype=float).reshape(-1, 3), g[prefix + "lift"])
    clamp = np.array(trace.clamp_events, dtype=float).reshape(-1, 4)
    assert clamp.shape == g[prefix + "clamp"].shape
    gaps = np.array(trace.fraction_gaps, dtype=float).reshape(-1, 3)
    assert gaps.shape == g[prefix + "gaps"].shape
    assert np.allclose(gaps, g[prefix + "gaps"], rtol=0, atol=1e-12)


def _c1(mm, P=1000, N=10, K=5):
    spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
    model = mm.make_perturbed_ou(spec)
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=0.1, particles=P,
                            step=mm.StepConfig(dt=1e-3, steps_per_slice=100), integrator=mm.EulerConfig(1e-2))
    return model, mm.unimodal_rhs(model), mm.InitialDistribution.normal(1.0, 0.01), cfg, mm.NoisePlan(0)


def test_config1_shape_matches_reference(mm, golden):
    g = golden("traces")
    model, ode, init, cfg, plan = _c1(mm)
    tr = mm.run_micro_macro(model, ode, init, cfg, plan)
    _check(tr, g, "c1_", bitwise_macro=True)
    seq = mm.sequential_fine(model, init, cfg, plan)
    assert np.array_equal(np.array([e.positions for e in seq]), g["c1_seq"])


def test_exactness_k_ge_n_bitwise(mm):
    model, ode, init, cfg, plan = _c1(mm)
    tr = mm.run_micro_macro(model, ode, init, cfg, plan)
    seq = mm.sequential_fine(model, init, cfg, plan)
    for k in range(1, cfg.iterations + 1):
        for n in range(k + 1):
            assert np.array_equal(tr.snapshots[k][n].positions, seq[n].positions), (k, n)


def test_reuse_converged_coarse_is_bitwise_neutral(mm):
    model, ode, init, cfg, plan = _c1(mm, P=3000)
    a = mm.run_micro_macro(model, ode, init, cfg, plan, reuse_converged_coarse=True)
    b = mm.run_micro_macro(model, ode, init, cfg, plan, reuse_converged_coarse=False)
    assert np.array_equal(_packed(a, "macro"), _packed(b, "macro"))
    assert np.array_equal(_snap(a), _snap(b))


def test_retain_snapshots_off_same_moments(mm):
    model, ode, init, cfg, plan = _c1(mm)
    a = mm.run_micro_macro(model, ode, init, cfg, plan)
    import dataclasses
    cfg2 = dataclasses.replace(cfg, retain_snapshots=False)
    b = mm.run_micro_macro(model, ode, init, cfg2, plan)
    assert b.snapshots is None
    assert np.array_equal(_packed(a, "macro"), _packed(b, "macro"))
    assert np.array_equal(_packed(a, "micro_stats"), _packed(b, "micro_stats"))


@pytest.mark.parametrize("prefix,ode_kind,seed", [("dp_", "perturbed", 77), ("dpu_", "unimodal", 78)])
def test_reference_default_dp54(mm, golden, prefix, ode_kind, seed):
    g = golden("traces")
    spec = mm.PerturbedOUSpec(B=1.0)
    model = mm.make_perturbed_ou(spec)
    ode = mm.perturbed_ou_rhs(spec) if ode_kind == "perturbed" else mm.unimodal_rhs(model)
    cfg = mm.PararealConfig(n_slices=6, iterations=4, slice_length=0.25, particles=500,
                            step=mm.StepConfig(dt=0.05, steps_per_slice=5))
    tr = mm.run_micro_macro(model, ode, mm.InitialDistribution.normal(1.0, 0.5), cfg, mm.NoisePlan(seed))
    _check(tr, g, prefix)


def _bimodal_init(mm):
    return mm.bimodal_initial(-1.0, 1.0, 0.2)


def test_config3_shape_matches_reference(mm, golden):
    g = golden("traces")
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    model = mm.make_double_well(dw)
    part = dw.default_partition()
    ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
    cfg = mm.PararealConfig(n_slices=8, iterations=4, slice_length=0.0625, particles=1000,
                            step=mm.StepConfig(dt=2.0 ** -10, steps_per_slice=64), partition=part,
                            integrator=mm.EulerConfig(2.0 ** -6))
    tr = mm.run_micro_macro(model, ode, _bimodal_init(mm), cfg, mm.NoisePlan(0))
    _check(tr, g, "c3_")
    seq = mm.sequential_fine(model, _bimodal_init(mm), cfg, mm.NoisePlan(0))
    assert _rel(np.array([e.positions for e in seq]), g["c3_seq"]) <= TRAJ_TOL


def test_config2_shape_matches_reference(mm, golden):
    g = golden("traces")
    spec = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
    model = mm.make_cubic_meanfield(spec)
    cfg = mm.PararealConfig(n_slices=8, iterations=4, slice_length=0.0625, particles=1000,
                            step=mm.StepConfig(dt=2.0 ** -10, steps_per_slice=64), integrator=mm.EulerConfig(2.0 ** -6))
    tr = mm.run_micro_macro(model, mm.gaussian_closure_rhs(spec), mm.InitialDistribution.normal(0.5, 0.04), cfg,
                            mm.NoisePlan(0))
    _check(tr, g, "c2_", bitwise_macro=True)


def test_config5_shape_matches_reference(mm, golden):
    g = golden("traces")
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.3 * math.sqrt(1.8))
    model = mm.make_double_well_multiplicative(dw, 0.3)
    part = dw.default_partition()
    ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
    cfg = mm.PararealConfig(n_slices=4, iterations=3, slice_length=0.1, particles=1000,
                            step=mm.StepConfig(dt=5e-4, steps_per_slice=200), partition=part,
                            integrator=mm.EulerConfig(1e-2))
    tr = mm.run_micro_macro(model, ode, _bimodal_init(mm), cfg, mm.NoisePlan(0))
    _check(tr, g, "c5_")


def test_injected_increments_against_oracle(mm):
    """Injected-increment mode: both sides consume the same seeded array."""
    P, N, K, S = 2000, 6, 3, 20
    rng = np.random.default_rng(4)
    xi = rng.standard_normal((N, S, P))
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * 1e-3, particles=P,
                            step=mm.StepConfig(1e-3, S), integrator=mm.EulerConfig(2e-3))
    ens0 = rng.normal(1.0, 0.1, P)
    tr = mm.run_micro_macro(model, mm.unimodal_rhs(model), mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(0),
                            increments=lambda n, k: xi[n])
    om = O.model_ou(-1.0, 0.5, 0.5)
    ref = O.run_micro_macro(om, O.ode_unimodal(om), ens0, N, K, S * 1e-3, 1e-3, S, 0, integ=O.Euler(2e-3),
                            noise=lambda n, k: xi[n])
    assert np.array_equal(_packed(tr, "macro"), ref.macro)
    assert np.array_equal(_snap(tr), np.array([[e for e in row] for row in ref.snapshots]))


def test_config4_full_size_properties(mm):
    """BASELINE config 4 at G=1 (N=64, P=1e5, S=100, K=5): size-independent
    checks -- k >= n exactness (bitwise vs the GPU's own serial fine
    solution), macro/micro consistency, and slice 0..1 against the oracle."""
    N, P, K = 64, 100_000, 5
    spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
    model = mm.make_perturbed_ou(spec)
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=0.1, particles=P,
                            step=mm.StepConfig(dt=1e-3, steps_per_slice=100), integrator=mm.EulerConfig(1e-2))
    plan = mm.NoisePlan(0)
    init = mm.InitialDistribution.normal(1.0, 0.01)
    tr = mm.run_micro_macro(model, mm.unimodal_rhs(model), init, cfg, plan)
    seq = mm.sequential_fine(model, init, cfg, plan)
    for k in range(1, K + 1):
        for n in range(k + 1):
            assert np.array_equal(tr.snapshots[k][n].positions, seq[n].positions), (k, n)
    for k in range(K + 1):
        for n in range(N + 1):
            mac, mic = tr.macro[k][n], tr.micro_stats[k][n]
            assert abs(mac.means[0] - mic.means[0]) < 1e-9 * max(1.0, abs(mac.means[0]))
            assert abs(mac.variances[0] - mic.variances[0]) < 1e-9 * max(1.0, mac.variances[0])
    ens0 = seq[0].positions
    om = O.model_ou(-1.0, 0.5, 0.5)
    x1 = O.propagate_fine(om, ens0, 0, 0.0, 1e-3, 100, O.slice_noise(0, 0, 100, P))
    assert _rel(seq[1].positions, x1) <= TRAJ_TOL


def test_blowup_raises_first_error_in_reference_order(mm):
    model = mm.make_double_well(mm.DoubleWellSpec(sigma=0.0))
    cfg = mm.PararealConfig(n_slices=4, iterations=2, slice_length=1.0, particles=16,
                            step=mm.StepConfig(dt=0.5, steps_per_slice=2), integrator=mm.EulerConfig(0.5))
    ens = mm.ParticleEnsemble(np.linspace(50.0, 60.0, 16))
    with pytest.raises((mm.NumericalBlowup, mm.IntegrationFailure)):
        mm.run_micro_macro(model, mm.unimodal_rhs(model), ens, cfg, mm.NoisePlan(0))


@pytest.mark.parametrize("mode", ["frozen", "fresh"])
@pytest.mark.parametrize("use_graph", [True, False])
def test_noise_batching_is_bitwise_neutral(mm, monkeypatch, mode, use_graph):
    """Increments held for a batch of slices at a time (regenerated per
    iteration) give the same run as holding every slice's increments."""
    model, ode, init, cfg, _ = _c1(mm, P=3000)
    plan = mm.NoisePlan(5, mm.NoiseMode.FRESH if mode == "fresh" else mm.NoiseMode.FROZEN)
    a = mm.run_micro_macro(model, ode, init, cfg, plan, use_graph=use_graph)
    sa, ma = _snap(a), _packed(a, "macro")
    monkeypatch.setenv("MMPR_NOISE_SLICES", "3")
    b = mm.run_micro_macro(model, ode, init, cfg, plan, use_graph=use_graph)
    assert np.array_equal(ma, _packed(b, "macro"))
    assert np.array_equal(sa, _snap(b))


def test_config5_large_ensemble_properties(mm):
    """BASELINE config 5 shape at one GPU (P = 2^20 per slice -- the grid
    reduction kernel -- bimodal multiplicative noise, dt = 5e-4) with fewer
    slices and steps: k >= n exactness against the GPU's own serial fine
    solution, per-region macro/micro consistency after matching, and slice
    0 -> 1 against the oracle."""
    P, N, K, S = 1 << 20, 4, 2, 40
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.3 * math.sqrt(1.8))
    model = mm.make_double_well_multiplicative(dw, 0.3)
    part = dw.default_partition()
    ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * 5e-4, particles=P,
                            step=mm.StepConfig(dt=5e-4, steps_per_slice=S), partition=part,
                            integrator=mm.EulerConfig(1e-2))
    plan = mm.NoisePlan(0)
    tr = mm.run_micro_macro(model, ode, _bimodal_init(mm), cfg, plan)
    seq = mm.sequential_fine(model, _bimodal_init(mm), cfg, plan)
    for k in range(1, K + 1):
        for n in range(k + 1):
            assert np.array_equal(tr.snapshots[k][n].positions, seq[n].positions), (k, n)
    for k in range(K + 1):
        for n in range(1, N + 1):
            mac, mic = tr.macro[k][n], tr.micro_stats[k][n]
            for i in range(2):
                assert abs(mac.means[i] - mic.means[i]) < 1e-8, (k, n, i)
    om = O.model_dw_mult(0.25, 0.4, 0.2, 0.0, 0.3)
    x1 = O.propagate_fine(om, seq[0].positions, 0, 0.0, 5e-4, S, O.slice_noise(0, 0, S, P))
    assert _rel(seq[1].positions, x1) <= TRAJ_TOL


def test_wasserstein_stop_criterion(mm, golden):
    """stop_wasserstein_tol (engine.py:244-253): stop after the first
    iteration whose max slice W1 change is <= tol; rows up to it unchanged."""
    import dataclasses
    g = golden("traces")
    model, ode, init, cfg, plan = _c1(mm)
    full = mm.run_micro_macro(model, ode, init, cfg, plan)
    N = cfg.n_slices
    deltas = [max(mm.wasserstein_1d(full.snapshots[k][n], full.snapshots[k - 1][n]) for n in range(1, N + 1))
              for k in range(1, cfg.iterations + 1)]
    big = mm.run_micro_macro(model, ode, init, dataclasses.replace(cfg, stop_wasserstein_tol=1e9), plan)
    assert big.stopped_at == 1 and big.iterations == 1
    assert np.array_equal(_packed(big, "macro"), g["c1_macro"][:2])
    tol = deltas[2]
    want = 1 + next(i for i, d in enumerate(deltas) if d <= tol)
    tr = mm.run_micro_macro(model, ode, init, dataclasses.replace(cfg, stop_wasserstein_tol=tol), plan)
    assert tr.stopped_at == want
    assert np.array_equal(_packed(tr, "macro"), g["c1_macro"][:want + 1])
    assert np.array_equal(_snap(tr), g["c1_snap"][:want + 1])


class _LocalComm:
    """Single-rank stand-in for TorchComm (no process group needed)."""
    rank, world = 0, 1

    def all_gather_rows(self, local):
        return local.clone()

    def shift_right(self, send, recv):
        pass

    def all_max(self, value):
        return value


@pytest.mark.parametrize("bimodal", [False, True])
def test_sharded_path_on_gpu_backend_equals_engine(mm, bimodal):
    """The multi-GPU driver's per-rank code (GpuBackend kernels, fused
    restriction, statuses, end-of-run gather) at world size 1 reproduces the
    single-GPU engine bit for bit."""
    from paper_2310_11365_b200.distributed import GpuBackend, run_micro_macro_sharded
    if bimodal:
        dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
        model = mm.make_double_well(dw)
        part = dw.default_partition()
        ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
        cfg = mm.PararealConfig(n_slices=8, iterations=3, slice_length=0.0625, particles=3000,
                                step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6))
        init = _bimodal_init(mm)
    else:
        model, ode, init, cfg, _ = _c1(mm, P=3000)
    plan = mm.NoisePlan(9)
    a = mm.run_micro_macro(model, ode, init, cfg, plan)
    b = run_micro_macro_sharded(model, ode, init, cfg, plan, comm=_LocalComm(), backend=GpuBackend(model, ode, cfg))
    assert np.array_equal(_packed(a, "macro"), _packed(b, "macro"))
    assert np.array_equal(_packed(a, "micro_stats"), _packed(b, "micro_stats"))
    assert np.array_equal(_snap(a), _snap(b))


@pytest.mark.parametrize("N,K", [(1, 0), (1, 1), (3, 0), (4, 4), (5, 2)])
def test_small_shapes_against_oracle(mm, N, K):
    """Degenerate run shapes (K = 0, N = 1, K = N) against the oracle, bitwise."""
    P = 777
    model, ode, init, _, _ = _c1(mm, P=P)
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=0.05, particles=P,
                            step=mm.StepConfig(dt=1e-3, steps_per_slice=50), integrator=mm.EulerConfig(1e-2))
    rng = np.random.default_rng(N * 10 + K)
    ens0 = rng.normal(1.0, 0.1, P)
    tr = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(3))
    om = O.model_ou(-1.0, 0.5, 0.5)
    ref = O.run_micro_macro(om, O.ode_unimodal(om), ens0, N, K, 0.05, 1e-3, 50, 3, integ=O.Euler(1e-2))
    assert tr.iterations == K and tr.n_slices == N
    assert np.array_equal(_packed(tr, "macro"), ref.macro)
    assert np.array_equal(_packed(tr, "micro_stats"), ref.micro)
    assert np.array_equal(_snap(tr), np.array([[e for e in row] for row in ref.snapshots]))


def test_fresh_noise_against_oracle(mm):
    """FRESH noise (a new stream per iteration, particles.py:55-60) against
    the oracle, bitwise, eager and graph-replayed."""
    P, N, K = 1500, 6, 3
    model, ode, init, _, _ = _c1(mm, P=P)
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=0.05, particles=P,
                            step=mm.StepConfig(dt=1e-3, steps_per_slice=50), integrator=mm.EulerConfig(1e-2))
    ens0 = np.random.default_rng(1).normal(1.0, 0.1, P)
    om = O.model_ou(-1.0, 0.5, 0.5)
    ref = O.run_micro_macro(om, O.ode_unimodal(om), ens0, N, K, 0.05, 1e-3, 50, 8, integ=O.Euler(1e-2), fresh=True)
    ref_snap = np.array([[e for e in row] for row in ref.snapshots])
    for use_graph in (False, True, True):
        tr = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(8, mm.NoiseMode.FRESH),
                                use_graph=use_graph)
        assert np.array_equal(_packed(tr, "macro"), ref.macro)
        assert np.array_equal(_snap(tr), ref_snap)
    # converged-slice coarse reuse is disabled for FRESH noise (inputs change)
    a = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(8, mm.NoiseMode.FRESH),
                           reuse_converged_coarse=True)
    b = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(8, mm.NoiseMode.FRESH),
                           reuse_converged_coarse=False)
    assert np.array_equal(_packed(a, "macro"), _packed(b, "macro"))


def test_graph_cache_eviction_and_reuse(mm):
    """Alternating configurations (plan cache of 2, eviction) keep results exact."""
    model, ode, init, cfg, plan = _c1(mm)
    import dataclasses
    cfgs = [cfg, dataclasses.replace(cfg, iterations=2), dataclasses.replace(cfg, n_slices=6, iterations=3)]
    first = [_packed(mm.run_micro_macro(model, ode, init, c, plan), "macro") for c in cfgs]
    for _ in range(2):
        for c, ref in zip(cfgs, first):
            assert np.array_equal(_packed(mm.run_micro_macro(model, ode, init, c, plan), "macro"), ref)


@pytest.mark.parametrize("use_graph", [False, True])
def test_snapshots_streamed_to_host(mm, golden, use_graph):
    """snapshots_to_host: every iterate's ensembles reach pinned host memory
    during the run (side-stream copies), equal to the device snapshots."""
    g = golden("traces")
    model, ode, init, cfg, plan = _c1(mm)
    for _ in range(2):  # second pass replays the cached graph
        tr = mm.run_micro_macro(model, ode, init, cfg, plan, snapshots_to_host=True, use_graph=use_graph)
        assert np.array_equal(tr.snapshot_positions, g["c1_snap"])
        assert np.array_equal(_snap(tr), g["c1_snap"])


def test_sharded_path_over_nccl_world_one(mm):
    """The multi-GPU driver with its real communicator (torch.distributed over
    NCCL, one rank): device all-gather / shift / max plumbing works and the run
    equals the single-GPU engine bit for bit."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2310_11365_b200.distributed import TorchComm, run_micro_macro_sharded
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        model, ode, init, cfg, plan = _c1(mm, P=3000)
        import dataclasses
        cfg = dataclasses.replace(cfg, stop_wasserstein_tol=1e-12)
        a = mm.run_micro_macro(model, ode, init, cfg, plan)
        b = run_micro_macro_sharded(model, ode, init, cfg, plan, comm=TorchComm())
        assert np.array_equal(_packed(a, "macro"), _packed(b, "macro"))
        assert np.array_equal(_snap(a), _snap(b))
        assert a.stopped_at == b.stopped_at
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("which", ["config2", "config3"])
def test_full_size_configs_2_and_3_properties(mm, which):
    """BASELINE configs 2 and 3 at full size (N = 32, P = 1e5, S = 64, K = 8 /
    10): k >= n exactness against the GPU's own serial fine solution
    (bitwise), macro/micro mean consistency after matching (unimodal), and
    slice 0 -> 1 against the oracle's numpy restatement (1e-12)."""
    if which == "config2":
        spec = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
        model = mm.make_cubic_meanfield(spec)
        ode = mm.gaussian_closure_rhs(spec)
        part = mm.SINGLE_REGION
        init = mm.InitialDistribution.normal(0.5, 0.04)
        K = 8
        om = O.model_cubic(1.0, 1.0, 1.0, 0.4)
    else:
        dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
        model = mm.make_double_well(dw)
        part = dw.default_partition()
        ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
        init = _bimodal_init(mm)
        K = 10
        om = O.model_double_well(0.25, 0.4, 0.2, 0.0, 0.5)
    N, P = 32, 100_000
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=0.0625, particles=P,
                            step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6))
    plan = mm.NoisePlan(0)
    tr = mm.run_micro_macro(model, ode, init, cfg, plan)
    seq = mm.sequential_fine(model, init, cfg, plan)
    for k in range(1, K + 1):
        for n in range(k + 1):
            assert np.array_equal(tr.snapshots[k][n].positions, seq[n].positions), (k, n)
    if part.n_regions == 1:
        # (bimodal: matched particles that cross the separatrix are not
        # re-assigned, so re-restriction need not reproduce the targets --
        # the reference's documented behaviour, coupling.py:7-9)
        for k in range(K + 1):
            for n in range(1, N + 1):
                mac, mic = tr.macro[k][n], tr.micro_stats[k][n]
                assert abs(mac.means[0] - mic.means[0]) < 1e-9 * max(1.0, abs(mac.means[0])), (k, n)
    x1 = O.propagate_fine(om, seq[0].positions, 0, 0.0, 2.0 ** -10, 64, O.slice_noise(0, 0, 64, P))
    assert _rel(seq[1].positions, x1) <= TRAJ_TOL


def _ou_pipeline_cfg(mm, N=6, K=4, S=20, P=100_000, **kw):
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * 1e-3, particles=P,
                            step=mm.StepConfig(1e-3, S), integrator=mm.EulerConfig(1e-2), **kw)
    return model, mm.unimodal_rhs(model), cfg


def test_stop_criterion_at_pipeline_size(mm):
    """stop_wasserstein_tol at an ensemble size the iteration pipeline
    supports: the run falls back to per-iteration kernels so the criterion is
    evaluated after every iteration (engine.py:244-253)."""
    import dataclasses
    model, ode, cfg = _ou_pipeline_cfg(mm)
    init, plan = mm.InitialDistribution.normal(1.0, 0.01), mm.NoisePlan(0)
    full = mm.run_micro_macro(model, ode, init, cfg, plan)
    assert mm.engine.last_run_info["pipeline"]
    N = cfg.n_slices
    deltas = [max(mm.wasserstein_1d(full.snapshots[k][n], full.snapshots[k - 1][n]) for n in range(1, N + 1))
              for k in range(1, cfg.iterations + 1)]
    tol = deltas[1]
    want = 1 + next(i for i, d in enumerate(deltas) if d <= tol)
    tr = mm.run_micro_macro(model, ode, init, dataclasses.replace(cfg, stop_wasserstein_tol=tol), plan)
    assert not mm.engine.last_run_info["pipeline"]
    assert tr.stopped_at == want and tr.iterations == want
    assert np.array_equal(_packed(tr, "macro"), _packed(full, "macro")[:want + 1])
    assert np.array_equal(_snap(tr), _snap(full)[:want + 1])


def test_callable_increments_at_pipeline_size(mm):
    """Per-iteration increment callables at P = 1e5 (pipeline-sized) are
    consumed every iteration, bitwise against the oracle."""
    N, K, S, P = 4, 3, 5, 100_000
    model, ode, cfg = _ou_pipeline_cfg(mm, N=N, K=K, S=S, P=P)
    rng = np.random.default_rng(9)
    xi = rng.standard_normal((N, S, P))
    inc = lambda n, k: xi[(n + k) % N]  # noqa: E731  (differs per iteration)
    ens0 = rng.normal(1.0, 0.1, P)
    tr = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(ens0), cfg, mm.NoisePlan(0), increments=inc)
    assert not mm.engine.last_run_info["pipeline"]
    om = O.model_ou(-1.0, 0.5, 0.5)
    ref = O.run_micro_macro(om, O.ode_unimodal(om), ens0, N, K, S * 1e-3, 1e-3, S, 0, integ=O.Euler(1e-2),
                            noise=inc)
    assert np.array_equal(_packed(tr, "macro"), ref.macro)
    assert np.array_equal(_snap(tr), np.array([[e for e in row] for row in ref.snapshots]))


def test_cached_plan_copy_on_reuse(mm):
    """A second graph-replayed run of the same configuration with another
    initial ensemble must not change the first trace's snapshots (rows read
    before and after the second run)."""
    model, ode, init, cfg, plan = _c1(mm, P=2000, N=6, K=3)
    rng = np.random.default_rng(5)
    e1, e2 = rng.normal(1.0, 0.1, 2000), rng.normal(0.5, 0.3, 2000)
    want = _snap(mm.run_micro_macro(model, ode, mm.ParticleEnsemble(e1), cfg, plan, use_graph=False))
    mm.engine.clear_graph_cache()
    a = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(e1), cfg, plan)
    early = a.snapshots[2][3]
    early_dev = early.device_positions
    b = mm.run_micro_macro(model, ode, mm.ParticleEnsemble(e2), cfg, plan)
    assert np.array_equal(_snap(a), want)
    assert np.array_equal(early.device_positions.cpu().numpy(), want[2][3])
    assert early.device_positions.data_ptr() != early_dev.data_ptr()
    assert not np.array_equal(_snap(b), want)
    assert np.array_equal(_snap(b), _snap(mm.run_micro_macro(model, ode, mm.ParticleEnsemble(e2), cfg, plan,
                                                             use_graph=False)))
