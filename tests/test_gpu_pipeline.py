"""GPU parity of the iteration pipeline (mmpr_parareal_pipeline: iterations
1..K as one persistent, dependency-driven kernel) against the per-iteration
kernel sequence (MMPR_PIPELINE=0) -- bit for bit, every trace field -- and
against the oracle (trajectories 1e-12, moments 1e-10)."""

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


def _run(mm, monkeypatch, pipeline, *args, **kw):
    monkeypatch.setenv("MMPR_PIPELINE", "1" if pipeline else "0")
    mm.engine.clear_graph_cache()
    tr = mm.run_micro_macro(*args, **kw)
    assert mm.engine.last_run_info["pipeline"] is pipeline
    out = {"macro": _packed(tr, "macro"), "micro": _packed(tr, "micro_stats"),
           "gaps": np.array(tr.fraction_gaps, dtype=float), "clamp": np.array(tr.clamp_events, dtype=float),
           "lift": np.array(tr.lift_collapses, dtype=float)}
    if tr.snapshots is not None:
        out["snap"] = np.array([[e.positions for e in row] for row in tr.snapshots])
    mm.engine.clear_graph_cache()
    return out


def _same(a, b):
    assert a.keys() == b.keys()
    for key in a:
        assert a[key].shape == b[key].shape, key
        assert np.array_equal(a[key], b[key]), key


def _ou_case(mm, N, K, S, P=100_000, retain=True, dt=1e-3):
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * dt, particles=P,
                            step=mm.StepConfig(dt, S), integrator=mm.EulerConfig(1e-2), retain_snapshots=retain)
    return model, mm.unimodal_rhs(model), mm.InitialDistribution.normal(1.0, 0.01), cfg


@pytest.mark.parametrize("N,K,S,P", [(6, 4, 20, 100_000), (3, 1, 10, 100_000), (4, 4, 10, 98_307),
                                     (40, 3, 6, 100_000), (20, 6, 4, 106_496),
                                     # smaller clusters of the 13-element geometry (8 x 512, 8 x 256 threads; tail)
                                     (4, 3, 8, 50_000), (4, 3, 8, 25_000), (3, 2, 6, 49_157),
                                     # the 10-element geometry (config 1: 4 x 256; 8 x 256, 8 x 512, 16 x 512,
                                     # 2 x 256 threads; tail; more slices than iterations, as many)
                                     (5, 3, 10, 10_000), (4, 3, 8, 20_000), (4, 2, 6, 40_000), (3, 2, 6, 80_000),
                                     (4, 3, 8, 5_000), (4, 3, 8, 9_221), (12, 5, 10, 10_000), (6, 6, 5, 10_000),
                                     # the 16-element geometry (powers of two and sizes just below: 4 x 256,
                                     # 2 x 256, 8 x 256, 8 x 512 and 16 x 512 threads -- the last two with one
                                     # CTA per SM, 64 KB per increment stage; tail)
                                     (5, 3, 8, 16_384), (4, 2, 6, 8_192), (4, 3, 6, 32_768), (4, 2, 6, 65_536),
                                     (20, 3, 4, 131_072), (4, 3, 8, 7_685), (3, 2, 6, 122_885),
                                     # the any-size form (16 per lane, at least 8 populated): 9..15 elements,
                                     # ragged leaves, tails, the smallest and largest ensembles of one cluster
                                     (4, 3, 8, 9_999), (4, 3, 8, 30_000), (3, 2, 6, 70_000), (3, 2, 6, 120_001),
                                     (4, 2, 6, 4_608), (4, 3, 8, 12_345), (6, 4, 10, 60_000), (3, 3, 6, 90_000),
                                     # ragged sizes on the specialised forms (13 / 10 per lane + a tail element)
                                     (4, 3, 8, 99_999), (4, 3, 8, 100_003), (4, 3, 8, 10_001)])
def test_pipeline_equals_per_iteration_kernels_ou(mm, monkeypatch, N, K, S, P):
    model, ode, init, cfg = _ou_case(mm, N, K, S, P)
    plan = mm.NoisePlan(0)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan)
    _same(a, b)


def test_pipeline_ou_matches_oracle_bitwise(mm, monkeypatch):
    N, K, S, P = 6, 4, 20, 100_000
    model, ode, init, cfg = _ou_case(mm, N, K, S, P)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, mm.NoisePlan(0))
    om = O.model_ou(-1.0, 0.5, 0.5)
    ens0 = O.sample_normal_initial(0, 1.0, 0.01, P)
    ref = O.run_micro_macro(om, O.ode_unimodal(om), ens0, N, K, S * 1e-3, 1e-3, S, 0, integ=O.Euler(1e-2))
    # numpy-exact noise (tail draws included) and numpy-order arithmetic:
    # every snapshot and macro state equals the reference's bit for bit
    ref_snap = np.array([[e for e in row] for row in ref.snapshots])
    assert np.array_equal(a["snap"], ref_snap)
    assert np.array_equal(a["macro"], np.asarray(ref.macro))
    assert np.array_equal(a["micro"], np.asarray(ref.micro))


def test_pipeline_without_retained_snapshots(mm, monkeypatch):
    model, ode, init, cfg = _ou_case(mm, 8, 5, 8, retain=False)
    plan = mm.NoisePlan(0)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan)
    _same(a, b)
    # and the retained run's macro rows are the same numbers
    model, ode, init, cfg = _ou_case(mm, 8, 5, 8, retain=True)
    c = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    assert np.array_equal(a["macro"], c["macro"]) and np.array_equal(a["micro"], c["micro"])


def test_pipeline_cubic_gaussian_closure(mm, monkeypatch):
    """BASELINE config 2's model and closure at reduced N / K."""
    spec = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
    model = mm.make_cubic_meanfield(spec)
    cfg = mm.PararealConfig(n_slices=10, iterations=5, slice_length=0.0625, particles=100_000,
                            step=mm.StepConfig(2.0 ** -10, 64), integrator=mm.EulerConfig(2.0 ** -6))
    args = (model, mm.gaussian_closure_rhs(spec), mm.InitialDistribution.normal(0.5, 0.04), cfg, mm.NoisePlan(0))
    a = _run(mm, monkeypatch, True, *args)
    b = _run(mm, monkeypatch, False, *args)
    _same(a, b)


def _bimodal_case(mm, N, K, S, P=100_000, retain=True, init=None):
    """BASELINE config 3's model, partition and closure at reduced N / K / S."""
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    model = mm.make_double_well(dw)
    part = dw.default_partition()
    dt = 2.0 ** -10
    cfg = mm.PararealConfig(n_slices=N, iterations=K, slice_length=S * dt, particles=P, step=mm.StepConfig(dt, S),
                            partition=part, integrator=mm.EulerConfig(2.0 ** -6), retain_snapshots=retain)
    ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
    return model, ode, init or mm.bimodal_initial(-1.0, 1.0, 0.2), cfg


@pytest.mark.parametrize("N,K,S,P,retain", [(8, 4, 16, 100_000, True), (20, 3, 8, 100_000, False),
                                            (5, 5, 8, 98_307, True), (3, 1, 4, 106_496, True),
                                            (6, 3, 8, 50_000, True), (4, 2, 8, 25_000, False),
                                            (4, 3, 8, 99_999, True)])
def test_pipeline_bimodal_equals_per_iteration_kernels(mm, monkeypatch, N, K, S, P, retain):
    """Two regions (config 3): per-region match with pre-transform
    membership and region restrictions over compacted members inside the
    units -- every trace field bit for bit against the per-iteration
    kernels (separate match + multi-kernel restriction)."""
    model, ode, init, cfg = _bimodal_case(mm, N, K, S, P, retain)
    plan = mm.NoisePlan(0)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan)
    _same(a, b)


def test_pipeline_bimodal_degenerate_match_like_reference(mm, monkeypatch):
    """An ensemble started right of the separatrix: the reference (the
    oracle) raises DegenerateMatch for region 0 in this run; the pipeline's
    per-region match raises the same error as the per-iteration kernels."""
    model, ode, _, cfg = _bimodal_case(mm, 6, 3, 8)
    init = mm.InitialDistribution.normal(1.0, 0.05)
    plan = mm.NoisePlan(0)
    with pytest.raises(mm.DegenerateMatch) as ea:
        _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    with pytest.raises(mm.DegenerateMatch) as eb:
        _run(mm, monkeypatch, False, model, ode, init, cfg, plan)
    assert ea.value.region == eb.value.region == 0
    assert str(ea.value) == str(eb.value)


def test_pipeline_bimodal_matches_oracle(mm, monkeypatch):
    """Against the numpy restatement: trajectories within 1e-12, moments
    within 1e-10 (the double well's x**3 is numpy's vectorised pow)."""
    N, K, S, P = 4, 3, 16, 100_000
    model, ode, init, cfg = _bimodal_case(mm, N, K, S, P)
    plan = mm.NoisePlan(0)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    ens0 = mm.sample_initial(init, plan, P).positions.copy()
    om = O.model_double_well(0.25, 0.4, 0.2, 0.0, 0.5)
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    part = dw.default_partition()
    opart = O.Partition(tuple(part.separatrices), tuple(part.peaks))
    oode = O.ode_multimodal(om, opart, dw.potential, dw.sigma)
    ref = O.run_micro_macro(om, oode, ens0, N, K, S * 2.0 ** -10, 2.0 ** -10, S, 0, integ=O.Euler(2.0 ** -6),
                            part=opart)
    ref_snap = np.array([[e for e in row] for row in ref.snapshots])
    dx = np.max(np.abs(a["snap"] - ref_snap)) / max(1.0, np.max(np.abs(ref_snap)))
    dm = np.max(np.abs(a["macro"] - np.asarray(ref.macro))) / max(1.0, np.max(np.abs(ref.macro)))
    du = np.max(np.abs(a["micro"] - np.asarray(ref.micro))) / max(1.0, np.max(np.abs(ref.micro)))
    assert dx <= 1e-12, dx
    assert dm <= 1e-10 and du <= 1e-10, (dm, du)


@pytest.mark.parametrize("mode", ["PHILOX", "PHILOX_FRESH"])
def test_pipeline_counter_noise_equals_per_iteration_kernels(mm, monkeypatch, mode):
    """Counter-based noise generated in registers by the pipeline's units
    (FRESH: unit (k, n) draws iteration k's field) -- bitwise the
    per-iteration sweeps with the same counter noise."""
    model, ode, init, cfg = _ou_case(mm, 6, 3, 12)
    plan = mm.NoisePlan(0, getattr(mm.NoiseMode, mode))
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan)
    _same(a, b)


def test_small_geometry_is_one_rank_numpy_noise_only(mm, monkeypatch):
    """The 10-element geometry and the two-region units exist for one rank
    and numpy-stream / injected increments: with counter noise the engine
    keeps the per-iteration kernels (and still matches the pipeline-free
    run bit for bit, trivially), and the support query says so."""
    from paper_2310_11365_b200 import kernels
    from paper_2310_11365_b200.models import device_model
    from paper_2310_11365_b200.moments import device_ode
    from paper_2310_11365_b200.rk54 import integrator_descriptor
    model, ode, init, cfg = _ou_case(mm, 4, 2, 6, 10_000)
    ode_d, ode_model_d = device_ode(ode)
    args = (device_model(model), ode_d, ode_model_d, integrator_descriptor(cfg.integrator))
    assert kernels.pipeline_supported(*args, 10_000)
    assert not kernels.pipeline_supported(*args, 10_000, counter_noise=True)
    assert not kernels.pipeline_supported(*args, 10_000, n_ranks=2)
    assert kernels.pipeline_supported(*args, 100_000, counter_noise=True, n_ranks=2)
    assert kernels.pipeline_supported(*args, 9_999) and not kernels.pipeline_supported(*args, 9_999, counter_noise=True)
    assert not kernels.pipeline_supported(*args, 4_096)
    monkeypatch.setenv("MMPR_PIPELINE", "1")
    mm.engine.clear_graph_cache()
    mm.run_micro_macro(model, ode, init, cfg, mm.NoisePlan(0, mm.NoiseMode.PHILOX))
    assert mm.engine.last_run_info["pipeline"] is False
    mm.engine.clear_graph_cache()


def test_pipeline_cubic_small_geometry(mm, monkeypatch):
    """The cubic mean-field model with its Gaussian closure at P = 2e4 (10 elements per lane, 8 x 256 threads)."""
    spec = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
    model = mm.make_cubic_meanfield(spec)
    cfg = mm.PararealConfig(n_slices=6, iterations=3, slice_length=0.03125, particles=20_000,
                            step=mm.StepConfig(2.0 ** -10, 32), integrator=mm.EulerConfig(2.0 ** -6))
    args = (model, mm.gaussian_closure_rhs(spec), mm.InitialDistribution.normal(0.5, 0.04), cfg, mm.NoisePlan(0))
    a = _run(mm, monkeypatch, True, *args)
    b = _run(mm, monkeypatch, False, *args)
    _same(a, b)


def test_pipeline_without_converged_reuse_and_injected(mm, monkeypatch):
    model, ode, init, cfg = _ou_case(mm, 5, 3, 12)
    plan = mm.NoisePlan(0)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan, reuse_converged_coarse=False)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan, reuse_converged_coarse=False)
    _same(a, b)
    import torch
    gen = torch.Generator(device="cuda").manual_seed(7)
    xi = torch.randn((5, 12, 100_000), dtype=torch.float64, device="cuda", generator=gen)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan, increments=xi)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan, increments=xi)
    _same(a, b)


def test_pipeline_eager_timings(mm, monkeypatch):
    model, ode, init, cfg = _ou_case(mm, 4, 2, 5)
    monkeypatch.setenv("MMPR_PIPELINE", "1")
    tr = mm.run_micro_macro(model, ode, init, cfg, mm.NoisePlan(0), record_timings=True)
    assert mm.engine.last_run_info["pipeline"]
    assert sum(tr.stage_timings["iterations"]) > 0.0
    assert len(tr.timings["fine"]) == 4 * 2 and all(v > 0.0 for v in tr.timings["fine"])
    assert set(tr.timings) == {"coarse", "fine", "restrict", "match"}


def test_pipeline_blowup_is_reported_like_the_sweep(mm, monkeypatch):
    """A diverging ensemble raises NumericalBlowup at the same (slice, step)
    on both paths (the pipeline finishes its units and reports afterwards)."""
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=1e5, a_E=0.0, B=0.5))
    cfg = mm.PararealConfig(n_slices=6, iterations=3, slice_length=0.1, particles=100_000,
                            step=mm.StepConfig(1e-3, 100), integrator=mm.EulerConfig(1e-2))
    errs = []
    for pipeline in (True, False):
        monkeypatch.setenv("MMPR_PIPELINE", "1" if pipeline else "0")
        mm.engine.clear_graph_cache()
        with pytest.raises(mm.NumericalBlowup) as e:
            mm.run_micro_macro(model, mm.unimodal_rhs(model), mm.InitialDistribution.normal(1.0, 0.01), cfg,
                               mm.NoisePlan(0))
        errs.append((e.value.slice_index, e.value.step_index))
        assert mm.engine.last_run_info["pipeline"] is pipeline
    mm.engine.clear_graph_cache()
    assert errs[0] == errs[1]


def test_pipeline_full_config4(mm, monkeypatch):
    """BASELINE config 4 at one GPU (N = 64, P = 1e5, S = 100, K = 5): the
    pipeline's trace equals the per-iteration kernels' bit for bit."""
    model, ode, init, cfg = _ou_case(mm, 64, 5, 100)
    plan = mm.NoisePlan(0)
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan)
    _same(a, b)


def _emulated_ranks(mm, G, model, ode, init, cfg, plan, epochs=1, sys_scope=False):
    """The multi-rank pipeline over G ranks on one GPU: per-rank buffers and
    prologues, ONE launch over every rank's units (ranks reading each other's
    exchange arrays), merged like the multi-GPU driver does."""
    import torch
    from paper_2310_11365_b200 import sharded_pipeline as SP
    from paper_2310_11365_b200.models import device_model
    from paper_2310_11365_b200.moments import device_ode
    from paper_2310_11365_b200.rk54 import integrator_descriptor
    N, K, P, S = cfg.n_slices, cfg.iterations, cfg.particles, cfg.step.steps_per_slice
    model_d = device_model(model)
    ode_d, odm = device_ode(ode)
    integ_d = integrator_descriptor(cfg.integrator)
    times = torch.tensor([cfg.t_start + n * cfg.slice_length for n in range(N + 1)], dtype=torch.float64,
                         device="cuda")
    x0 = mm.sample_initial(init, plan, P).device_positions
    ranks = [SP.RankBuffers(r, G, N, K, P, S, cfg.retain_snapshots) for r in range(G)]
    for epoch in range(1, epochs + 1):
        for rb in ranks:
            rb.prologue(ode_d, odm, integ_d, times, x0, plan.master_seed)
        ios = [rb.io(times) for rb in ranks]
        SP.launch(model_d, ode_d, odm, integ_d, cfg.step.dt, S, True, ios, 0, G, epoch, epochs == 1, sys_scope, N, K,
                  P)
    torch.cuda.synchronize()
    Ng = N // G
    out = {}
    for name, kind in (("macro", "boundary"), ("micro", "boundary"), ("micro_counts", "boundary"),
                       ("fine_stats", "slice"), ("fine_counts", "slice"), ("bad", "slice"), ("raw", "shifted"),
                       ("cache", "shifted"), ("coarse_status", "shifted"), ("match_status", "shifted")):
        out[name] = SP.merge_rows([getattr(rb, name).cpu().numpy() for rb in ranks], Ng, G, N, kind)
    rows = ranks[0].snap.shape[0]
    snap = np.stack([ranks[SP.owner(n, Ng, G)].snap[:, n].cpu().numpy() for n in range(N + 1)], axis=1)
    out["snap"] = snap[:rows]
    return out


@pytest.mark.parametrize("G,N,K,rank_tickets", [(2, 8, 4, 0), (4, 16, 5, 0), (8, 16, 3, 0), (3, 9, 9, 0),
                                                (2, 16, 4, 1), (4, 16, 5, 1), (8, 32, 3, 1)])
def test_multi_rank_pipeline_emulated_on_one_gpu(mm, monkeypatch, G, N, K, rank_tickets):
    """Ranks exchange only through each other's exchange arrays and flags;
    the merged result equals the single-rank pipeline bit for bit -- with one
    global unit order, and with every rank taking only its own units on its
    own clusters (MMPR_PIPELINE_RANK_TICKETS=1: the multi-GPU schedule, in
    which ranks wait on their predecessor's coarse chain)."""
    monkeypatch.setenv("MMPR_PIPELINE_RANK_TICKETS", str(rank_tickets))
    model, ode, init, cfg = _ou_case(mm, N, K, 12)
    plan = mm.NoisePlan(0)
    ref = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    emu = _emulated_ranks(mm, G, model, ode, init, cfg, plan)
    assert np.array_equal(emu["macro"], ref["macro"])
    assert np.array_equal(emu["micro"], ref["micro"])
    assert np.array_equal(emu["snap"], ref["snap"])
    for name in ("bad", "coarse_status", "match_status"):
        assert (emu[name] == mm._lib.STAT_OK).all(), name


def test_multi_rank_pipeline_system_scope(mm, monkeypatch):
    """The multi-GPU instruction paths (ld.acquire.sys / st.release.sys /
    red.release.sys, uncached loads of a peer's outputs) executed on one
    GPU under the per-rank schedule: same bits."""
    monkeypatch.setenv("MMPR_PIPELINE_RANK_TICKETS", "1")
    model, ode, init, cfg = _ou_case(mm, 16, 4, 10)
    plan = mm.NoisePlan(0)
    ref = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    emu = _emulated_ranks(mm, 4, model, ode, init, cfg, plan, sys_scope=True)
    assert np.array_equal(emu["macro"], ref["macro"])
    assert np.array_equal(emu["snap"], ref["snap"])


def test_multi_rank_pipeline_epochs(mm, monkeypatch):
    """Flags accumulate across runs (no reset between them): the second run,
    waiting for epoch 2, reproduces the first."""
    model, ode, init, cfg = _ou_case(mm, 8, 3, 10, retain=False)
    plan = mm.NoisePlan(0)
    one = _emulated_ranks(mm, 4, model, ode, init, cfg, plan, epochs=1)
    two = _emulated_ranks(mm, 4, model, ode, init, cfg, plan, epochs=2)
    for key in one:
        assert np.array_equal(one[key], two[key]), key
    ref = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    assert np.array_equal(one["macro"], ref["macro"])


def test_sharded_driver_takes_the_pipeline_over_nccl_world_one(mm, monkeypatch):
    """run_micro_macro_sharded with its real communicator (NCCL, one rank)
    runs the multi-GPU pipeline path (rank buffers, epoch-tagged flags, the
    ownership merge) and equals the single-GPU engine bit for bit, run after
    run (flags accumulate across epochs)."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2310_11365_b200 import distributed as D
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    monkeypatch.setenv("MMPR_SHARDED_PIPELINE", "1")
    try:
        model, ode, init, cfg = _ou_case(mm, 8, 4, 16)
        plan = mm.NoisePlan(0)
        ref = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
        for _ in range(3):
            tr = D.run_micro_macro_sharded(model, ode, init, cfg, plan, comm=D.TorchComm())
            assert D.last_run_info["pipeline"]
            assert np.array_equal(_packed(tr, "macro"), ref["macro"])
            assert np.array_equal(_packed(tr, "micro_stats"), ref["micro"])
            assert np.array_equal(np.array([[e.positions for e in row] for row in tr.snapshots]), ref["snap"])
            assert np.array_equal(np.array(tr.fraction_gaps, dtype=float), ref["gaps"])
    finally:
        dist.destroy_process_group()


def _ipc_worker(rank, port, result_path):
    """One of two processes on GPU 0: export an exchange block, open the
    other rank's through CUDA IPC, read its macro array (no kernel waits on
    the other process)."""
    import ctypes
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        import paper_2310_11365_b200 as mm
        from paper_2310_11365_b200 import _lib, sharded_pipeline as SP
        from paper_2310_11365_b200.distributed import TorchComm
        comm = TorchComm()
        rb = SP.RankBuffers(rank, 2, 8, 2, 100_000, 4, False, raw_exchange=True)
        rb.macro.copy_(torch.full_like(rb.macro, 10.0 + rank))
        torch.cuda.synchronize()
        handle = (ctypes.c_ubyte * 64)()
        _lib.call("mmpr_ipc_handle", ctypes.c_void_p(rb.block.ptr), handle)
        handles = comm.all_gather_bytes(bytes(handle))
        other = 1 - rank
        ptr = ctypes.c_void_p()
        _lib.call("mmpr_ipc_open", (ctypes.c_ubyte * 64).from_buffer_copy(handles[other]), ctypes.byref(ptr))
        io = rb.peer_io(int(ptr.value), rb.io(torch.zeros(9, dtype=torch.float64, device="cuda")))

        class _View:
            pass
        v = _View()
        v.__cuda_array_interface__ = {"shape": (rb.macro.numel(),), "typestr": "<f8", "data": (io.macro, False),
                                      "version": 2}
        seen = torch.as_tensor(v, device="cuda").clone()
        torch.cuda.synchronize()
        ok = bool((seen == 10.0 + other).all())
        dist.barrier()  # the peer keeps its block alive until both have read
        _lib.call("mmpr_ipc_close", ptr)
        rb.free()
        with open(f"{result_path}.{rank}", "w") as fh:
            fh.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


def test_exchange_block_ipc_roundtrip(tmp_path):
    """The multi-GPU pipeline's plumbing: an exchange block exported by one
    process is mapped by another (cudaIpcOpenMemHandle) at the exchange-layout
    offsets peer_io computes."""
    import socket
    import torch.multiprocessing as tmp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "ipc")
    tmp.spawn(_ipc_worker, args=(port, path), nprocs=2, join=True)
    assert open(path + ".0").read() == "ok"
    assert open(path + ".1").read() == "ok"


@pytest.mark.parametrize("case", ["perturbed_ou_closure", "linear", "cubic_unimodal"])
def test_pipeline_other_instantiations_equal_per_iteration(mm, monkeypatch, case):
    """Every (model, closure) pair with a pipeline instantiation, against the
    per-iteration kernels, bit for bit (linear: multiplicative noise b(x))."""
    if case == "perturbed_ou_closure":
        spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
        model, ode = mm.make_perturbed_ou(spec), mm.perturbed_ou_rhs(spec)
    elif case == "linear":
        model = mm.make_linear(mm.LinearMcKVSpec(A=-1.0, A_E=0.3, A_0=0.1, B=0.05, B_E=0.0, B_0=0.4))
        ode = mm.unimodal_rhs(model)
    else:
        model = mm.make_cubic_meanfield(mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4))
        ode = mm.unimodal_rhs(model)
    cfg = mm.PararealConfig(n_slices=6, iterations=3, slice_length=0.02, particles=100_000,
                            step=mm.StepConfig(1e-3, 20), integrator=mm.EulerConfig(1e-2))
    args = (model, ode, mm.InitialDistribution.normal(0.8, 0.04), cfg, mm.NoisePlan(5))
    a = _run(mm, monkeypatch, True, *args)
    b = _run(mm, monkeypatch, False, *args)
    _same(a, b)


def test_pipeline_watchdog_is_recoverable(mm, monkeypatch):
    """An expired dependency wait (forced with a tiny watchdog) ends the
    launch cleanly with MMPR_STAT_WATCHDOG statuses -> MmprError, and the
    CUDA context stays usable (no sticky trap)."""
    model, ode, init, cfg = _ou_case(mm, 8, 4, 20)
    plan = mm.NoisePlan(0)
    monkeypatch.setenv("MMPR_PIPELINE_WATCHDOG", "1")
    with pytest.raises(mm._lib.MmprError, match="watchdog"):
        mm.run_micro_macro(model, ode, init, cfg, plan, use_graph=False)
    monkeypatch.delenv("MMPR_PIPELINE_WATCHDOG")
    a = _run(mm, monkeypatch, True, model, ode, init, cfg, plan)
    b = _run(mm, monkeypatch, False, model, ode, init, cfg, plan)
    _same(a, b)
