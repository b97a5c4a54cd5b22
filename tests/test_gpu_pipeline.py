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
                                     (40, 3, 6, 100_000), (20, 6, 4, 106_496)])
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
    # the device's Marsaglia-tail draws may differ from numpy's by one ulp
    # (log1p), so trajectories are held to the acceptance-1 metric
    ref_snap = np.array([[e for e in row] for row in ref.snapshots])
    assert np.max(np.abs(a["snap"] - ref_snap)) / max(1.0, np.max(np.abs(ref_snap))) <= 1e-12
    ref_macro = np.asarray(ref.macro)
    assert np.max(np.abs(a["macro"] - ref_macro)) / max(1.0, np.max(np.abs(ref_macro))) <= 1e-10


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
    assert sum(tr.timings["iterations"]) > 0.0


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
