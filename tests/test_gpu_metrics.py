"""GPU parity: error metrics (metrics.cu + paper_2310_11365_b200/metrics.py)
and batched floor replicas against the reference's golden values -- all
bitwise (sorting is exact, the means follow numpy's pairwise tree, the
2-norms are the reference's numpy expressions on the same doubles)."""

import numpy as np
import pytest

from oracle import mm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import paper_2310_11365_b200 as mm
    mm._lib.load()
    return mm


def _c1(mm, P=1000):
    spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
    model = mm.make_perturbed_ou(spec)
    cfg = mm.PararealConfig(n_slices=10, iterations=5, slice_length=0.1, particles=P,
                            step=mm.StepConfig(dt=1e-3, steps_per_slice=100), integrator=mm.EulerConfig(1e-2))
    return model, mm.unimodal_rhs(model), mm.InitialDistribution.normal(1.0, 0.01), cfg


def _report(r):
    return (np.array([r.e_mean, r.e_var, r.e_wass, r.normalized_mean, r.normalized_var, r.normalized_wass]),
            np.array([r.mean_err_per_slice, r.var_err_per_slice, r.wass_per_slice]))


def test_relative_errors_match_reference(mm, golden):
    g = golden("metrics")
    model, ode, init, cfg = _c1(mm)
    tr = mm.run_micro_macro(model, ode, init, cfg, mm.NoisePlan(0))
    for k in range(tr.iterations + 1):
        for pre, vd in (("rel_", "variance"), ("relm_", "mean")):
            scal, per = _report(mm.relative_errors(tr, k, var_denominator=vd))
            assert np.array_equal(scal, g[f"{pre}c1_k{k}_scalars"]), (k, vd)
            assert np.array_equal(per, g[f"{pre}c1_k{k}_per_slice"]), (k, vd)
    scal, _ = _report(mm.relative_errors(tr, 1, reference_k=3))
    assert np.array_equal(scal, g["rel_c1_k1_ref3_scalars"])
    with pytest.raises(ValueError):
        mm.relative_errors(tr, 9)
    with pytest.raises(ValueError):
        mm.relative_errors(tr, 0, var_denominator="bogus")


def test_floor_replicas_match_reference(mm, golden):
    g = golden("metrics")
    model, _, init, cfg = _c1(mm)
    plans = [mm.NoisePlan(int(s)) for s in g["floor_seeds"]]
    paths = mm.sequential_fine_batch(model, init, cfg, plans)
    finals = [p[-1] for p in paths]
    assert np.array_equal(np.array([f.positions for f in finals]), g["floor_final_positions"])
    # batched replicas == separate serial runs, bitwise
    one = mm.sequential_fine(model, init, cfg, plans[1])
    assert all(np.array_equal(a.positions, b.positions) for a, b in zip(one, paths[1]))
    for vd in ("variance", "mean"):
        fl = mm.floor_from_references(paths, vd)
        assert np.array_equal(np.array([fl.e_mean, fl.e_var, fl.e_wass, fl.n_replicas]), g[f"floor_{vd}"]), vd
    assert mm.statistical_floor(finals) == g["floor_raw"][0]
    assert np.array_equal(np.array(mm.moment_spread(finals)), g["floor_spread"])
    with pytest.raises(ValueError):
        mm.floor_from_references(paths[:1])


def test_wasserstein_examples(mm, golden):
    g = golden("metrics")
    a, b = g["w1_a"], g["w1_b"]
    assert [mm.wasserstein_1d(a, b), mm.wasserstein_1d(b, a), mm.wasserstein_1d(a, a)] == list(g["w1_ab"])
    with pytest.raises(mm.UnsupportedComparison):
        mm.wasserstein_1d(a, b[:-1])
    with pytest.raises(mm.UnsupportedComparison):
        mm.wasserstein_1d([], [])


@pytest.mark.parametrize("P", [1, 7, 100_000, 1 << 20])
def test_wasserstein_sizes_against_oracle(mm, P):
    rng = np.random.default_rng(P)
    a = rng.standard_normal(P)
    b = rng.standard_t(3, P)
    assert mm.wasserstein_1d(a, b) == O.w1(a, b)


def test_floor_config4_size(mm):
    """Floor of config-4-size replicas (P = 1e5, 3 replicas x 4 slices)
    against the oracle's restatement on the GPU's own trajectories."""
    model, _, init, cfg = _c1(mm, P=100_000)
    import dataclasses
    cfg = dataclasses.replace(cfg, n_slices=4, iterations=2)
    paths = mm.sequential_fine_batch(model, init, cfg, [mm.NoisePlan(s) for s in (11, 12, 13)])
    host = [[e.positions for e in p] for p in paths]
    fl = mm.floor_from_references(paths)
    assert np.array_equal(np.array([fl.e_mean, fl.e_var, fl.e_wass, fl.n_replicas]), O.floor_from_references(host))


def test_fd_histograms_match_reference(mm, golden):
    """Freedman-Diaconis edges and histogram counts of the harness's
    histogram.csv (harness.py:209-227, 300-323) on the device."""
    g = golden("metrics")
    model, ode, init, cfg = _c1(mm)
    tr = mm.run_micro_macro(model, ode, init, cfg, mm.NoisePlan(0))
    for n in (1, 5, 10):
        data = [tr.snapshots[k][n] for k in range(tr.iterations + 1)]
        edges = mm.metrics.fd_edges(tr.snapshots[tr.iterations][n], data + [tr.snapshots[tr.iterations][n]])
        assert np.array_equal(edges, g[f"hist_c1_n{n}_edges"]), n
        assert np.array_equal(mm.metrics.histograms(data, edges), g[f"hist_c1_n{n}_counts"]), n


@pytest.mark.parametrize("P", [1, 10, 4097, 100_000])
def test_histogram_edge_cases_against_numpy(mm, P):
    rng = np.random.default_rng(P)
    x = np.round(rng.normal(0.0, 1.0, P), 2)  # values on the edges
    for edges in (np.linspace(-1.0, 1.0, 11), np.array([-5.0, 0.0, 0.0, 5.0]), np.array([0.0, 0.01])):
        assert np.array_equal(mm.metrics.histogram(x, edges), np.histogram(x, edges)[0])
