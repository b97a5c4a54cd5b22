"""Pin the CPU oracle (oracle/mm_oracle.py) against golden vectors produced by
the unmodified reference (tests/golden/make_golden.py).  CPU only.

Exact (bitwise) equality is required everywhere: the oracle restates the
reference's numpy operations in the same order.
"""

import math

import numpy as np
import pytest

from oracle import mm_oracle as O


def test_noise_streams_match_reference(golden):
    g = golden("noise")
    for c in range(5):
        seed, fresh, n, j, P, k = (int(v) for v in g[f"case{c}_meta"])
        got = O.step_normals(seed, n, j, P, k, fresh=bool(fresh))
        assert np.array_equal(got, g[f"case{c}_normals"]), c
    for c in range(2):
        seed, mean, var, P = g[f"init{c}_meta"]
        got = O.sample_normal_initial(int(seed), mean, var, int(P))
        assert np.array_equal(got, g[f"init{c}"])


MODEL_BUILDERS = {
    "ou": lambda: O.model_ou(-1.0, 0.5, 0.5),
    "ou_default": lambda: O.model_ou(-1.0, -0.5, 0.01),
    "linear": lambda: O.model_linear(-0.7, 0.3, 0.1, 0.2, 0.05, 0.4),
    "double_well": lambda: O.model_double_well(0.25, 0.4, 0.2, 0.0, 0.5),
    "double_well_tilt": lambda: O.model_double_well(0.25, 0.5, 0.3, 0.2, 0.7),
    "cubic": lambda: O.model_cubic(1.0, 1.0, 1.0, 0.4),
    "dw_mult": lambda: O.model_dw_mult(0.25, 0.4, 0.2, 0.0, 0.3),
}


@pytest.mark.parametrize("name", sorted(MODEL_BUILDERS))
@pytest.mark.parametrize("P", [1, 5, 1000, 1001])
def test_propagate_fine_matches_reference(golden, name, P):
    g = golden("fine")
    key = f"{name}_P{P}"
    Pm, S, dt, n, t0, seed = g[key + "_meta"]
    x0 = g[key + "_x0"]
    assert np.array_equal(x0, O.sample_normal_initial(int(seed), 0.3, 0.5, int(Pm)))
    noise = O.slice_noise(int(seed), int(n), int(S), int(Pm))
    x1 = O.propagate_fine(MODEL_BUILDERS[name](), x0, int(n), t0, dt, int(S), noise)
    assert np.array_equal(x1, g[key + "_x1"])


def test_em_step_known_answers(golden):
    g = golden("fine")
    m = O.model_ou(-1.0, -0.5, 0.01)
    assert np.array_equal(O.em_step_raw(m, np.array([100.0]), 0.0, 0.01, np.zeros(1)), g["em_zero_noise"])
    assert g["em_zero_noise"][0] == pytest.approx(98.5)
    m2 = O.model_ou(0.0, 0.0, 2.0)
    assert np.array_equal(O.em_step_raw(m2, np.array([1.0]), 0.0, 0.25, np.array([3.0])), g["em_sqrt_dt"])


PARTS = {"single": O.SINGLE, "two": O.Partition((0.0,), (-1.5, 1.5)),
         "three": O.Partition((0.0, 2.0), (-1.0, 1.0, 3.0))}


def test_restrict_matches_reference(golden):
    g = golden("coupling")
    for en in g["ens_names"]:
        x = g[f"ens_{en}"]
        for pn, part in PARTS.items():
            got, counts = O.restrict(x, part)
            ref = g[f"restrict_{pn}_{en}"]
            assert np.array_equal(got, ref), (pn, en)
            assert np.array_equal(counts < 2, g[f"restrict_{pn}_{en}_deg"]), (pn, en)


def test_match_matches_reference(golden):
    g = golden("coupling")
    names = list(g["ens_names"])
    part_list = list(PARTS.values())
    hp = g["hyp_part"]
    part_list.append(O.Partition((hp[0],), (hp[1], hp[2])))
    for c in range(10):
        pi, ei, collapse, status = (int(v) for v in g[f"match{c}_meta"])
        part = part_list[pi]
        x = g[f"ens_{names[ei]}"]
        t = g[f"match{c}_target"]
        I = part.n_regions
        target = np.concatenate([t[:I], t[I:], np.full(I, 1.0 / I)])
        policy = "collapse" if collapse else "raise"
        if status >= 0:
            with pytest.raises(O.OracleDegenerateMatch) as err:
                O.match(target, x, part, policy)
            assert err.value.region == status
        else:
            got, _ = O.match(target, x, part, policy)
            assert np.array_equal(got, g[f"match{c}_out"]), c


def _check_trace(tr, g, prefix, snapshots=True):
    assert np.array_equal(tr.macro, g[prefix + "macro"])
    assert np.array_equal(tr.micro, g[prefix + "micro"])
    if snapshots:
        snap = np.array([[e for e in row] for row in tr.snapshots])
        assert np.array_equal(snap, g[prefix + "snap"])
    assert np.array_equal(np.array(tr.clamp_events, dtype=float).reshape(-1, 4), g[prefix + "clamp"])
    assert np.array_equal(np.array(tr.fraction_gaps, dtype=float).reshape(-1, 3), g[prefix + "gaps"])
    assert np.array_equal(np.array(tr.lift_collapses, dtype=float).reshape(-1, 3), g[prefix + "lift"])


def test_trace_config1_shape_euler(golden):
    g = golden("traces")
    m = O.model_ou(-1.0, 0.5, 0.5)
    ens0 = O.sample_normal_initial(0, 1.0, 0.01, 1000)
    tr = O.run_micro_macro(m, O.ode_unimodal(m), ens0, 10, 5, 0.1, 1e-3, 100, 0, integ=O.Euler(1e-2))
    _check_trace(tr, g, "c1_")
    seq = O.sequential_fine(m, ens0, 10, 0.1, 1e-3, 100, 0)
    assert np.array_equal(np.array(seq), g["c1_seq"])
    # k >= n exactness against the serial fine solution (engine.py:11-14)
    for k in range(1, 6):
        for n in range(k + 1):
            assert np.array_equal(tr.snapshots[k][n], seq[n])


@pytest.mark.parametrize("prefix,ode_kind,seed", [("dp_", "perturbed", 77), ("dpu_", "unimodal", 78)])
def test_trace_reference_default_dp54(golden, prefix, ode_kind, seed):
    g = golden("traces")
    m = O.model_ou(-1.0, -0.5, 1.0)
    ode = O.ode_perturbed_ou(-1.0, -0.5, 1.0) if ode_kind == "perturbed" else O.ode_unimodal(m)
    ens0 = O.sample_normal_initial(seed, 1.0, 0.5, 500)
    tr = O.run_micro_macro(m, ode, ens0, 6, 4, 0.25, 0.05, 5, seed, integ=O.DP54())
    _check_trace(tr, g, prefix)


def _bimodal(seed, P):
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, 0))))
    signs = np.where(rng.random(P) < 0.5, -1.0, 1.0)
    return signs + 0.2 * rng.standard_normal(P)


def _dw_partition(alpha, gamma, J):
    tilt = J * math.sqrt(alpha / (2.0 * gamma))
    roots = np.roots([4.0 * alpha, 0.0, -2.0 * gamma, tilt])
    real = np.sort(roots[np.abs(roots.imag) < 1e-9].real)
    return O.Partition((float(real[1]),), (float(real[0]), float(real[2])))


def _potential(alpha, gamma, J):
    tilt = J * math.sqrt(alpha / (2.0 * gamma))
    return lambda x: alpha * np.asarray(x, float) ** 4 - gamma * np.asarray(x, float) ** 2 + tilt * np.asarray(x, float)


def test_trace_config3_shape_bimodal(golden):
    g = golden("traces")
    part = _dw_partition(0.25, 0.4, 0.0)
    assert np.array_equal(np.array([part.seps[0], part.peaks[0], part.peaks[1]]), g["c3_part"])
    m = O.model_double_well(0.25, 0.4, 0.2, 0.0, 0.5)
    ode = O.ode_multimodal(m, part, _potential(0.25, 0.4, 0.0), 0.5)
    ens0 = _bimodal(0, 1000)
    tr = O.run_micro_macro(m, ode, ens0, 8, 4, 0.0625, 2.0 ** -10, 64, 0, part=part, integ=O.Euler(2.0 ** -6))
    _check_trace(tr, g, "c3_")
    seq = O.sequential_fine(m, ens0, 8, 0.0625, 2.0 ** -10, 64, 0)
    assert np.array_equal(np.array(seq), g["c3_seq"])


def test_trace_config2_shape_cubic(golden):
    g = golden("traces")
    m = O.model_cubic(1.0, 1.0, 1.0, 0.4)
    ens0 = O.sample_normal_initial(0, 0.5, 0.04, 1000)
    tr = O.run_micro_macro(m, O.ode_gaussian_cubic(1.0, 1.0, 1.0, 0.4), ens0, 8, 4, 0.0625, 2.0 ** -10, 64, 0,
                           integ=O.Euler(2.0 ** -6))
    _check_trace(tr, g, "c2_")


def test_trace_config5_shape_multiplicative(golden):
    g = golden("traces")
    part = _dw_partition(0.25, 0.4, 0.0)
    m = O.model_dw_mult(0.25, 0.4, 0.2, 0.0, 0.3)
    sigma = 0.3 * math.sqrt(1.8)
    ode = O.ode_multimodal(m, part, _potential(0.25, 0.4, 0.0), sigma)
    ens0 = _bimodal(0, 1000)
    tr = O.run_micro_macro(m, ode, ens0, 4, 3, 0.1, 5e-4, 200, 0, part=part, integ=O.Euler(1e-2))
    _check_trace(tr, g, "c5_")


# ---- metrics (metrics.py:35-218) ---------------------------------------------
def test_oracle_metrics_match_reference(golden):
    g, tr = golden("metrics"), golden("traces")
    snaps = tr["c1_snap"]  # the reference trace the metrics fixture was computed on
    K = snaps.shape[0] - 1
    for k in range(K + 1):
        for pre, vd in (("rel_", "variance"), ("relm_", "mean")):
            scal, per = O.relative_errors(snaps, k, K, vd)
            assert np.array_equal(scal, g[f"{pre}c1_k{k}_scalars"]), (k, vd)
            assert np.array_equal(per, g[f"{pre}c1_k{k}_per_slice"]), (k, vd)
    scal, per = O.relative_errors(snaps, 1, 3)
    assert np.array_equal(scal, g["rel_c1_k1_ref3_scalars"])
    a, b = g["w1_a"], g["w1_b"]
    assert [O.w1(a, b), O.w1(b, a), O.w1(a, a)] == list(g["w1_ab"])


def test_oracle_floor_matches_reference(golden):
    g = golden("metrics")
    om = O.model_ou(-1.0, 0.5, 0.5)
    paths = []
    for s in g["floor_seeds"]:
        x0 = O.sample_normal_initial(int(s), 1.0, 0.01, 1000)
        paths.append(O.sequential_fine(om, x0, 10, 0.1, 1e-3, 100, int(s)))
    assert np.array_equal(np.array([p[-1] for p in paths]), g["floor_final_positions"])
    for vd in ("variance", "mean"):
        assert np.array_equal(O.floor_from_references(paths, vd), g[f"floor_{vd}"]), vd
    finals = [p[-1] for p in paths]
    assert O.statistical_floor(finals) == g["floor_raw"][0]
    assert np.array_equal(np.array(O.moment_spread(finals)), g["floor_spread"])


# ---- ROTATOR_SUM / EMPIRICAL_CDF models (models.py:61-83, 286-334) -----------
STAT_MODELS = {"rotator": lambda: O.model_rotator(0.5, 0.1, True),
               "rotator_nowrap": lambda: O.model_rotator(1.5, 0.3, False),
               "burgers": lambda: O.model_burgers(math.sqrt(0.2))}


@pytest.mark.parametrize("name", sorted(STAT_MODELS))
@pytest.mark.parametrize("P", [1, 7, 1000, 4099])
def test_oracle_stat_models_propagate_fine(golden, name, P):
    g = golden("stats")
    Pm, S, dt, n, t0, seed = g[f"{name}_P{P}_meta"]
    xi = O.slice_noise(int(seed), int(n), int(S), int(Pm))
    got = O.propagate_fine(STAT_MODELS[name](), g[f"{name}_P{P}_x0"], int(n), t0, dt, int(S), xi)
    assert np.array_equal(got, g[f"{name}_P{P}_x1"])


def test_oracle_statistics(golden):
    g = golden("stats")
    assert np.array_equal(O.statistic(O.model_burgers(1.0), g["cdf_x"]), g["cdf_s"])
    assert np.array_equal(np.array(O.statistic(O.model_rotator(0.5, 0.1), g["cdf_x"])), g["rot_s"])


@pytest.mark.parametrize("name", ["rot_uni", "rot_taylor", "burgers"])
def test_oracle_stat_model_runs(golden, name):
    g = golden("stats")
    om = O.model_burgers(math.sqrt(0.2)) if name == "burgers" else O.model_rotator(0.5, 0.1, True)
    ode = {"rot_uni": O.ode_unimodal(om), "rot_taylor": O.ode_rotator_taylor(0.5, 0.1),
           "burgers": O.ode_burgers(math.sqrt(0.2))}[name]
    x0 = O.sample_normal_initial(21, 2.5, 0.04, 1000)
    tr = O.run_micro_macro(om, ode, x0, 6, 3, 25 * 2.0 ** -8, 2.0 ** -8, 25, 21, integ=O.Euler(2.0 ** -6))
    assert np.array_equal(tr.macro, g[f"run_{name}_macro"])
    assert np.array_equal(tr.micro, g[f"run_{name}_micro"])
    assert np.array_equal(np.array([[e for e in row] for row in tr.snapshots]), g[f"run_{name}_snap"])
