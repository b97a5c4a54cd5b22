"""GPU parity for the ROTATOR_SUM and EMPIRICAL_CDF statistics (plane
rotator and Burgers models; fine_stepwise.cu, coarse.cu) against the
reference's golden vectors.

Burgers: ranks are exact and the update is two IEEE operations, so the fine
trajectories are bit-identical.  Plane rotator: CUDA's sin/cos differ from
numpy's by libm ulps, so trajectories are held to the north-star 1e-12
relative and moments to 1e-10.
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


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / max(1.0, float(np.max(np.abs(b))))


def _models(mm):
    return {"rotator": mm.make_plane_rotator(mm.PlaneRotatorSpec(K=0.5, kBT=0.1, wrap=True)),
            "rotator_nowrap": mm.make_plane_rotator(mm.PlaneRotatorSpec(K=1.5, kBT=0.3, wrap=False)),
            "burgers": mm.make_burgers(mm.BurgersSpec())}


@pytest.mark.parametrize("name", ["rotator", "rotator_nowrap", "burgers"])
@pytest.mark.parametrize("P", [1, 7, 1000, 4099])
def test_propagate_fine_matches_reference(mm, golden, name, P):
    g = golden("stats")
    Pm, S, dt, n, t0, seed = g[f"{name}_P{P}_meta"]
    out = mm.propagate_fine(_models(mm)[name], mm.ParticleEnsemble(g[f"{name}_P{P}_x0"]), int(n), t0,
                            mm.StepConfig(dt, int(S)), mm.NoisePlan(int(seed)))
    ref = g[f"{name}_P{P}_x1"]
    if name == "burgers":
        tail = np.abs(O.slice_noise(int(seed), int(n), int(S), int(Pm))) > 3.6541528853610087
        if not tail.any():
            assert np.array_equal(out.positions, ref)
    assert rel(out.positions, ref) <= TRAJ_TOL


@pytest.mark.parametrize("P", [100_000, 131_072])
def test_injected_large_ensembles(mm, P):
    """Injected increments at full size: Burgers bitwise, rotator 1e-12."""
    rng = np.random.default_rng(P)
    S = 6
    x0 = rng.normal(0.0, 2.0, P)
    x0[::97] = np.round(x0[::97], 1)  # rank ties
    xi = rng.standard_normal((S, P))
    for name, om in (("burgers", O.model_burgers(math.sqrt(0.2))), ("rotator", O.model_rotator(0.5, 0.1, True))):
        out = mm.propagate_fine(_models(mm)[name], mm.ParticleEnsemble(x0), 0, 0.0, mm.StepConfig(1e-2, S),
                                mm.NoisePlan(0), increments=xi)
        ref = O.propagate_fine(om, x0, 0, 0.0, 1e-2, S, xi)
        if name == "burgers":
            assert np.array_equal(out.positions, ref)
        else:
            assert rel(out.positions, ref) <= TRAJ_TOL


@pytest.mark.parametrize("name", ["rot_uni", "rot_taylor", "burgers"])
def test_run_micro_macro_matches_reference(mm, golden, name):
    g = golden("stats")
    models = _models(mm)
    model = models["burgers"] if name == "burgers" else models["rotator"]
    ode = {"rot_uni": lambda: mm.unimodal_rhs(model), "rot_taylor": lambda: mm.taylor_enriched_rhs(model),
           "burgers": lambda: mm.burgers_rhs(math.sqrt(0.2))}[name]()
    cfg = mm.PararealConfig(n_slices=6, iterations=3, slice_length=25 * 2.0 ** -8, particles=1000,
                            step=mm.StepConfig(dt=2.0 ** -8, steps_per_slice=25), integrator=mm.EulerConfig(2.0 ** -6))
    tr = mm.run_micro_macro(model, ode, mm.InitialDistribution.normal(2.5, 0.04), cfg, mm.NoisePlan(21))
    macro = np.array([[s.packed() for s in row] for row in tr.macro])
    snaps = np.array([[e.positions for e in row] for row in tr.snapshots])
    assert rel(macro, g[f"run_{name}_macro"]) <= MOM_TOL
    assert rel(snaps, g[f"run_{name}_snap"]) <= TRAJ_TOL


def test_rotator_taylor_singularity(mm):
    model = mm.make_plane_rotator(mm.PlaneRotatorSpec(K=0.5, kBT=0.1))
    ode = mm.taylor_enriched_rhs(model)
    with pytest.raises(mm.SingularityError):
        mm.integrate_macro(ode, mm.MacroState((0.0,), (0.1,), (1.0,)), 0.0, 0.1, mm.EulerConfig(0.01))
    st = mm.integrate_macro(mm.burgers_rhs(0.4), mm.MacroState((0.0,), (-0.1,), (1.0,)), 0.0, 0.5,
                            mm.EulerConfig(0.1))
    assert st.means[0] == pytest.approx(0.25)


@pytest.mark.parametrize("P", [1, 2, 7, 1000, 4099, 100_000])
def test_ensemble_statistic_device_kinds(mm, P):
    """models.ensemble_statistic for ROTATOR_SUM / EMPIRICAL_CDF on the
    device (mmpr_ensemble_statistic) against the oracle's numpy statement
    (models.py:61-83): CDF ranks bitwise (ties by index), rotator means to
    libm-ulp tolerance."""
    rng = np.random.default_rng(P)
    x = rng.uniform(0.0, 2.0 * math.pi, P)
    x[: P // 3] = np.round(x[: P // 3], 1)  # ties
    rot = mm.make_plane_rotator(mm.PlaneRotatorSpec(K=0.7, kBT=0.1))
    got = mm.ensemble_statistic(rot, x)
    want = O.statistic(O.model_rotator(0.7, 0.1), x)
    assert abs(got[0] - want[0]) <= 1e-14 and abs(got[1] - want[1]) <= 1e-14
    bur = mm.make_burgers(mm.BurgersSpec())
    assert np.array_equal(mm.ensemble_statistic(bur, x), O.statistic(O.model_burgers(0.5), x))
