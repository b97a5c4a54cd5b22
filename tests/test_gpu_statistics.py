"""Statistical properties the reference's own tests check (test_particles.py
EM mean / variance-bias tests, test_acceptance.py criteria 2 and 10),
restated for the device path."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import paper_2310_11365_b200 as mm
    mm._lib.load()
    return mm


def test_em_mean_follows_linear_recursion(mm):
    """a + a_E linear in x and the mean: the ensemble mean obeys
    m_{j+1} = (1 + (a + a_E) dt) m_j up to noise (within 6 SE)."""
    spec = mm.PerturbedOUSpec(a=-1.0, a_E=-0.5, B=0.01)
    model = mm.make_perturbed_ou(spec)
    plan = mm.NoisePlan(314)
    dt, steps, count = 0.01, 100, 10_000
    ens = mm.sample_initial(mm.InitialDistribution.dirac(100.0), plan, count)
    out = mm.propagate_fine(model, ens, 0, 0.0, mm.StepConfig(dt, steps), plan)
    expected = 100.0 * (1.0 + (spec.a + spec.a_E) * dt) ** steps
    se = spec.B / math.sqrt(2.0) / math.sqrt(count)
    assert abs(mm.empirical_mean(out) - expected) <= 6 * se


def test_em_variance_bias_first_order(mm):
    """Plain OU: the EM stationary-variance bias halves with dt (common
    random numbers: coarse increments are pairwise sums of fine ones)."""
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.0, B=1.0))
    plan = mm.NoisePlan(2718)
    count, t_end, dt_c = 100_000, 3.0, 0.2
    steps_c = round(t_end / dt_c)
    ens0 = mm.sample_initial(mm.InitialDistribution.normal(0.0, 0.5), plan, count)
    fine = ens0
    for j in range(2 * steps_c):
        fine = mm.em_step(model, fine, j * dt_c / 2, dt_c / 2, plan.normals(0, j, count))
    coarse = ens0
    for j in range(steps_c):
        agg = (plan.normals(0, 2 * j, count) + plan.normals(0, 2 * j + 1, count)) / math.sqrt(2.0)
        coarse = mm.em_step(model, coarse, j * dt_c, dt_c, agg)
    b_c = mm.empirical_variance(coarse) - 0.5
    b_f = mm.empirical_variance(fine) - 0.5
    assert b_c > 0 and b_f > 0
    assert 1.0 <= b_c / b_f <= 4.0


def test_monte_carlo_moments_match_exact_ou_flow(mm):
    """100 seeded ensembles of 1e5 particles over T = 1: mean and variance
    within 4 standard errors of the closed-form OU moments in >= 95 cases."""
    a, a_E, B, m0, v0, T = -1.0, -0.5, 1.0, 1.0, 0.5, 1.0
    model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=a, a_E=a_E, B=B))
    dist = mm.InitialDistribution.normal(m0, v0)
    exact_mean = m0 * math.exp((a + a_E) * T)
    exact_var = v0 * math.exp(2 * a * T) + B * B / (-2 * a) * (1.0 - math.exp(2 * a * T))
    P, hits = 100_000, 0
    for rep in range(100):
        plan = mm.NoisePlan(7_000 + rep)
        ens = mm.propagate_fine(model, mm.sample_initial(dist, plan, P), 0, 0.0, mm.StepConfig(0.01, 100), plan)
        st = mm.restrict(ens)
        m, v = st.means[0], st.variances[0]
        if abs(m - exact_mean) <= 4 * math.sqrt(v / P) and abs(v - exact_var) <= 4 * v * math.sqrt(2.0 / (P - 1)):
            hits += 1
    assert hits >= 95


def test_byte_identical_reruns(mm):
    """Identical bytes across reruns (eager, first graph capture, replay)."""
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.1, sigma=0.5)
    model = mm.make_double_well(dw)
    part = dw.default_partition()
    ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
    cfg = mm.PararealConfig(n_slices=5, iterations=3, slice_length=0.0625, particles=500,
                            step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6))
    outs = []
    for use_graph in (False, True, True):
        tr = mm.run_micro_macro(model, ode, mm.bimodal_initial(-1.0, 1.0, 0.2), cfg, mm.NoisePlan(10),
                                use_graph=use_graph)
        outs.append(np.array([[e.positions for e in row] for row in tr.snapshots]).tobytes()
                    + np.array([[s.packed() for s in row] for row in tr.macro]).tobytes())
    assert outs[0] == outs[1] == outs[2]
