"""Generate golden vectors from the UNMODIFIED reference (run in the build
container only; /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is produced by the reference's own public API
(mcparareal.*, /root/reference/pkg/src/mcparareal).  Where a BASELINE config
needs a piece the reference does not ship, the piece is plugged into the
reference engine through its own extension points and labelled here:
  * forward-Euler coarse: engine.integrate_macro is replaced by a fixed-step
    Euler over the reference's MomentODE.rhs / pack_state / unpack_state;
  * cubic mean-field model (config 2), double-well with multiplicative noise
    (config 5): McKeanVlasovModel dataclasses with numpy closures, plus a
    Gaussian-closure MomentODE for config 2.
Sizes are reduced from the BASELINE configs (P, N) so fixtures stay small;
full-size parity is checked on the GPU through size-independent properties.
"""

from __future__ import annotations

import math
import os
import sys
from contextlib import contextmanager

import numpy as np

import mcparareal as ref
from mcparareal import engine as ref_engine
from mcparareal.moments import pack_state, unpack_state

OUT = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# builder pieces plugged into the reference
# ---------------------------------------------------------------------------
def euler_integrate_macro(dt):
    def integrate_macro(ode, state, t0, t1, cfg=None):
        y = pack_state(state)
        span = t1 - t0
        if span == 0:
            return unpack_state(y, ode.n_regions)
        n = max(1, int(round(span / dt)))
        h = span / n
        for i in range(n):
            y = y + h * ode.rhs(t0 + i * h, y)
        return unpack_state(y, ode.n_regions)
    return integrate_macro


@contextmanager
def euler_coarse(dt):
    saved = ref_engine.integrate_macro
    ref_engine.integrate_macro = euler_integrate_macro(dt)
    try:
        yield
    finally:
        ref_engine.integrate_macro = saved


def make_cubic(c1, c3, cE, sigma):
    return ref.McKeanVlasovModel(
        name="cubic-meanfield",
        drift=lambda x, s, t: cE * s - c1 * x - c3 * (x * x * x),
        diffusion=lambda x, s, t: np.full_like(np.asarray(x, float), sigma),
        drift_dx=lambda x, s, t: -c1 - 3.0 * c3 * (x * x),
        diffusion_dx=lambda x, s, t: np.zeros_like(np.asarray(x, float)),
        diffusion_dxx=lambda x, s, t: np.zeros_like(np.asarray(x, float)),
        statistic_kind=ref.StatisticKind.MEAN_OF_F)


def gaussian_cubic_ode(c1, c3, cE, sigma):
    def rhs(t, y):
        m, v, _ = y
        dm = cE * m - c1 * m - c3 * (m * m * m + 3.0 * m * v)
        dv = -2.0 * c1 * v - 6.0 * c3 * v * (m * m + v) + sigma * sigma
        return np.array([dm, dv, 0.0])
    return ref.MomentODE(rhs, 1, "gaussian-closure")


def make_dw_mult(spec, s0):
    base = ref.make_double_well(spec)
    return ref.McKeanVlasovModel(
        name="double-well-multiplicative",
        drift=base.drift,
        diffusion=lambda x, s, t: s0 * np.sqrt(1.0 + x * x),
        drift_dx=base.drift_dx,
        diffusion_dx=lambda x, s, t: s0 * x / np.sqrt(1.0 + x * x),
        diffusion_dxx=lambda x, s, t: s0 / ((1.0 + x * x) * np.sqrt(1.0 + x * x)),
        statistic_kind=ref.StatisticKind.MEAN_OF_F)


def bimodal_sampler(rng, count):
    """0.5 N(-1, 0.2^2) + 0.5 N(1, 0.2^2) (BASELINE configs 3 and 5)."""
    signs = np.where(rng.random(count) < 0.5, -1.0, 1.0)
    return signs + 0.2 * rng.standard_normal(count)


# ---------------------------------------------------------------------------
# fixtures
# ---------------------------------------------------------------------------
def noise_fixture():
    out = {}
    cases = [(0, "frozen", 0, 0, 1000, 0), (0, "frozen", 3, 17, 1000, 5), (20240601, "frozen", 9, 99, 5000, 0),
             (7, "fresh", 2, 3, 1000, 4), (2 ** 40 + 5, "frozen", 1, 1, 257, 0)]
    for c, (seed, mode, n, j, P, k) in enumerate(cases):
        out[f"case{c}_meta"] = np.array([seed, 1 if mode == "fresh" else 0, n, j, P, k], dtype=np.uint64)
        out[f"case{c}_normals"] = ref.NoisePlan(seed, mode).normals(n, j, P, k)
    for c, (seed, mean, var, P) in enumerate([(0, 1.0, 0.01, 1000), (5, 0.5, 0.04, 333)]):
        plan = ref.NoisePlan(seed)
        out[f"init{c}_meta"] = np.array([seed, mean, var, P])
        out[f"init{c}"] = ref.sample_initial(ref.InitialDistribution.normal(mean, var), plan, P).positions
    return out


MODELS = {
    "ou": (lambda: ref.make_perturbed_ou(ref.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)), (1, (-1.0, 0.5, 0.5))),
    "ou_default": (lambda: ref.make_perturbed_ou(ref.PerturbedOUSpec()), (1, (-1.0, -0.5, 0.01))),
    "linear": (lambda: ref.make_linear(ref.LinearMcKVSpec(A=-0.7, A_E=0.3, A_0=0.1, B=0.2, B_E=0.05, B_0=0.4)),
               (2, (-0.7, 0.3, 0.1, 0.2, 0.05, 0.4))),
    "double_well": (lambda: ref.make_double_well(ref.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0,
                                                                     sigma=0.5)), None),
    "double_well_tilt": (lambda: ref.make_double_well(ref.DoubleWellSpec(alpha=0.25, gamma=0.5, beta=0.3, J=0.2,
                                                                          sigma=0.7)), None),
    "cubic": (lambda: make_cubic(1.0, 1.0, 1.0, 0.4), None),
    "dw_mult": (lambda: make_dw_mult(ref.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0), 0.3), None),
}


def fine_fixture():
    out = {}
    for name, (factory, _) in MODELS.items():
        model = factory()
        for P, S, dt, n, t0 in [(1, 4, 1e-2, 0, 0.0), (5, 6, 1e-2, 2, 0.5), (1000, 20, 1e-3, 3, 0.3),
                                (1001, 17, 2.0 ** -10, 1, 0.0)]:
            plan = ref.NoisePlan(11)
            x0 = ref.sample_initial(ref.InitialDistribution.normal(0.3, 0.5), plan, P)
            cfg = ref.StepConfig(dt=dt, steps_per_slice=S)
            x1 = ref.propagate_fine(model, x0, n, t0, cfg, plan)
            key = f"{name}_P{P}"
            out[key + "_meta"] = np.array([P, S, dt, n, t0, 11.0])
            out[key + "_x0"] = x0.positions
            out[key + "_x1"] = x1.positions
    # em_step known answers (test_particles.py:103-116)
    out["em_zero_noise"] = ref.em_step(ref.make_perturbed_ou(ref.PerturbedOUSpec()), ref.ParticleEnsemble([100.0]),
                                       0.0, 0.01, np.zeros(1)).positions
    out["em_sqrt_dt"] = ref.em_step(ref.make_perturbed_ou(ref.PerturbedOUSpec(a=0.0, a_E=0.0, B=2.0)),
                                    ref.ParticleEnsemble([1.0]), 0.0, 0.25, np.array([3.0])).positions
    return out


def coupling_fixture():
    out = {}
    rng = np.random.default_rng(5)
    parts = {"single": ref.RegionPartition(),
             "two": ref.RegionPartition(separatrices=(0.0,), peaks=(-1.5, 1.5)),
             "three": ref.RegionPartition(separatrices=(0.0, 2.0), peaks=(-1.0, 1.0, 3.0))}
    ens = {
        "frozen4": np.array([-2.0, -1.0, 1.0, 2.0]),
        "empty_left": np.array([1.0, 2.0, 3.0]),
        "single_left": np.array([-0.5, 1.0, 3.0]),
        "boundary": np.array([0.0, -1.0]),
        "ties": np.array([0.4, 0.4, 0.4, 0.4, 0.4]),
        "hyp_fail": np.array([0.0, 0.4, 0.4, 0.4, 0.125]),
        "rand100": rng.normal(0.0, 2.0, 100),
        "rand1000": rng.normal(0.3, 1.5, 1000),
        "rand4097": rng.normal(-0.2, 1.0, 4097),
        "bimodal": bimodal_sampler(rng, 3000),
    }
    for pn, part in parts.items():
        for en, x in ens.items():
            st = ref.restrict(ref.ParticleEnsemble(x), part)
            key = f"restrict_{pn}_{en}"
            out[key] = np.array(st.means + st.variances + st.fractions)
            out[key + "_deg"] = np.array(st.degenerate)
    out["ens_names"] = np.array(list(ens.keys()))
    for en, x in ens.items():
        out[f"ens_{en}"] = x
    # match cases: (partition, ensemble, target, policy)
    cases = [
        ("single", "frozen4", (3.0,), (4.0,), "raise"),
        ("two", "frozen4", (-1.2, 1.7), (0.09, 0.16), "raise"),
        ("single", "rand100", (5.0,), (0.25,), "raise"),
        ("single", "ties", (5.0,), (1.0,), "collapse"),
        ("single", "ties", (5.0,), (0.0,), "raise"),
        ("two", "empty_left", (-1.0, 2.5), (1.0, 0.5), "raise"),
        ("single", "rand1000", (2.0,), (-0.5,), "raise"),
        ("three", "rand4097", (-1.0, 1.0, 3.0), (0.2, 0.1, 0.3), "raise"),
        ("two", "bimodal", (-0.9, 1.1), (0.05, 0.02), "raise"),
        ("two", "hyp_fail", (-0.25 + 0.0, 0.75), (0.01, 0.01), "raise"),
    ]
    hyp_part = ref.RegionPartition(separatrices=(0.25,), peaks=(-0.75, 1.25))
    for c, (pn, en, mu, var, policy) in enumerate(cases):
        part = hyp_part if en == "hyp_fail" else parts[pn]
        n = part.n_regions
        target = ref.MacroState(mu, var, (1.0 / n,) * n)
        try:
            res = ref.match(target, ref.ParticleEnsemble(ens[en]), part, policy).positions
            status = -1
        except ref.DegenerateMatch as err:
            res = np.array([])
            status = err.region
        out[f"match{c}_meta"] = np.array([list(parts).index(pn) if en != "hyp_fail" else 3,
                                          list(ens).index(en), 1 if policy == "collapse" else 0, status])
        out[f"match{c}_target"] = np.array(mu + var)
        out[f"match{c}_out"] = res
    out["hyp_part"] = np.array([0.25, -0.75, 1.25])
    return out


def trace_to_arrays(trace, prefix, out, snapshots=True):
    K = trace.iterations
    N = trace.n_slices
    pack = lambda st: np.array(st.means + st.variances + st.fractions)  # noqa: E731
    out[prefix + "macro"] = np.array([[pack(trace.macro[k][n]) for n in range(N + 1)] for k in range(K + 1)])
    out[prefix + "micro"] = np.array([[pack(trace.micro_stats[k][n]) for n in range(N + 1)]
                                      for k in range(K + 1)])
    if snapshots:
        out[prefix + "snap"] = np.array([[trace.snapshots[k][n].positions for n in range(N + 1)]
                                         for k in range(K + 1)])
    out[prefix + "clamp"] = np.array(trace.clamp_events, dtype=float).reshape(-1, 4)
    out[prefix + "gaps"] = np.array(trace.fraction_gaps, dtype=float).reshape(-1, 3)
    out[prefix + "lift"] = np.array(trace.lift_collapses, dtype=float).reshape(-1, 3)


def trace_fixture():
    out = {}
    # E1: config-1 shape (P reduced), Euler coarse on unimodal_rhs
    spec = ref.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
    model = ref.make_perturbed_ou(spec)
    cfg = ref.PararealConfig(n_slices=10, iterations=5, slice_length=0.1, particles=1000,
                             step=ref.StepConfig(dt=1e-3, steps_per_slice=100))
    plan = ref.NoisePlan(0)
    initial = ref.InitialDistribution.normal(1.0, 0.01)
    with euler_coarse(1e-2):
        tr = ref.run_micro_macro(model, ref.unimodal_rhs(model), initial, cfg, plan)
    trace_to_arrays(tr, "c1_", out)
    out["c1_seq"] = np.array([e.positions for e in ref.sequential_fine(model, initial, cfg, plan)])

    # E2: reference default DP5(4) coarse (no builder pieces at all)
    spec2 = ref.PerturbedOUSpec(B=1.0)
    model2 = ref.make_perturbed_ou(spec2)
    cfg2 = ref.PararealConfig(n_slices=6, iterations=4, slice_length=0.25, particles=500,
                              step=ref.StepConfig(dt=0.05, steps_per_slice=5))
    tr2 = ref.run_micro_macro(model2, ref.perturbed_ou_rhs(spec2), ref.InitialDistribution.normal(1.0, 0.5), cfg2,
                              ref.NoisePlan(77))
    trace_to_arrays(tr2, "dp_", out)
    tr2u = ref.run_micro_macro(model2, ref.unimodal_rhs(model2), ref.InitialDistribution.normal(1.0, 0.5), cfg2,
                               ref.NoisePlan(78))
    trace_to_arrays(tr2u, "dpu_", out)

    # E3: config-3 shape: bimodal double well, two regions, multimodal coarse + Euler
    dw = ref.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    m3 = ref.make_double_well(dw)
    part3 = dw.default_partition()
    ode3 = ref.multimodal_rhs(m3, part3, dw.potential, dw.sigma)
    cfg3 = ref.PararealConfig(n_slices=8, iterations=4, slice_length=0.0625, particles=1000,
                              step=ref.StepConfig(dt=2.0 ** -10, steps_per_slice=64), partition=part3)
    init3 = ref.InitialDistribution.custom(bimodal_sampler, 0.0, 1.04)
    with euler_coarse(2.0 ** -6):
        tr3 = ref.run_micro_macro(m3, ode3, init3, cfg3, ref.NoisePlan(0))
    trace_to_arrays(tr3, "c3_", out)
    out["c3_part"] = np.array([part3.separatrices[0], part3.peaks[0], part3.peaks[1]])
    out["c3_seq"] = np.array([e.positions for e in ref.sequential_fine(m3, init3, cfg3, ref.NoisePlan(0))])

    # E4: config-2 shape: cubic mean field + Gaussian closure + Euler
    m4 = make_cubic(1.0, 1.0, 1.0, 0.4)
    cfg4 = ref.PararealConfig(n_slices=8, iterations=4, slice_length=0.0625, particles=1000,
                              step=ref.StepConfig(dt=2.0 ** -10, steps_per_slice=64))
    with euler_coarse(2.0 ** -6):
        tr4 = ref.run_micro_macro(m4, gaussian_cubic_ode(1.0, 1.0, 1.0, 0.4),
                                  ref.InitialDistribution.normal(0.5, 0.04), cfg4, ref.NoisePlan(0))
    trace_to_arrays(tr4, "c2_", out)

    # E5: config-5 shape: multiplicative noise double well, two regions
    dw5 = ref.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.3 * math.sqrt(1.8))
    m5 = make_dw_mult(dw5, 0.3)
    part5 = dw5.default_partition()
    ode5 = ref.multimodal_rhs(m5, part5, dw5.potential, dw5.sigma)
    cfg5 = ref.PararealConfig(n_slices=4, iterations=3, slice_length=0.1, particles=1000,
                              step=ref.StepConfig(dt=5e-4, steps_per_slice=200), partition=part5)
    with euler_coarse(1e-2):
        tr5 = ref.run_micro_macro(m5, ode5, init3, cfg5, ref.NoisePlan(0))
    trace_to_arrays(tr5, "c5_", out)
    return out


def stats_fixture():
    """ROTATOR_SUM and EMPIRICAL_CDF models: propagate_fine and the
    statistics themselves, from the reference factories."""
    out = {}
    models = {"rotator": ref.make_plane_rotator(ref.PlaneRotatorSpec(K=0.5, kBT=0.1, wrap=True)),
              "rotator_nowrap": ref.make_plane_rotator(ref.PlaneRotatorSpec(K=1.5, kBT=0.3, wrap=False)),
              "burgers": ref.make_burgers(ref.BurgersSpec())}
    for name, model in models.items():
        for P, S, dt, n, t0 in [(1, 4, 1e-2, 0, 0.0), (7, 5, 1e-2, 2, 0.5), (1000, 20, 1e-3, 3, 0.3),
                                (4099, 12, 2.0 ** -8, 1, 0.0)]:
            plan = ref.NoisePlan(13)
            x0 = ref.sample_initial(ref.InitialDistribution.normal(3.0, 1.5), plan, P)
            x1 = ref.propagate_fine(model, x0, n, t0, ref.StepConfig(dt=dt, steps_per_slice=S), plan)
            key = f"{name}_P{P}"
            out[key + "_meta"] = np.array([P, S, dt, n, t0, 13.0])
            out[key + "_x0"] = x0.positions
            out[key + "_x1"] = x1.positions
    # full mM runs (Euler coarse plugged in as for the BASELINE configs)
    runs = {"rot_uni": (models["rotator"], ref.unimodal_rhs(models["rotator"])),
            "rot_taylor": (models["rotator"], ref.taylor_enriched_rhs(models["rotator"])),
            "burgers": (models["burgers"], ref.burgers_rhs(math.sqrt(0.2)))}
    for name, (model, ode) in runs.items():
        cfg = ref.PararealConfig(n_slices=6, iterations=3, slice_length=25 * 2.0 ** -8, particles=1000,
                                 step=ref.StepConfig(dt=2.0 ** -8, steps_per_slice=25))
        init = ref.InitialDistribution.normal(2.5, 0.04)
        with euler_coarse(2.0 ** -6):
            tr = ref.run_micro_macro(model, ode, init, cfg, ref.NoisePlan(21))
        trace_to_arrays(tr, f"run_{name}_", out)
    # statistics with ties and signed zeros (ranks are stable by index)
    x = np.array([0.5, -0.0, 0.0, 0.5, -1.0, 0.0, 2.0, 0.5, -0.0])
    out["cdf_x"] = x
    out["cdf_s"] = ref.ensemble_statistic(models["burgers"], x)
    out["rot_s"] = np.array(ref.ensemble_statistic(models["rotator"], x))
    return out


def report_to_arrays(rep, prefix, out):
    out[prefix + "scalars"] = np.array([rep.e_mean, rep.e_var, rep.e_wass, rep.normalized_mean, rep.normalized_var,
                                        rep.normalized_wass])
    out[prefix + "per_slice"] = np.array([rep.mean_err_per_slice, rep.var_err_per_slice, rep.wass_per_slice])


def metrics_fixture():
    """mcparareal.metrics on reference traces and serial fine replicas."""
    from mcparareal import metrics as M
    out = {}
    spec = ref.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
    model = ref.make_perturbed_ou(spec)
    cfg = ref.PararealConfig(n_slices=10, iterations=5, slice_length=0.1, particles=1000,
                             step=ref.StepConfig(dt=1e-3, steps_per_slice=100))
    initial = ref.InitialDistribution.normal(1.0, 0.01)
    with euler_coarse(1e-2):
        tr = ref.run_micro_macro(model, ref.unimodal_rhs(model), initial, cfg, ref.NoisePlan(0))
    for k in range(tr.iterations + 1):
        report_to_arrays(M.relative_errors(tr, k), f"rel_c1_k{k}_", out)
        report_to_arrays(M.relative_errors(tr, k, var_denominator="mean"), f"relm_c1_k{k}_", out)
    report_to_arrays(M.relative_errors(tr, 1, reference_k=3), "rel_c1_k1_ref3_", out)
    # histogram artefacts (harness.py:300-323): FD edges on the final iterate
    from mcparareal import harness as H
    for n in (1, 5, 10):
        data = [tr.snapshots[k][n].positions for k in range(tr.iterations + 1)]
        reference = tr.snapshots[tr.iterations][n].positions
        edges = H._fd_edges(reference, data + [reference])
        out[f"hist_c1_n{n}_edges"] = edges
        out[f"hist_c1_n{n}_counts"] = np.array([np.histogram(d, edges)[0] for d in data])
    # floor replicas exactly as harness.replicate_seeds derives them (harness.py:158-165)
    base = ref.NoisePlan(0)
    seeds = [base.derived_seed(10_000 + j) for j in range(3)]
    out["floor_seeds"] = np.array(seeds, dtype=np.uint64)
    paths = [ref.sequential_fine(model, initial, cfg, ref.NoisePlan(s)) for s in seeds]
    for vd in ("variance", "mean"):
        fl = M.floor_from_references(paths, vd)
        out[f"floor_{vd}"] = np.array([fl.e_mean, fl.e_var, fl.e_wass, fl.n_replicas])
    finals = [p[-1] for p in paths]
    out["floor_raw"] = np.array([M.statistical_floor(finals)])
    out["floor_spread"] = np.array(M.moment_spread(finals))
    out["floor_final_positions"] = np.array([f.positions for f in finals])
    # W1 examples: ties, signed zeros, different scales
    rng = np.random.default_rng(5)
    a = np.round(rng.normal(0.0, 1.0, 3001), 1)
    b = np.round(rng.normal(0.2, 1.5, 3001), 1)
    a[:5] = [0.0, -0.0, 0.0, -0.0, 1.0]
    out["w1_a"], out["w1_b"] = a, b
    out["w1_ab"] = np.array([M.wasserstein_1d(a, b), M.wasserstein_1d(b, a), M.wasserstein_1d(a, a)])
    return out


def main():
    np.savez_compressed(os.path.join(OUT, "noise.npz"), **noise_fixture())
    np.savez_compressed(os.path.join(OUT, "fine.npz"), **fine_fixture())
    np.savez_compressed(os.path.join(OUT, "coupling.npz"), **coupling_fixture())
    np.savez_compressed(os.path.join(OUT, "traces.npz"), **trace_fixture())
    np.savez_compressed(os.path.join(OUT, "metrics.npz"), **metrics_fixture())
    np.savez_compressed(os.path.join(OUT, "stats.npz"), **stats_fixture())
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] in ("metrics", "stats"):
        fixture = {"metrics": metrics_fixture, "stats": stats_fixture}[sys.argv[1]]
        np.savez_compressed(os.path.join(OUT, sys.argv[1] + ".npz"), **fixture())
    else:
        sys.exit(main())
