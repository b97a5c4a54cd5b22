"""Moment-ODE coarse propagators (drop-in for mcparareal.moments,
/root/reference/pkg/src/mcparareal/moments.py).

Each factory returns a ``MomentODE`` with the reference's packed-vector
``rhs`` callable (host, for direct use) and a POD ``descriptor`` evaluated by
the device integrators (coarse.cu) with the same operation order.
``integrate_macro`` runs on the GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib, kernels
from ._device import device, torch
from .errors import IntegrationFailure, McPararealError, SingularityError
from .models import (McKeanVlasovModel, PerturbedOUSpec, StatisticKind, device_model, mixture_statistic,
                     point_statistic)
from .rk54 import EulerConfig, IntegratorConfig, integrator_descriptor
from .state import MacroState, RegionPartition

SQRT_2PI = math.sqrt(2.0 * math.pi)


@dataclass(frozen=True)
class MomentODE:
    rhs: Callable
    n_regions: int
    variant: str
    has_fraction_dynamics: bool = False
    descriptor: _lib.MomentOde | None = None
    model: McKeanVlasovModel | None = None


def pack_state(state: MacroState) -> np.ndarray:
    return np.array(state.means + state.variances + state.fractions, dtype=float)


def unpack_state(y, n_regions: int) -> MacroState:
    y = np.asarray(y, dtype=float)
    if y.shape != (3 * n_regions,):
        raise ValueError(f"expected packed vector of length {3 * n_regions}")
    return MacroState(tuple(y[:n_regions]), tuple(y[n_regions:2 * n_regions]), tuple(y[2 * n_regions:]))


def _ode(kind: int, n: int, params=()) -> _lib.MomentOde:
    d = _lib.MomentOde()
    d.kind = kind
    d.n_regions = n
    for i, v in enumerate(params):
        d.p[i] = float(v)
    return d


def device_ode(ode: MomentODE):
    """(ode descriptor, model descriptor) or TypeError."""
    if ode.descriptor is None:
        raise TypeError(f"moment model {ode.variant!r} has no device descriptor (no CPU fallback)")
    if ode.model is not None:
        return ode.descriptor, device_model(ode.model)
    return ode.descriptor, _lib.Model()


def unimodal_rhs(model: McKeanVlasovModel) -> MomentODE:
    """First-order closure dM = a + b_xx/2, dS = (2a_x + b_x^2) S + b^2."""
    if model.statistic_kind is StatisticKind.EMPIRICAL_CDF:
        raise ValueError("rank-interaction models need their dedicated moment model (burgers_rhs); "
                         "the point-mass closure loses the variance dynamics")

    def rhs(t, y):
        m, var, _ = y
        s = point_statistic(model, m)
        d_mean = float(model.drift(m, s, t)) + 0.5 * float(model.diffusion_dxx(m, s, t))
        b = float(model.diffusion(m, s, t))
        b_x = float(model.diffusion_dx(m, s, t))
        d_var = (2.0 * float(model.drift_dx(m, s, t)) + b_x * b_x) * var + b * b
        return np.array([d_mean, d_var, 0.0])

    desc = _ode(_lib.ODE_UNIMODAL, 1) if getattr(model, "descriptor", None) is not None else None
    return MomentODE(rhs, 1, "first-order", descriptor=desc, model=model)


def perturbed_ou_rhs(spec: PerturbedOUSpec) -> MomentODE:
    mean_rate = (spec.a + spec.a_E) * (1.0 + spec.eps_mean)
    var_rate = 2.0 * spec.a * (1.0 + spec.eps_mean)
    var_source = spec.B ** 2 * (1.0 + spec.eps_var) ** 2

    def rhs(t, y):
        m, var, _ = y
        return np.array([mean_rate * m, var_rate * var + var_source, 0.0])

    return MomentODE(rhs, 1, "perturbed-ou",
                     descriptor=_ode(_lib.ODE_PERTURBED_OU, 1, (mean_rate, var_rate, var_source)))


def gaussian_closure_rhs(spec) -> MomentODE:
    """Gaussian moment closure of the cubic mean-field model (BASELINE config 2):
    dM = cE M - c1 M - c3 (M^3 + 3 M S), dS = -2 c1 S - 6 c3 S (M^2 + S) + sigma^2."""
    c1, c3, cE, sigma = spec.c1, spec.c3, spec.cE, spec.sigma

    def rhs(t, y):
        m, v, _ = y
        dm = cE * m - c1 * m - c3 * (m * m * m + 3.0 * m * v)
        dv = -2.0 * c1 * v - 6.0 * c3 * v * (m * m + v) + sigma * sigma
        return np.array([dm, dv, 0.0])

    return MomentODE(rhs, 1, "gaussian-closure", descriptor=_ode(_lib.ODE_GAUSSIAN_CUBIC, 1, (c1, c3, cE, sigma)))


def multimodal_rhs(model: McKeanVlasovModel, partition: RegionPartition, potential: Callable, sigma: float,
                   weight_mode: str = "plain") -> MomentODE:
    """Per-region first-order closure with fractions relaxing to potential weights."""
    n = partition.n_regions
    if n < 2:
        raise ValueError("multimodal closure needs at least two regions")
    peaks = np.asarray(partition.peaks, dtype=float)
    if weight_mode == "plain":
        w = np.exp(-np.asarray(potential(peaks), dtype=float))
    elif weight_mode == "gibbs":
        w = np.exp(-np.asarray(potential(peaks), dtype=float) / (2.0 * sigma ** 2))
    else:
        raise ValueError(f"unknown weight mode {weight_mode!r}")
    targets = w / np.sum(w)
    gaps = np.abs(np.diff(peaks))
    dists = np.empty(n)
    dists[0] = gaps[0]
    dists[1:] = gaps
    rates = sigma ** 2 / (2.0 * dists)

    def rhs(t, y):
        means, variances, fractions = y[:n], y[n:2 * n], y[2 * n:]
        s = mixture_statistic(model, means, fractions)
        d_means, d_vars = np.empty(n), np.empty(n)
        for i in range(n):
            m = means[i]
            d_means[i] = float(model.drift(m, s, t)) + 0.5 * float(model.diffusion_dxx(m, s, t))
            b = float(model.diffusion(m, s, t))
            b_x = float(model.diffusion_dx(m, s, t))
            d_vars[i] = (2.0 * float(model.drift_dx(m, s, t)) + b_x * b_x) * variances[i] + b * b
        return np.concatenate([d_means, d_vars, -rates * (fractions - targets)])

    desc = None
    if getattr(model, "descriptor", None) is not None and n <= _lib.MAX_REGIONS:
        desc = _ode(_lib.ODE_MULTIMODAL, n, tuple(targets) + tuple(rates))
    return MomentODE(rhs, n, "multimodal", has_fraction_dynamics=True, descriptor=desc, model=model)


def taylor_enriched_rhs(model: McKeanVlasovModel) -> MomentODE:
    """Variance-enriched single-region closure (moments.py:71-108): the
    model's own closure when it has one (plane rotator: ODE_ROTATOR_TAYLOR),
    else the first-order closure at s = f(M) + (S/2) f''(M) (ODE_TAYLOR)."""
    desc_m = getattr(model, "descriptor", None)
    if model.enriched_moment_rhs is not None:
        custom = model.enriched_moment_rhs

        def rhs(t, y):
            m, var, _ = y
            d_mean, d_var = custom(m, var, t)
            return np.array([float(d_mean), float(d_var), 0.0])

        desc = None
        if desc_m is not None and desc_m.kind == _lib.MODEL_ROTATOR:
            desc = _ode(_lib.ODE_ROTATOR_TAYLOR, 1, (desc_m.p[0], desc_m.p[3]))
        return MomentODE(rhs, 1, "taylor", descriptor=desc)
    if model.statistic_kind is not StatisticKind.MEAN_OF_F:
        raise ValueError(f"model {model.name!r} has no enriched closure and no mean-of-f statistic to enrich")

    def rhs(t, y):
        m, var, _ = y
        f_val = m if model.f is None else float(model.f(m))
        s = f_val + 0.5 * var * (0.0 if model.f_dd is None else float(model.f_dd(m)))
        d_mean = float(model.drift(m, s, t)) + 0.5 * float(model.diffusion_dxx(m, s, t))
        b = float(model.diffusion(m, s, t))
        b_x = float(model.diffusion_dx(m, s, t))
        return np.array([d_mean, (2.0 * float(model.drift_dx(m, s, t)) + b_x * b_x) * var + b * b, 0.0])

    desc = None
    if desc_m is not None and model.f is None and model.f_dd is None:
        desc = _ode(_lib.ODE_TAYLOR, 1)
    return MomentODE(rhs, 1, "taylor", descriptor=desc, model=model if desc is not None else None)


def burgers_rhs(sigma: float) -> MomentODE:
    """Rank-interaction moment model (moments.py:128-142): dM = 1/2,
    dS = -(2/sqrt(2 pi)) sqrt(max(S, 0)) + sigma^2 (device ODE_BURGERS)."""
    sig_sq = float(sigma) ** 2

    def rhs(t, y):
        _, var, _ = y
        return np.array([0.5, -(2.0 / SQRT_2PI) * math.sqrt(max(var, 0.0)) + sig_sq, 0.0])

    return MomentODE(rhs, 1, "first-order", descriptor=_ode(_lib.ODE_BURGERS, 1, (sig_sq, -(2.0 / SQRT_2PI))))


def integrate_macro(ode: MomentODE, state: MacroState, t0: float, t1: float,
                    cfg: IntegratorConfig | EulerConfig = IntegratorConfig()) -> MacroState:
    """Propagate a macro state through the moment ODE over [t0, t1] (GPU)."""
    if state.n_regions != ode.n_regions:
        raise McPararealError(f"macro state has {state.n_regions} regions, moment model expects {ode.n_regions}")
    if t1 < t0:
        raise ValueError("t1 must not precede t0")
    ode_d, model_d = device_ode(ode)
    y = torch.from_numpy(pack_state(state).reshape(1, -1)).to(device())
    out = torch.empty_like(y)
    status = torch.empty(1, dtype=torch.int32, device=device())
    ta = torch.tensor([float(t0)], dtype=torch.float64, device=device())
    tb = torch.tensor([float(t1)], dtype=torch.float64, device=device())
    kernels.integrate_macro(ode_d, model_d, integrator_descriptor(cfg), ta, tb, y, out, status)
    st = int(status.cpu()[0])
    if st == _lib.STAT_SINGULAR:
        raise SingularityError(f"moment closure singular on [{t0}, {t1}]")
    if st != _lib.STAT_OK:
        raise IntegrationFailure(f"coarse integration failed on [{t0}, {t1}]")
    return unpack_state(out.cpu().numpy()[0], ode.n_regions)
