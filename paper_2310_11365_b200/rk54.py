"""Coarse integrator configurations (drop-in for mcparareal.rk54,
/root/reference/pkg/src/mcparareal/rk54.py:41-54).

``IntegratorConfig`` selects the reference's adaptive Dormand-Prince 5(4)
with PI control; ``EulerConfig`` the fixed-step forward Euler the BASELINE
configs ask for ("coarse ... forward Euler dt=..."), with
n = round((t1 - t0)/dt) >= 1 equal steps per slice.  Both run on the device
(coarse.cu); ``descriptor()`` packs them into ``mmpr_integrator``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as _np

from . import _lib
from .errors import IntegrationFailure


@dataclass(frozen=True)
class IntegratorConfig:
    rel_tol: float = 1e-8
    abs_tol: float = 1e-10
    max_steps: int = 100_000
    first_step: float | None = None

    def __post_init__(self):
        if self.rel_tol <= 0 or self.abs_tol <= 0:
            raise ValueError("tolerances must be positive")
        if self.max_steps < 1:
            raise ValueError("max_steps must be at least 1")

    def descriptor(self) -> _lib.Integrator:
        d = _lib.Integrator()
        d.kind = _lib.INTEG_DP54
        d.max_steps = min(int(self.max_steps), 2 ** 31 - 1)
        d.rel_tol = float(self.rel_tol)
        d.abs_tol = float(self.abs_tol)
        d.first_step = float(self.first_step) if self.first_step is not None else 0.0
        return d


@dataclass(frozen=True)
class EulerConfig:
    dt: float

    def __post_init__(self):
        if not self.dt > 0:
            raise ValueError("dt must be positive")

    def descriptor(self) -> _lib.Integrator:
        d = _lib.Integrator()
        d.kind = _lib.INTEG_EULER
        d.dt = float(self.dt)
        d.max_steps = 1
        return d


def integrator_descriptor(cfg) -> _lib.Integrator:
    if not hasattr(cfg, "descriptor"):
        raise TypeError(f"unsupported integrator configuration {cfg!r}")
    return cfg.descriptor()


# ---------------------------------------------------------------------------
# Generic host integrators for user-supplied Python callables
# (drop-in for mcparareal.rk54.integrate / integrate_fixed,
# /root/reference/pkg/src/mcparareal/rk54.py:69-144).
#
# A Python ``rhs(t, y)`` cannot run inside a kernel, so these two stay on the
# host; the engine never calls them (moment models built by the package's
# closures carry a device descriptor and go through coarse.cu, which follows
# the same Dormand-Prince 5(4) / PI-controller recipe).  They exist so code
# written against the reference's ``integrate`` keeps working.
# ---------------------------------------------------------------------------
_DP_NODES = (0.0, 1 / 5, 3 / 10, 4 / 5, 8 / 9, 1.0, 1.0)
# stage rows of the Dormand-Prince tableau; row 6 is also the 5th-order weight row (FSAL)
_DP_ROWS = (
    (),
    (1 / 5,),
    (3 / 40, 9 / 40),
    (44 / 45, -56 / 15, 32 / 9),
    (19372 / 6561, -25360 / 2187, 64448 / 6561, -212 / 729),
    (9017 / 3168, -355 / 33, 46732 / 5247, 49 / 176, -5103 / 18656),
    (35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84),
)
_DP_W5 = _np.array(_DP_ROWS[6] + (0.0,))
_DP_W4 = _np.array((5179 / 57600, 0.0, 7571 / 16695, 393 / 640, -92097 / 339200, 187 / 2100, 1 / 40))
_DP_WERR = _DP_W5 - _DP_W4
_PI_ALPHA, _PI_BETA = 0.7 / 5.0, 0.4 / 5.0
_STEP_SAFETY, _STEP_SHRINK, _STEP_GROW = 0.9, 0.2, 5.0


def _dp_step(rhs, t, y, h, slope0):
    """One Dormand-Prince step from (t, y) with the first stage given:
    (5th-order solution, embedded error vector, last stage)."""
    stages = _np.empty((7,) + y.shape)
    stages[0] = slope0
    for i in range(1, 7):
        row = _DP_ROWS[i]
        incr = row[0] * stages[0] if i == 1 else _np.dot(_np.array(row), stages[:i])
        stages[i] = _np.asarray(rhs(t + _DP_NODES[i] * h, y + h * incr), dtype=float)
    return y + h * (_DP_W5 @ stages), h * (_DP_WERR @ stages), stages[6]


def _rms(v) -> float:
    return float(_np.sqrt(_np.mean(v * v)))


def _first_step(y, slope, cfg) -> float:
    scale = cfg.abs_tol + cfg.rel_tol * _np.abs(y)
    size_y, size_f = _rms(y / scale), _rms(slope / scale)
    return 1e-6 if (size_y < 1e-5 or size_f < 1e-5) else 0.01 * size_y / size_f


def integrate(rhs, y0, t0: float, t1: float, cfg: IntegratorConfig = IntegratorConfig()) -> "_np.ndarray":
    """dy/dt = rhs(t, y) from t0 to t1: adaptive DP5(4), mixed tolerance
    abs_tol + rel_tol * max(|y|, |y_new|), PI step control.  Raises
    IntegrationFailure on a non-finite right-hand side or solution, on step
    underflow, and when ``cfg.max_steps`` attempts are used up."""
    y = _np.array(_np.atleast_1d(_np.asarray(y0, dtype=float)), copy=True)
    if t1 < t0:
        raise ValueError("t1 must not precede t0")
    if t1 == t0:
        return y
    t = t0
    slope = _np.asarray(rhs(t, y), dtype=float)
    if not _np.isfinite(slope).all():
        raise IntegrationFailure(f"right-hand side not finite at t={t0}")
    h = min(cfg.first_step if cfg.first_step is not None else _first_step(y, slope, cfg), t1 - t0)
    h_floor = 1e-14 * max(abs(t0), abs(t1), 1.0)
    last_err = 1.0
    for _ in range(cfg.max_steps):
        h = min(h, t1 - t)
        y_try, err, slope_try = _dp_step(rhs, t, y, h, slope)
        if not _np.isfinite(y_try).all():
            raise IntegrationFailure(f"solution not finite near t={t} with step {h}")
        e = _rms(err / (cfg.abs_tol + cfg.rel_tol * _np.maximum(_np.abs(y), _np.abs(y_try))))
        if e <= 1.0:  # accept; the last stage is the next step's first (FSAL)
            t, y, slope = t + h, y_try, slope_try
            if t >= t1 - h_floor:
                return y
            e = max(e, 1e-10)
            h *= min(_STEP_GROW, max(_STEP_SHRINK, _STEP_SAFETY * e ** (-_PI_ALPHA) * last_err ** _PI_BETA))
            last_err = e
        else:
            h *= min(1.0, max(_STEP_SHRINK, _STEP_SAFETY * e ** (-_PI_ALPHA)))
        if h < h_floor:
            raise IntegrationFailure(f"step size underflow at t={t} (stalled integration)")
    raise IntegrationFailure(f"exceeded {cfg.max_steps} steps integrating [{t0}, {t1}]")


def integrate_fixed(rhs, y0, t0: float, t1: float, n_steps: int) -> "_np.ndarray":
    """n_steps equal Dormand-Prince steps (the 5th-order solution), for order checks."""
    if n_steps < 1:
        raise ValueError("n_steps must be at least 1")
    y = _np.array(_np.atleast_1d(_np.asarray(y0, dtype=float)), copy=True)
    h = (t1 - t0) / n_steps
    for j in range(n_steps):
        t = t0 + j * h
        y, _, _ = _dp_step(rhs, t, y, h, _np.asarray(rhs(t, y), dtype=float))
        if not _np.isfinite(y).all():
            raise IntegrationFailure(f"solution not finite near t={t}")
    return y
