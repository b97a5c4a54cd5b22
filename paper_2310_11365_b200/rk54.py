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

from . import _lib


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
