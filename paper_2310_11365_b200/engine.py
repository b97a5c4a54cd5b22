"""Micro-macro Parareal on the GPU (drop-in for mcparareal.engine,
/root/reference/pkg/src/mcparareal/engine.py:39-277).

    iteration 0:   rho_{n+1} = C(rho_n),  u_{n+1} = lift(rho_{n+1})
    iteration k+1: rho_{n+1} = R(F(u_n^k)) + [C(rho_n^{k+1}) - C(rho_n^k)]
                   u_{n+1}   = match(rho_{n+1}, F(u_n^k))

Every stage of an iteration is a stream-ordered kernel on device-resident
data: fine sweep over all slices (fine.cu) -> restriction (coupling.cu) ->
serial coarse row + correction in one warp (coarse.cu) -> match (coupling.cu)
-> restriction of the matched ensembles.  The host issues launches only; the
single device->host transfer happens after the last iteration, and errors are
reported in the reference's order from device status arrays.  With frozen
noise the increments of all slices are materialised once per run
(noise.cu) and re-read by every iteration's sweep.
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, kernels
from ._device import device, require_cuda, torch
from .errors import ConfigError, DegenerateMatch, IntegrationFailure, NumericalBlowup
from .models import InitialDistribution, McKeanVlasovModel, device_model
from .moments import MomentODE, device_ode
from .noise import row_pitch, slice_noise
from .particles import NoisePlan, ParticleEnsemble, StepConfig, sample_initial
from .rk54 import EulerConfig, IntegratorConfig, integrator_descriptor
from .state import SINGLE_REGION, MacroState, RegionPartition

logger = logging.getLogger("mcparareal.engine")


@dataclass(frozen=True)
class PararealConfig:
    """Shape of one micro-macro Parareal run (engine.py:39-76)."""

    n_slices: int
    iterations: int
    slice_length: float
    particles: int
    step: StepConfig
    partition: RegionPartition = SINGLE_REGION
    integrator: IntegratorConfig | EulerConfig = IntegratorConfig()
    workers: int = 1
    t_start: float = 0.0
    retain_snapshots: bool = True
    stop_wasserstein_tol: float | None = None

    def __post_init__(self):
        if self.n_slices < 1:
            raise ConfigError("n_slices must be at least 1")
        if not 0 <= self.iterations <= self.n_slices:
            raise ConfigError("iterations must lie in [0, n_slices]; beyond n_slices the iteration is exact already")
        if self.slice_length <= 0:
            raise ConfigError("slice_length must be positive")
        if self.particles < 1:
            raise ConfigError("particles must be at least 1")
        if self.workers < 1:
            raise ConfigError("workers must be at least 1")
        covered = self.step.slice_length
        if abs(covered - self.slice_length) > 1e-9 * max(self.slice_length, 1.0):
            raise ConfigError(f"dt * steps_per_slice = {covered!r} does not cover the slice length "
                              f"{self.slice_length!r}")

    @property
    def horizon(self) -> float:
        return self.n_slices * self.slice_length


@dataclass
class PararealTrace:
    """Macro and micro iterates plus diagnostics of one run (engine.py:79-107).

    ``snapshots[k][n]`` are device-resident ensembles (views into the run's
    snapshot buffer).  ``timings`` holds per-stage device times in seconds.
    """

    times: tuple[float, ...]
    macro: list
    micro_stats: list
    snapshots: list | None
    noise_mode: str
    master_seed: int
    clamp_events: list = field(default_factory=list)
    fraction_gaps: list = field(default_factory=list)
    lift_collapses: list = field(default_factory=list)
    timings: dict = field(default_factory=dict)
    stopped_at: int | None = None
    d2h_bytes: int = 0

    @property
    def n_slices(self) -> int:
        return len(self.times) - 1

    @property
    def iterations(self) -> int:
        return len(self.macro) - 1


class _StageTimer:
    """CUDA-event timing of engine stages, resolved after the run."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.marks: list[tuple[str, object, object]] = []

    def start(self):
        if not self.enabled:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def stop(self, key, start):
        if not self.enabled:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((key, start, e))

    def resolve(self) -> dict:
        out = {"coarse": [], "fine": [], "restrict": [], "match": [], "noise": []}
        for key, a, b in self.marks:
            out.setdefault(key, []).append(a.elapsed_time(b) / 1e3)
        return out


def _initial_ensemble(initial, cfg: PararealConfig, plan: NoisePlan) -> ParticleEnsemble:
    if isinstance(initial, ParticleEnsemble):
        if initial.size != cfg.particles:
            raise ConfigError(f"initial ensemble has {initial.size} particles, config wants {cfg.particles}")
        return initial
    return sample_initial(initial, plan, cfg.particles)


class _Workspace:
    """Device buffers of one run (sized for 180 GB HBM: increments of every
    slice, snapshots of every iterate when retained)."""

    def __init__(self, K: int, N: int, P: int, S: int, I: int, retain: bool):
        dev = device()
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        nv = 3 * I
        self.snap = torch.empty((K + 1 if retain else 2, N + 1, P), **f64)
        self.fine = torch.empty((N, P), **f64)
        self.xi = torch.empty((N, S, row_pitch(P)), **f64)
        self.macro = torch.empty((K + 1, N + 1, nv), **f64)
        self.micro = torch.empty((K + 1, N + 1, nv), **f64)
        self.micro_counts = torch.empty((K + 1, N + 1, I), **i64)
        self.fine_stats = torch.empty((max(K, 1), N, nv), **f64)
        self.fine_counts = torch.empty((max(K, 1), N, I), **i64)
        self.raw = torch.empty((max(K, 1), N, nv), **f64)
        self.cache = torch.empty((K + 1, N, nv), **f64)
        self.bad = torch.full((max(K, 1), N), _lib.STAT_OK, **i32)
        self.coarse_status = torch.full((K + 1, N), _lib.STAT_OK, **i32)
        self.match_status = torch.full((K + 1, N), _lib.STAT_OK, **i32)
        self.rho0 = torch.empty((1, nv), **f64)
        self.counts0 = torch.empty((1, I), **i64)
        self.scratch = torch.empty(((N + 1) * I * P,), **f64) if I > 1 else None


def _wasserstein_delta(a, b, part_desc, scratch_stats, scratch_counts) -> float:
    """max_n mean|sort(a_n) - sort(b_n)| (engine.py:244-253) on the device."""
    diff = (torch.sort(a, dim=1).values - torch.sort(b, dim=1).values).abs_()
    kernels.restrict(part_desc, diff, scratch_stats, scratch_counts)
    return float(scratch_stats[:, 0].max().cpu())


def run_micro_macro(model: McKeanVlasovModel, coarse: MomentODE, initial: InitialDistribution | ParticleEnsemble,
                    cfg: PararealConfig, plan: NoisePlan, *, reuse_converged_coarse: bool = True,
                    record_timings: bool = True, increments=None) -> PararealTrace:
    """Run the micro-macro Parareal iteration on the GPU and record every iterate.

    ``increments`` (optional) injects the Brownian increments as a callable
    (n, k) -> (steps, P) array, or a device tensor (N, steps, >=P) used for
    every iteration (injected-increment mode of the parity tests).
    ``reuse_converged_coarse`` copies C(rho_n) for n < k from the previous
    row instead of re-integrating (bitwise identical: those inputs have
    converged exactly, engine.py:11-14).
    """
    require_cuda()
    if coarse.n_regions != cfg.partition.n_regions:
        raise ConfigError(f"moment model has {coarse.n_regions} regions but the partition has "
                          f"{cfg.partition.n_regions}")
    model_d = device_model(model)
    ode_d, ode_model_d = device_ode(coarse)
    integ_d = integrator_descriptor(cfg.integrator)
    part = cfg.partition
    part_d = part.descriptor()
    ens0 = _initial_ensemble(initial, cfg, plan)
    N, K, P, S, I = cfg.n_slices, cfg.iterations, cfg.particles, cfg.step.steps_per_slice, part.n_regions
    dt = cfg.step.dt
    times = tuple(cfg.t_start + n * cfg.slice_length for n in range(N + 1))
    times_d = torch.tensor(times, dtype=torch.float64, device=device())
    ws = _Workspace(K, N, P, S, I, cfg.retain_snapshots)
    timer = _StageTimer(record_timings)
    x0 = ens0.device_positions.reshape(1, P)

    def snap(k):
        return ws.snap[k if cfg.retain_snapshots else k % 2]

    # ---- iteration 0: coarse cascade + lift of the initial shape -------------
    snap(0)[0].copy_(ens0.device_positions)
    ev = timer.start()
    kernels.restrict(part_d, x0, ws.rho0, ws.counts0, ws.scratch)
    timer.stop("restrict", ev)
    ev = timer.start()
    kernels.coarse_row(ode_d, ode_model_d, integ_d, times_d, 0, ws.rho0, None, None, ws.macro[0], ws.cache[0],
                       None, ws.coarse_status[0])
    timer.stop("coarse", ev)
    ev = timer.start()
    kernels.match(part_d, ws.macro[0, 1:], ws.rho0, ws.counts0, x0, snap(0)[1:], 1, ws.match_status[0])
    timer.stop("match", ev)
    kernels.restrict(part_d, snap(0), ws.micro[0], ws.micro_counts[0], ws.scratch)

    # ---- increments ---------------------------------------------------------
    injected_fn = increments if callable(increments) else None
    if increments is not None and not callable(increments):
        ws.xi = increments
    elif injected_fn is None and not plan.fresh:
        ev = timer.start()
        slice_noise(plan.master_seed, 0, N, S, P, 0, False, out=ws.xi)
        timer.stop("noise", ev)

    stopped_at = None
    iterations_done = 0
    for k in range(K):
        if injected_fn is not None:
            for n in range(N):
                ws.xi[n, :, :P] = torch.as_tensor(np.asarray(injected_fn(n, k), dtype=float)).to(device())
        elif increments is None and plan.fresh:
            ev = timer.start()
            slice_noise(plan.master_seed, 0, N, S, P, k, True, out=ws.xi)
            timer.stop("noise", ev)
        cur, nxt = snap(k), snap(k + 1)
        ev = timer.start()
        kernels.fine_sweep(model_d, cur[:N], ws.fine, times_d[:N], S, dt, ws.xi, ws.bad[k])
        timer.stop("fine", ev)
        ev = timer.start()
        kernels.restrict(part_d, ws.fine, ws.fine_stats[k], ws.fine_counts[k], ws.scratch)
        timer.stop("restrict", ev)
        ev = timer.start()
        kernels.coarse_row(ode_d, ode_model_d, integ_d, times_d, k + 1, ws.rho0, ws.fine_stats[k], ws.cache[k],
                           ws.macro[k + 1], ws.cache[k + 1], ws.raw[k], ws.coarse_status[k + 1],
                           skip_until=(k + 1) if reuse_converged_coarse else 0)
        timer.stop("coarse", ev)
        ev = timer.start()
        kernels.match(part_d, ws.macro[k + 1, 1:], ws.fine_stats[k], ws.fine_counts[k], ws.fine, nxt[1:], 0,
                      ws.match_status[k + 1])
        nxt[0].copy_(ens0.device_positions)
        timer.stop("match", ev)
        kernels.restrict(part_d, nxt, ws.micro[k + 1], ws.micro_counts[k + 1], ws.scratch)
        iterations_done = k + 1
        if cfg.stop_wasserstein_tol is not None:
            st = torch.empty((N, 3), dtype=torch.float64, device=device())
            ct = torch.empty((N, 1), dtype=torch.int64, device=device())
            delta = _wasserstein_delta(nxt[1:], cur[1:], SINGLE_REGION.descriptor(), st, ct)
            if delta <= cfg.stop_wasserstein_tol:
                stopped_at = k + 1
                logger.info("stopping after iteration %d: max slice Wasserstein delta %.3e", k + 1, delta)
                break

    # ---- one device->host transfer, then the reference's error order --------
    torch.cuda.synchronize()
    Kd = iterations_done
    h = {name: getattr(ws, name).cpu().numpy() for name in
         ("macro", "micro", "micro_counts", "fine_stats", "raw", "bad", "coarse_status", "match_status",
          "rho0", "counts0")}
    _raise_first_error(h, N, Kd, I)
    trace = _build_trace(h, ws, cfg, plan, times, Kd, I, timer, stopped_at)
    trace.d2h_bytes = int(sum(v.nbytes for v in h.values()))
    return trace


def _raise_first_error(h, N: int, K: int, I: int) -> None:
    for n in range(N):
        if h["coarse_status"][0, n] != _lib.STAT_OK:
            raise IntegrationFailure(f"coarse integration failed on slice {n} (iteration 0)")
    for k in range(K):
        bad = h["bad"][k]
        for n in range(N):
            if bad[n] != _lib.STAT_OK:
                raise NumericalBlowup(f"non-finite particle position in slice {n}, step {int(bad[n])}",
                                      slice_index=n, step_index=int(bad[n]))
        for n in range(N):
            if h["coarse_status"][k + 1, n] != _lib.STAT_OK:
                raise IntegrationFailure(f"coarse integration failed on slice {n} (iteration {k + 1})")
            region = int(h["match_status"][k + 1, n])
            if region >= 0:
                var_t = h["macro"][k + 1, n + 1, I + region]
                raise DegenerateMatch(f"region {region}: cannot scale a zero-variance group to variance "
                                      f"{var_t:.3e}", region=region)


def _build_trace(h, ws, cfg, plan, times, K, I, timer, stopped_at) -> PararealTrace:
    N = cfg.n_slices
    trace = PararealTrace(times=times, macro=[], micro_stats=[], snapshots=[] if cfg.retain_snapshots else None,
                          noise_mode=plan.mode.value, master_seed=plan.master_seed, stopped_at=stopped_at)
    rho0_deg = tuple(h["counts0"][0] < 2)
    for k in range(K + 1):
        row = [MacroState.from_packed(h["macro"][k, 0], I, rho0_deg)]
        row += [MacroState.from_packed(h["macro"][k, n], I) for n in range(1, N + 1)]
        trace.macro.append(row)
        trace.micro_stats.append([MacroState.from_packed(h["micro"][k, n], I, tuple(h["micro_counts"][k, n] < 2))
                                  for n in range(N + 1)])
        if trace.snapshots is not None:
            trace.snapshots.append([ParticleEnsemble._wrap(ws.snap[k, n]) for n in range(N + 1)])
    rho0 = h["rho0"][0]
    for n in range(N):
        for i in range(I):
            if rho0[I + i] == 0.0 and h["macro"][0, n + 1, I + i] > 0.0 and rho0[2 * I + i] > 0.0:
                trace.lift_collapses.append((0, n + 1, i))
    for n in range(1, N + 1):
        gap = max(abs(a - b) for a, b in zip(h["macro"][0, n, 2 * I:].tolist(), h["micro"][0, n, 2 * I:].tolist()))
        trace.fraction_gaps.append((0, n, gap))
    for k in range(K):
        for n in range(N):
            raw = h["raw"][k, n].tolist()
            fine = h["fine_stats"][k, n].tolist()
            trace.fraction_gaps.append((k + 1, n + 1, max(abs(a - b) for a, b in zip(raw[2 * I:], fine[2 * I:]))))
            for i in range(I):
                if raw[I + i] < 0.0:
                    trace.clamp_events.append((k + 1, n + 1, i, raw[I + i]))
    trace.timings = timer.resolve()
    return trace


def _fine_sweep(model, ensembles, times, cfg: PararealConfig, plan: NoisePlan, iteration: int, pool=None):
    """F(u_n) for every slice start n in one launch (engine.py:110-124);
    returns (ensembles, per-launch seconds)."""
    desc = device_model(model)
    N, P, S = cfg.n_slices, cfg.particles, cfg.step.steps_per_slice
    x = torch.stack([e.device_positions for e in list(ensembles)[:N]])
    out = torch.empty_like(x)
    bad = torch.empty(N, dtype=torch.int32, device=device())
    xi = slice_noise(plan.master_seed, 0, N, S, P, iteration, plan.fresh)
    t0 = torch.tensor(list(times[:N]), dtype=torch.float64, device=device())
    start = time.perf_counter()
    kernels.fine_sweep(desc, x, out, t0, S, cfg.step.dt, xi, bad)
    b = bad.cpu().numpy()
    elapsed = time.perf_counter() - start
    for n in range(N):
        if b[n] != _lib.STAT_OK:
            raise NumericalBlowup(f"non-finite particle position in slice {n}, step {int(b[n])}",
                                  slice_index=n, step_index=int(b[n]))
    return [ParticleEnsemble._wrap(out[n]) for n in range(N)], [elapsed] * N


def sequential_fine(model: McKeanVlasovModel, initial: InitialDistribution | ParticleEnsemble,
                    cfg: PararealConfig, plan: NoisePlan, iteration: int = 0) -> list[ParticleEnsemble]:
    """Serial fine propagation over all slices (engine.py:262-277): one
    launch per slice, increments of every slice generated in one launch."""
    desc = device_model(model)
    ens = initial if isinstance(initial, ParticleEnsemble) else sample_initial(initial, plan, cfg.particles)
    N, P, S = cfg.n_slices, ens.size, cfg.step.steps_per_slice
    xs = torch.empty((N + 1, P), dtype=torch.float64, device=device())
    xs[0].copy_(ens.device_positions)
    xi = slice_noise(plan.master_seed, 0, N, S, P, iteration, plan.fresh)
    t0 = torch.tensor([cfg.t_start + n * cfg.slice_length for n in range(N)], dtype=torch.float64,
                      device=device())
    bad = torch.empty(N, dtype=torch.int32, device=device())
    for n in range(N):
        kernels.fine_sweep(desc, xs[n:n + 1], xs[n + 1:n + 2], t0[n:n + 1], S, cfg.step.dt, xi[n:n + 1],
                           bad[n:n + 1])
    b = bad.cpu().numpy()
    for n in range(N):
        if b[n] != _lib.STAT_OK:
            raise NumericalBlowup(f"non-finite particle position in slice {n}, step {int(b[n])}",
                                  slice_index=n, step_index=int(b[n]))
    return [ens] + [ParticleEnsemble._wrap(xs[n]) for n in range(1, N + 1)]
