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
import os
import time
import weakref
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _lib, kernels
from ._device import device, require_cuda, torch
from .errors import ConfigError, DegenerateMatch, IntegrationFailure, NumericalBlowup, SingularityError
from .models import InitialDistribution, McKeanVlasovModel, device_model
from .moments import MomentODE, device_ode
from .noise import fill_normals, row_pitch, slice_noise, step_keys
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
    snapshot buffer).  ``timings`` has the reference's keys: "fine" holds
    one device time per slice propagation (iteration-major, seconds);
    "coarse" / "restrict" / "match" hold CUDA-event stage times when the run
    recorded timings.  ``stage_timings``: every recorded stage (also
    "noise" and "iterations", the pipeline launch).
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
    stage_timings: dict = field(default_factory=dict)
    stopped_at: int | None = None
    d2h_bytes: int = 0
    snapshot_positions: np.ndarray | None = None  # host copy streamed during the run (snapshots_to_host)

    @property
    def n_slices(self) -> int:
        return len(self.times) - 1

    def _detach(self) -> None:
        """Give this trace private copies of the cached run buffers its
        snapshots view (called before the next run of the same
        configuration overwrites them: ensembles stay immutable)."""
        if isinstance(self.snapshots, _SnapshotRows):
            self.snapshots.detach()
        if self.snapshot_positions is not None:
            self.snapshot_positions = self.snapshot_positions.copy()

    @property
    def iterations(self) -> int:
        return len(self.macro) - 1

    def __getattr__(self, name):
        # diagnostics of an engine-built trace (clamp_events, fraction_gaps,
        # lift_collapses, timings) are lists of Python tuples built on first
        # access: building them eagerly is host time the GPU idles behind
        lazy = self.__dict__.get("_lazy")
        if lazy is not None and name in lazy:
            value = lazy.pop(name)()
            self.__dict__[name] = value
            return value
        raise AttributeError(name)


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
    slice, snapshots of every iterate when retained).  The small per-slice
    arrays the host reads back are views of three packed report buffers, so
    the end-of-run transfer is three copies."""

    F64 = ("macro", "micro", "fine_stats", "raw", "rho0")
    I64 = ("micro_counts", "fine_counts", "counts0", "fine_times")
    I32 = ("bad", "coarse_status", "match_status")

    def __init__(self, K: int, N: int, P: int, S: int, I: int, retain: bool, noise_slices: int | None = None,
                 counter: bool = False):
        dev = device()
        nv = 3 * I
        Kc = max(K, 1)
        shapes = {"macro": (K + 1, N + 1, nv), "micro": (K + 1, N + 1, nv), "fine_stats": (Kc, N, nv),
                  "raw": (Kc, N, nv), "rho0": (1, nv), "micro_counts": (K + 1, N + 1, I),
                  "fine_counts": (Kc, N, I), "counts0": (1, I), "fine_times": (Kc, N, 2), "bad": (Kc, N),
                  "coarse_status": (K + 1, N),
                  "match_status": (K + 1, N)}
        self.report = {}
        self.layout = {}  # dtype -> [(name, offset, size, shape)] of the packed report buffer
        for names, dtype in ((self.F64, torch.float64), (self.I64, torch.int64), (self.I32, torch.int32)):
            sizes = [int(np.prod(shapes[n])) for n in names]
            flat = torch.zeros(sum(sizes), dtype=dtype, device=dev)
            self.report[dtype] = flat
            off = 0
            self.layout[dtype] = []
            for n, size in zip(names, sizes):
                setattr(self, n, flat[off:off + size].view(shapes[n]))
                self.layout[dtype].append((n, off, size, shapes[n]))
                off += size
        self.snap = torch.empty((K + 1 if retain else 2, N + 1, P), dtype=torch.float64, device=dev)
        self.fine = torch.empty((N, P), dtype=torch.float64, device=dev)
        self.cache = torch.empty((K + 1, N, nv), dtype=torch.float64, device=dev)
        self.scratch = (torch.empty((kernels.restrict_scratch(N + 1, P, I),), dtype=torch.float64, device=dev)
                        if I > 1 else None)
        self.x0 = torch.empty((1, P), dtype=torch.float64, device=dev)
        self.host = {dt: torch.empty(t.shape, dtype=dt, pin_memory=True) for dt, t in self.report.items()}
        # increments of a batch of slices: all N when they fit (frozen noise is
        # then generated once per run), else batches regenerated per iteration
        if counter:  # increments generated in registers: no stream buffer
            self.noise_slices = N
            self.xi = torch.empty((1, 1, 2), dtype=torch.float64, device=dev)
            return
        self.noise_slices = noise_slices if noise_slices else _noise_batch(N, S, P)
        self.xi = torch.empty((self.noise_slices, S, row_pitch(P)), dtype=torch.float64, device=dev)

    def reset_status(self):
        self.report[torch.int32].fill_(_lib.STAT_OK)

    def read_back(self) -> dict:
        """Stream-ordered copy of the report buffers into pinned memory, one sync."""
        for dt, t in self.report.items():
            self.host[dt].copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        # (host time from here to the next run's first launch is GPU idle
        # time: one copy per packed buffer -- the pinned buffers are reused by
        # the next run -- and views into it)
        h = {}
        for dt, entries in self.layout.items():
            flat = self.host[dt].numpy().copy()
            for n, off, size, shape in entries:
                h[n] = flat[off:off + size].reshape(shape)
        return h

    def report_bytes(self) -> int:
        return int(sum(t.numel() * t.element_size() for t in self.report.values()))


def _noise_batch(N: int, S: int, P: int) -> int:
    """Slices whose increments are held at once: all of them when they fit in
    80% of the free device memory (MMPR_NOISE_SLICES overrides)."""
    env = os.environ.get("MMPR_NOISE_SLICES")
    if env:
        return max(1, min(N, int(env)))
    per_slice = max(1, S) * row_pitch(P) * 8
    free, _ = torch.cuda.mem_get_info()
    return max(1, min(N, int(0.8 * free) // per_slice))


class _RunPlan:
    """One run configuration: its workspace and its launch sequence
    (replayed from a CUDA graph when the configuration repeats)."""

    def __init__(self, model_d, ode_d, ode_model_d, integ_d, part_d, cfg: PararealConfig, plan: NoisePlan,
                 reuse: bool, injected: bool = False, host_snapshots: bool = False, allow_pipeline: bool = True):
        self.model_d, self.ode_d, self.ode_model_d, self.integ_d, self.part_d = \
            model_d, ode_d, ode_model_d, integ_d, part_d
        self.cfg, self.plan, self.reuse = cfg, plan, reuse
        N, K, P, S, I = cfg.n_slices, cfg.iterations, cfg.particles, cfg.step.steps_per_slice, \
            cfg.partition.n_regions
        self.N, self.K, self.P, self.S, self.I = N, K, P, S, I
        self.times = tuple(cfg.t_start + n * cfg.slice_length for n in range(N + 1))
        self.times_d = torch.tensor(self.times, dtype=torch.float64, device=device())
        self.counter = plan.counter_based and not injected
        self.ws = _Workspace(K, N, P, S, I, cfg.retain_snapshots, noise_slices=N if injected else None,
                             counter=self.counter)
        # single-region restriction of the fine outputs fused into the sweep
        self.fused_restrict = I == 1 and model_d.stat_kind == _lib.STAT_MEAN_OF_F
        # several regions: match and micro restriction in one cluster pass
        # (kernels.match_restrict_regions) only with MMPR_RESTRICT_CLUSTER=1 --
        # measured slower than the separate passes on config 3 (12.2-12.5 vs
        # 11.3-11.8 ms per run: 14 clusters at a time, latency-bound phases)
        self.regions_fused = I > 1 and os.environ.get("MMPR_RESTRICT_CLUSTER", "0") == "1"
        # snapshot rows streamed to pinned host memory on a side stream while
        # the next iteration computes (harness artefacts need them on the host)
        self.host_snap = None
        self.copy_stream = None
        if host_snapshots:
            self.host_snap = torch.empty((K + 1, N + 1, P), dtype=torch.float64, pin_memory=True)
            self.copy_stream = torch.cuda.Stream()
        self.batch = self.ws.noise_slices
        self.side_stream = None
        self.graph = None
        self.launches_per_run = 0
        # iterations 1..K as one persistent kernel (mmpr_parareal_pipeline)
        # when the configuration has an instantiation; every iterate is
        # bitwise the one of the per-iteration kernel sequence.  Not with the
        # Wasserstein stop criterion (a host decision after every iteration)
        # or per-iteration increment callables (allow_pipeline=False).
        self.prev_trace = None  # weakref to the last trace built on this plan's buffers
        # (two regions: the units restrict over compacted members themselves)
        pipe_restrict = self.fused_restrict or (I == 2 and model_d.stat_kind == _lib.STAT_MEAN_OF_F)
        # (FRESH noise: in the counter-based mode only -- each unit draws its
        # iteration's increments in registers; the numpy streams of a FRESH
        # run are materialised per iteration)
        self.pipeline = (allow_pipeline and K >= 1 and pipe_restrict and (not plan.fresh or self.counter)
                         and self.batch == N
                         and not host_snapshots and os.environ.get("MMPR_PIPELINE", "1") != "0"
                         and kernels.pipeline_supported(model_d, ode_d, ode_model_d, integ_d, P,
                                                        counter_noise=bool(self.counter)))
        self.rg_scratch = None
        if self.pipeline:
            self.ws.fine = torch.empty((2, N, P), dtype=torch.float64, device=device())
            self.flags = torch.empty((kernels.pipeline_flags_size(N, K),), dtype=torch.int32, device=device())
            if I > 1:
                self.rg_scratch = torch.empty((kernels.PIPELINE_SCRATCH_ROWS, I, P), dtype=torch.float64,
                                              device=device())

    def snap(self, k):
        return self.ws.snap[k if self.cfg.retain_snapshots else k % 2]

    def issue_prologue(self, timer, injected=False):
        """Iteration 0 (coarse cascade + lift) and, for frozen noise, the
        increments of every slice.  In front of the iteration pipeline the
        increments go first and iteration 0 runs on a side stream, in the
        SMs the noise kernel's last wave leaves free (untimed runs)."""
        ws = self.ws
        N, P, S = self.N, self.P, self.S
        ws.reset_status()
        self.snap(0)[0].copy_(ws.x0[0])
        noise_here = not injected and not self.counter and not self.plan.fresh and self.batch == N
        if noise_here and self.pipeline and not timer.enabled:
            main = torch.cuda.current_stream()
            if self.side_stream is None:
                self.side_stream = torch.cuda.Stream()
            self.side_stream.wait_stream(main)
            slice_noise(self.plan.master_seed, 0, N, S, P, 0, False, out=ws.xi)
            with torch.cuda.stream(self.side_stream):
                self._iteration_zero(timer)
            main.wait_stream(self.side_stream)
            return
        self._iteration_zero(timer)
        if noise_here:
            ev = timer.start()
            slice_noise(self.plan.master_seed, 0, N, S, P, 0, False, out=ws.xi)
            timer.stop("noise", ev)

    def _iteration_zero(self, timer):
        """rho0 = R(ens0), the coarse cascade, the lift (engine.py:153-195)."""
        ws, part_d = self.ws, self.part_d
        ev = timer.start()
        kernels.restrict(part_d, ws.x0, ws.rho0, ws.counts0, ws.scratch)
        timer.stop("restrict", ev)
        ev = timer.start()
        kernels.coarse_row(self.ode_d, self.ode_model_d, self.integ_d, self.times_d, 0, ws.rho0, None, None,
                           ws.macro[0], ws.cache[0], None, ws.coarse_status[0])
        timer.stop("coarse", ev)
        ev = timer.start()
        if self.fused_restrict:  # lift and micro restriction in one pass; row 0 is ens0 itself
            kernels.match_restrict(ws.macro[0, 1:], ws.rho0, ws.counts0, ws.x0, self.snap(0)[1:], 1,
                                   ws.match_status[0], ws.micro[0, 1:], ws.micro_counts[0, 1:])
            ws.micro[0, 0].copy_(ws.rho0[0])
            ws.micro_counts[0, 0].copy_(ws.counts0[0])
        elif self.regions_fused:  # per-region lift and restriction in one pass
            kernels.match_restrict_regions(part_d, ws.macro[0, 1:], ws.rho0, ws.counts0, ws.x0, self.snap(0)[1:], 1,
                                           ws.match_status[0], ws.micro[0, 1:], ws.micro_counts[0, 1:], ws.scratch)
            ws.micro[0, 0].copy_(ws.rho0[0])
            ws.micro_counts[0, 0].copy_(ws.counts0[0])
        else:
            kernels.match(part_d, ws.macro[0, 1:], ws.rho0, ws.counts0, ws.x0, self.snap(0)[1:], 1,
                          ws.match_status[0])
        timer.stop("match", ev)
        if not self.fused_restrict and not self.regions_fused:
            kernels.restrict(part_d, self.snap(0), ws.micro[0], ws.micro_counts[0], ws.scratch)

    def issue_iteration(self, k, timer, injected=False):
        ws, part_d, N, S, B = self.ws, self.part_d, self.N, self.S, self.batch
        cur, nxt = self.snap(k), self.snap(k + 1)
        counter = self.plan.counter_noise(k) if self.counter else None
        for a in range(0, N, B):
            nb = min(B, N - a)
            if counter is not None:
                counter.slice_offset = a
            elif not injected and (self.plan.fresh or B < N):
                ev = timer.start()
                slice_noise(self.plan.master_seed, a, nb, S, self.P, k, self.plan.fresh, out=ws.xi[:nb])
                timer.stop("noise", ev)
            ev = timer.start()
            if self.fused_restrict:  # R(F_n) computed by the sweep from registers
                kernels.fine_sweep(self.model_d, cur[a:a + nb], ws.fine[a:a + nb], self.times_d[a:a + nb], S,
                                   self.cfg.step.dt, ws.xi[:nb], ws.bad[k][a:a + nb],
                                   stats=ws.fine_stats[k][a:a + nb], counts=ws.fine_counts[k][a:a + nb],
                                   counter=counter, times=ws.fine_times[k][a:a + nb])
            else:
                kernels.fine_sweep(self.model_d, cur[a:a + nb], ws.fine[a:a + nb], self.times_d[a:a + nb], S,
                                   self.cfg.step.dt, ws.xi[:nb], ws.bad[k][a:a + nb], counter=counter,
                                   times=ws.fine_times[k][a:a + nb])
            timer.stop("fine", ev)
        if not self.fused_restrict:
            ev = timer.start()
            kernels.restrict(part_d, ws.fine, ws.fine_stats[k], ws.fine_counts[k], ws.scratch)
            timer.stop("restrict", ev)
        ev = timer.start()
        kernels.coarse_row(self.ode_d, self.ode_model_d, self.integ_d, self.times_d, k + 1, ws.rho0,
                           ws.fine_stats[k], ws.cache[k], ws.macro[k + 1], ws.cache[k + 1], ws.raw[k],
                           ws.coarse_status[k + 1], skip_until=(k + 1) if self.reuse else 0)
        timer.stop("coarse", ev)
        ev = timer.start()
        if self.fused_restrict:  # match and micro restriction in one pass; row 0 is ens0 itself
            kernels.match_restrict(ws.macro[k + 1, 1:], ws.fine_stats[k], ws.fine_counts[k], ws.fine, nxt[1:], 0,
                                   ws.match_status[k + 1], ws.micro[k + 1, 1:], ws.micro_counts[k + 1, 1:])
            ws.micro[k + 1, 0].copy_(ws.rho0[0])
            ws.micro_counts[k + 1, 0].copy_(ws.counts0[0])
        elif self.regions_fused:  # per-region match and micro restriction in one pass
            kernels.match_restrict_regions(part_d, ws.macro[k + 1, 1:], ws.fine_stats[k], ws.fine_counts[k], ws.fine,
                                           nxt[1:], 0, ws.match_status[k + 1], ws.micro[k + 1, 1:],
                                           ws.micro_counts[k + 1, 1:], ws.scratch)
            ws.micro[k + 1, 0].copy_(ws.rho0[0])
            ws.micro_counts[k + 1, 0].copy_(ws.counts0[0])
        else:
            kernels.match(part_d, ws.macro[k + 1, 1:], ws.fine_stats[k], ws.fine_counts[k], ws.fine, nxt[1:], 0,
                          ws.match_status[k + 1])
        nxt[0].copy_(ws.x0[0])
        timer.stop("match", ev)
        if not self.fused_restrict and not self.regions_fused:
            kernels.restrict(part_d, nxt, ws.micro[k + 1], ws.micro_counts[k + 1], ws.scratch)

    def issue_pipeline(self, timer):
        """Iterations 1..K in one launch (after issue_prologue)."""
        ws = self.ws
        ev = timer.start()
        kernels.parareal_pipeline(self.model_d, self.ode_d, self.ode_model_d, self.integ_d,
                                  self.cfg.step.dt, self.S, self.reuse, self.times_d, ws.x0, ws.rho0, ws.counts0,
                                  ws.xi, ws.snap, ws.fine, ws.macro, ws.micro, ws.micro_counts, ws.fine_stats,
                                  ws.fine_counts, ws.raw, ws.cache, ws.bad, ws.coarse_status, ws.match_status,
                                  self.flags, counter=self._pipeline_counter(),
                                  partition=self.part_d if self.I > 1 else None, region_scratch=self.rg_scratch,
                                  fine_times=ws.fine_times)
        timer.stop("iterations", ev)

    def _pipeline_counter(self):
        if not self.counter:
            return None
        c = self.plan.counter_noise(0)
        if self.plan.fresh:
            c.kfield = _lib.COUNTER_FRESH  # iteration k's units draw with field k + 1
        return c

    def stream_row(self, k):
        """Copy snapshot row k to pinned host memory on the side stream."""
        if self.host_snap is None:
            return
        main = torch.cuda.current_stream()
        self.copy_stream.wait_stream(main)
        with torch.cuda.stream(self.copy_stream):
            self.host_snap[k].copy_(self.snap(k), non_blocking=True)

    def join(self):
        if self.copy_stream is not None:
            torch.cuda.current_stream().wait_stream(self.copy_stream)

    def issue_all(self, timer):
        self.issue_prologue(timer)
        self.stream_row(0)
        if self.pipeline:
            self.issue_pipeline(timer)
        else:
            for k in range(self.K):
                self.issue_iteration(k, timer)
                self.stream_row(k + 1)
        self.join()

    def replay(self):
        """Launch the whole run as one CUDA graph (captured on first use)."""
        if self.graph is None:
            before = _lib.launch_count["total"]
            self.issue_all(_StageTimer(False))  # eager warm-up: sets kernel attributes, checks arguments
            self.launches_per_run = _lib.launch_count["total"] - before
            torch.cuda.current_stream().synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.issue_all(_StageTimer(False))
            self.graph = g
        self.graph.replay()


_PLANS: dict = {}
_PLANS_MAX = 2
# how the last run_micro_macro executed (tests and bench read it)
last_run_info: dict = {"pipeline": False}


def clear_graph_cache() -> None:
    """Drop cached run plans (workspaces and CUDA graphs)."""
    _PLANS.clear()


def _plan_key(model_d, ode_d, ode_model_d, integ_d, part_d, cfg, plan, reuse):
    return (bytes(model_d), bytes(ode_d), bytes(ode_model_d), bytes(integ_d), bytes(part_d), cfg.n_slices,
            cfg.iterations, cfg.particles, cfg.step.dt, cfg.step.steps_per_slice, cfg.slice_length, cfg.t_start,
            cfg.retain_snapshots, plan.master_seed, plan.mode, reuse, torch.cuda.current_device(),
            os.environ.get("MMPR_NOISE_SLICES"), os.environ.get("MMPR_PIPELINE", "1"),
            os.environ.get("MMPR_RESTRICT_CLUSTER", "0"))


def _wasserstein_delta(a, b) -> float:
    """max_n mean|sort(a_n) - sort(b_n)| (engine.py:244-253) on the device."""
    return float(kernels.mean_abs_diff(kernels.sort_rows(a), kernels.sort_rows(b)).max().cpu())


def run_micro_macro(model: McKeanVlasovModel, coarse: MomentODE, initial: InitialDistribution | ParticleEnsemble,
                    cfg: PararealConfig, plan: NoisePlan, *, reuse_converged_coarse: bool = True,
                    record_timings: bool = False, increments=None, use_graph: bool = True,
                    snapshots_to_host: bool = False) -> PararealTrace:
    """Run the micro-macro Parareal iteration on the GPU and record every iterate.

    ``increments`` (optional) injects the Brownian increments as a callable
    (n, k) -> (steps, P) array, or a device tensor (N, steps, >=P) used for
    every iteration (injected-increment mode of the parity tests).
    ``reuse_converged_coarse`` copies C(rho_n) for n < k from the previous
    row instead of re-integrating (bitwise identical: those inputs have
    converged exactly, engine.py:11-14).
    ``snapshots_to_host`` streams every iterate's snapshot row to pinned host
    memory on a side stream while the next iteration computes; the result is
    ``trace.snapshot_positions`` ((K+1, N+1, P) numpy, reused by the next run
    of the same configuration like the device snapshots).
    ``use_graph`` replays the run's launch sequence as one CUDA graph, cached
    per configuration (eager launches when timings are recorded, increments
    are injected or the Wasserstein stop criterion is active).
    Snapshots of a graph-replayed run view the cached workspace; when the
    same configuration runs again while an earlier trace is still
    referenced, that trace first receives its own copy (copy on reuse), so
    ensembles never change under the caller.
    """
    require_cuda()
    if coarse.n_regions != cfg.partition.n_regions:
        raise ConfigError(f"moment model has {coarse.n_regions} regions but the partition has "
                          f"{cfg.partition.n_regions}")
    model_d = device_model(model)
    ode_d, ode_model_d = device_ode(coarse)
    integ_d = integrator_descriptor(cfg.integrator)
    part_d = cfg.partition.descriptor()
    ens0 = _initial_ensemble(initial, cfg, plan)
    # Reusing C(rho_n) of converged slices relies on their inputs being
    # bitwise unchanged, which holds only when every iteration sees the same
    # increments (FROZEN noise, or one injected array for all iterations).
    reuse_converged_coarse = reuse_converged_coarse and not plan.fresh and not callable(increments)
    eager = record_timings or increments is not None or cfg.stop_wasserstein_tol is not None or not use_graph
    if snapshots_to_host and not cfg.retain_snapshots:
        raise ConfigError("snapshots_to_host needs retain_snapshots=True")
    if eager:
        rp = _RunPlan(model_d, ode_d, ode_model_d, integ_d, part_d, cfg, plan, reuse_converged_coarse,
                      injected=increments is not None, host_snapshots=snapshots_to_host,
                      allow_pipeline=cfg.stop_wasserstein_tol is None and not callable(increments))
    else:
        key = _plan_key(model_d, ode_d, ode_model_d, integ_d, part_d, cfg, plan, reuse_converged_coarse) + \
            (snapshots_to_host,)
        rp = _PLANS.get(key)
        if rp is None:
            while len(_PLANS) >= _PLANS_MAX:
                _PLANS.pop(next(iter(_PLANS)))
            rp = _RunPlan(model_d, ode_d, ode_model_d, integ_d, part_d, cfg, plan, reuse_converged_coarse,
                          host_snapshots=snapshots_to_host)
            _PLANS[key] = rp
        # the cached workspace is about to be overwritten: a trace of an
        # earlier run that is still referenced gets its own copy first
        prev = rp.prev_trace() if rp.prev_trace is not None else None
        if prev is not None:
            prev._detach()
    ws = rp.ws
    last_run_info["pipeline"] = rp.pipeline
    ws.x0.copy_(ens0.device_positions.reshape(1, -1))
    timer = _StageTimer(record_timings)
    N, K, P = rp.N, rp.K, rp.P
    stopped_at = None
    iterations_done = K
    if not eager:
        rp.replay()
        _lib.launch_count["total"] += rp.launches_per_run
    else:
        injected = increments is not None
        if injected and not callable(increments):
            ws.xi = increments
        rp.issue_prologue(timer, injected)
        rp.stream_row(0)
        if rp.pipeline:
            rp.issue_pipeline(timer)
        for k in range(0 if rp.pipeline else K):
            if callable(increments):
                for n in range(N):
                    ws.xi[n, :, :P] = torch.as_tensor(np.asarray(increments(n, k), dtype=float)).to(device())
            rp.issue_iteration(k, timer, injected)
            rp.stream_row(k + 1)
            iterations_done = k + 1
            if cfg.stop_wasserstein_tol is not None:
                delta = _wasserstein_delta(rp.snap(k + 1)[1:], rp.snap(k)[1:])
                if delta <= cfg.stop_wasserstein_tol:
                    stopped_at = k + 1
                    logger.info("stopping after iteration %d: max slice Wasserstein delta %.3e", k + 1, delta)
                    break

    rp.join()
    # ---- one device->host transfer, then the reference's error order --------
    h = ws.read_back()
    Kd = iterations_done
    for name in ("macro", "micro", "micro_counts"):
        h[name] = h[name][:Kd + 1]
    _raise_first_error(h, N, Kd, cfg.partition.n_regions)
    trace = _build_trace(h, ws, cfg, plan, rp.times, Kd, cfg.partition.n_regions, timer, stopped_at)
    trace.d2h_bytes = ws.report_bytes()
    if rp.host_snap is not None:
        trace.snapshot_positions = rp.host_snap.numpy()[:Kd + 1]
        trace.d2h_bytes += int(rp.host_snap[:Kd + 1].numel()) * 8
    if not eager:
        rp.prev_trace = weakref.ref(trace)
    return trace


def _coarse_error(status: int, n: int, k: int):
    if status == _lib.STAT_SINGULAR:
        return SingularityError(f"moment closure singular on slice {n} (iteration {k})")
    return IntegrationFailure(f"coarse integration failed on slice {n} (iteration {k})")


def _raise_first_error(h, N: int, K: int, I: int) -> None:
    if (h["bad"] == _lib.STAT_WATCHDOG).any() or (h["match_status"] == _lib.STAT_WATCHDOG).any():
        raise _lib.MmprError("iteration pipeline watchdog expired: a dependency between (k, n) units never "
                             "arrived; the run's results were discarded")
    # nothing to report (the usual case): three array comparisons instead of
    # the ordered scan below (which costs ~0.3 ms of host time for 64 x 5
    # units, with the GPU idle behind it)
    if (not (h["coarse_status"][:K + 1, :N] != _lib.STAT_OK).any() and not (h["bad"][:K, :N] != _lib.STAT_OK).any()
            and not (h["match_status"][1:K + 1, :N] >= 0).any()):
        return
    for n in range(N):
        if h["coarse_status"][0, n] != _lib.STAT_OK:
            raise _coarse_error(int(h["coarse_status"][0, n]), n, 0)
    for k in range(K):
        bad = h["bad"][k]
        for n in range(N):
            if bad[n] != _lib.STAT_OK:
                raise NumericalBlowup(f"non-finite particle position in slice {n}, step {int(bad[n])}",
                                      slice_index=n, step_index=int(bad[n]))
        for n in range(N):
            if h["coarse_status"][k + 1, n] != _lib.STAT_OK:
                raise _coarse_error(int(h["coarse_status"][k + 1, n]), n, k + 1)
            region = int(h["match_status"][k + 1, n])
            if region >= 0:
                var_t = h["macro"][k + 1, n + 1, I + region]
                raise DegenerateMatch(f"region {region}: cannot scale a zero-variance group to variance "
                                      f"{var_t:.3e}", region=region)


class _LazyRows(Sequence):
    """Read-only list of trace rows materialised on first access (building
    every MacroState eagerly costs more host time than the device run)."""

    def __init__(self, n: int, make_row):
        self._n = n
        self._make = make_row
        self._rows: dict = {}

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(self._n))]
        if k < 0:
            k += self._n
        if not 0 <= k < self._n:
            raise IndexError(k)
        row = self._rows.get(k)
        if row is None:
            row = self._rows[k] = self._make(k)
        return row

    def __repr__(self) -> str:
        return f"<{self._n} trace rows>"


class _SnapshotRows(_LazyRows):
    """trace.snapshots: rows of ensembles viewing the run's snapshot buffer."""

    def __init__(self, K: int, N: int, buf):
        self.buf, self.N = buf, N
        super().__init__(K + 1, self._row)

    def _row(self, k):
        return [ParticleEnsemble._wrap(self.buf[k, n]) for n in range(self.N + 1)]

    def detach(self) -> None:
        new = self.buf[:self._n].clone()
        for k, row in self._rows.items():
            for n, e in enumerate(row):
                e._dev = new[k, n]
        self.buf = new


def _build_trace(h, ws, cfg, plan, times, K, I, timer, stopped_at) -> PararealTrace:
    N = cfg.n_slices
    macro, micro, mcounts = h["macro"], h["micro"], h["micro_counts"]
    rho0_deg = tuple(h["counts0"][0] < 2)

    def macro_row(k):
        return [MacroState.from_packed(macro[k, 0], I, rho0_deg)] + \
            [MacroState.from_packed(macro[k, n], I) for n in range(1, N + 1)]

    def micro_row(k):
        return [MacroState.from_packed(micro[k, n], I, tuple(mcounts[k, n] < 2)) for n in range(N + 1)]

    snapshots = None
    if cfg.retain_snapshots and ws is not None:
        snapshots = _SnapshotRows(K, N, ws.snap)
    trace = PararealTrace(times=times, macro=_LazyRows(K + 1, macro_row), micro_stats=_LazyRows(K + 1, micro_row),
                          snapshots=snapshots, noise_mode=plan.mode.value, master_seed=plan.master_seed,
                          stopped_at=stopped_at)
    # diagnostics (engine.py:178-181, 218-228), vectorised (abs/sub/max are
    # exact) and built on first access (PararealTrace.__getattr__)
    rho0 = h["rho0"][0]

    def lift_collapses():
        lift = (rho0[I:2 * I] == 0.0) & (macro[0, 1:, I:2 * I] > 0.0) & (rho0[2 * I:] > 0.0)
        return [(0, int(n) + 1, int(i)) for n, i in np.argwhere(lift)]

    def fraction_gaps():
        gaps0 = np.max(np.abs(macro[0, 1:, 2 * I:] - micro[0, 1:, 2 * I:]), axis=1).tolist()
        out = [(0, n + 1, g) for n, g in enumerate(gaps0)]
        if K > 0:
            raw, fine = h["raw"][:K], h["fine_stats"][:K]
            gaps = np.max(np.abs(raw[:, :, 2 * I:] - fine[:, :, 2 * I:]), axis=2).tolist()
            out += [(k + 1, n + 1, gaps[k][n]) for k in range(K) for n in range(N)]
        return out

    def clamp_events():
        if K == 0:
            return []
        neg = h["raw"][:K][:, :, I:2 * I]
        return [(int(k) + 1, int(n) + 1, int(i), float(neg[k, n, i])) for k, n, i in np.argwhere(neg < 0.0)]

    # the reference's timings (engine.py:149-233): per-slice fine propagation
    # times, here device time between each slice's first and last step
    # (globaltimer, so per-slice times overlap as the slices run
    # concurrently); the other stages as recorded CUDA-event times
    # (record_timings=True), every stage including the noise and the
    # iteration pipeline in stage_timings
    stages = timer.resolve()

    def timings():
        ft = h.get("fine_times")
        if ft is not None:
            ft = ft[:K].astype(np.int64)
            fine = np.where((ft[..., 0] > 0) & (ft[..., 1] >= ft[..., 0]), (ft[..., 1] - ft[..., 0]) * 1e-9, 0.0)
        else:  # multi-rank drivers: not gathered
            fine = np.zeros((0,))
        return {"coarse": list(stages.get("coarse", [])), "fine": fine.reshape(-1).tolist(),
                "restrict": list(stages.get("restrict", [])), "match": list(stages.get("match", []))}

    lazy = {"lift_collapses": lift_collapses, "fraction_gaps": fraction_gaps, "clamp_events": clamp_events,
            "timings": timings}
    for name in lazy:
        del trace.__dict__[name]
    trace.__dict__["_lazy"] = lazy
    trace.stage_timings = stages
    return trace


def _fine_sweep(model, ensembles, times, cfg: PararealConfig, plan: NoisePlan, iteration: int, pool=None):
    """F(u_n) for every slice start n in one launch (engine.py:110-124);
    returns (ensembles, per-launch seconds)."""
    desc = device_model(model)
    N, P, S = cfg.n_slices, cfg.particles, cfg.step.steps_per_slice
    x = torch.stack([e.device_positions for e in list(ensembles)[:N]])
    out = torch.empty_like(x)
    bad = torch.empty(N, dtype=torch.int32, device=device())
    counter = plan.counter_noise(iteration) if plan.counter_based else None
    xi = None if counter is not None else slice_noise(plan.master_seed, 0, N, S, P, iteration, plan.fresh)
    t0 = torch.tensor(list(times[:N]), dtype=torch.float64, device=device())
    start = time.perf_counter()
    kernels.fine_sweep(desc, x, out, t0, S, cfg.step.dt, xi, bad, counter=counter)
    b = bad.cpu().numpy()
    elapsed = time.perf_counter() - start
    for n in range(N):
        if b[n] != _lib.STAT_OK:
            raise NumericalBlowup(f"non-finite particle position in slice {n}, step {int(b[n])}",
                                  slice_index=n, step_index=int(b[n]))
    return [ParticleEnsemble._wrap(out[n]) for n in range(N)], [elapsed] * N


def _serial_chains(desc, ens0, plans, cfg: PararealConfig, iteration: int):
    """R independent serial fine chains advanced together: one fine-sweep
    launch per slice over all R chains.  Increments are generated for a
    batch of slices of every chain at a time (one key launch per chain, one
    fill launch), within the device-memory budget of _noise_batch."""
    R, N, S = len(plans), cfg.n_slices, cfg.step.steps_per_slice
    P = ens0[0].size
    pitch = row_pitch(P)
    xs = torch.empty((R, N + 1, P), dtype=torch.float64, device=device())
    for r, e in enumerate(ens0):
        xs[r, 0].copy_(e.device_positions)
    if any(pl.counter_based for pl in plans):
        if not all(pl.counter_based for pl in plans):
            raise ValueError("replica plans must all use counter-based noise or none")
        return _serial_chains_counter(desc, ens0, plans, cfg, iteration, xs)
    B = max(1, min(N, _noise_batch(N * R, S, P) // R)) if N else 1
    xi = torch.empty((B, R, S, pitch), dtype=torch.float64, device=device())
    bad = torch.empty((max(N, 1), R), dtype=torch.int32, device=device())
    t0 = [torch.full((R,), cfg.t_start + n * cfg.slice_length, dtype=torch.float64, device=device())
          for n in range(N)]
    for a in range(0, N, B):
        nb = min(B, N - a)
        keys = torch.stack([step_keys(pl.master_seed, pl.fresh, iteration, a, nb, S) for pl in plans], dim=1)
        fill_normals(keys, P, xi[:nb], pitch)
        for n in range(a, a + nb):
            kernels.fine_sweep(desc, xs[:, n], xs[:, n + 1], t0[n], S, cfg.step.dt, xi[n - a], bad[n])
    b = bad.cpu().numpy()
    for r in range(R):  # chain by chain, as separate serial runs would raise
        for n in range(N):
            if b[n, r] != _lib.STAT_OK:
                raise NumericalBlowup(f"non-finite particle position in slice {n}, step {int(b[n, r])}",
                                      slice_index=n, step_index=int(b[n, r]))
    return [[ens0[r]] + [ParticleEnsemble._wrap(xs[r, n]) for n in range(1, N + 1)] for r in range(R)]


def _serial_chains_counter(desc, ens0, plans, cfg: PararealConfig, iteration: int, xs):
    """_serial_chains with counter-based increments (no noise buffers): one
    launch per (chain, slice)."""
    R, N, S = len(plans), cfg.n_slices, cfg.step.steps_per_slice
    bad = torch.empty((max(N, 1), R), dtype=torch.int32, device=device())
    t0 = [torch.tensor([cfg.t_start + n * cfg.slice_length], dtype=torch.float64, device=device()) for n in range(N)]
    for r, pl in enumerate(plans):
        for n in range(N):
            kernels.fine_sweep(desc, xs[r, n:n + 1], xs[r, n + 1:n + 2], t0[n], S, cfg.step.dt, None, bad[n, r:r + 1],
                               counter=pl.counter_noise(iteration, n))
    b = bad.cpu().numpy()
    for r in range(R):
        for n in range(N):
            if b[n, r] != _lib.STAT_OK:
                raise NumericalBlowup(f"non-finite particle position in slice {n}, step {int(b[n, r])}",
                                      slice_index=n, step_index=int(b[n, r]))
    return [[ens0[r]] + [ParticleEnsemble._wrap(xs[r, n]) for n in range(1, N + 1)] for r in range(R)]


def sequential_fine(model: McKeanVlasovModel, initial: InitialDistribution | ParticleEnsemble,
                    cfg: PararealConfig, plan: NoisePlan, iteration: int = 0) -> list[ParticleEnsemble]:
    """Serial fine propagation over all slices (engine.py:262-277): one
    launch per slice, increments generated per batch of slices."""
    desc = device_model(model)
    ens = initial if isinstance(initial, ParticleEnsemble) else sample_initial(initial, plan, cfg.particles)
    return _serial_chains(desc, [ens], [plan], cfg, iteration)[0]


def sequential_fine_batch(model: McKeanVlasovModel, initial: InitialDistribution | ParticleEnsemble,
                          cfg: PararealConfig, plans, iteration: int = 0) -> list[list[ParticleEnsemble]]:
    """``[sequential_fine(model, initial, cfg, plan) for plan in plans]`` --
    the floor replicas of harness.run_experiment (harness.py:257-265) --
    with the replicas advanced together (one launch per slice for all of
    them).  Results are bit-identical to the separate serial runs."""
    desc = device_model(model)
    plans = list(plans)
    if not plans:
        return []
    ens0 = [initial if isinstance(initial, ParticleEnsemble) else sample_initial(initial, pl, cfg.particles)
            for pl in plans]
    return _serial_chains(desc, ens0, plans, cfg, iteration)
