"""Particle ensembles, addressed noise and Euler-Maruyama fine propagation
(drop-in for mcparareal.particles, /root/reference/pkg/src/mcparareal/particles.py).

Ensembles live on the GPU.  ``propagate_fine`` / ``em_step`` run the sm_100a
fine-sweep kernel (``kernels.fine_sweep``); ``region_statistics`` the
restriction kernel; ``NoisePlan.normals`` the numpy-exact stream generator.
Results are bit-identical to the reference on the same inputs (cube-drift
models to within an ulp per step).
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np

from . import _lib, kernels, noise
from ._device import as_device_f64, device, require_cuda, torch
from .errors import NumericalBlowup
from .models import McKeanVlasovModel, device_model
from .state import MacroState, RegionPartition

_DOMAIN_INIT = noise.DOMAIN_INIT
_DOMAIN_DERIVED = noise.DOMAIN_DERIVED


class NoiseMode(enum.Enum):
    """FROZEN / FRESH: the reference's numpy streams (particles.py:22-71),
    reproduced bit for bit and materialised in HBM.  PHILOX / PHILOX_FRESH:
    the north star's counter-based mode -- numpy's ziggurat over
    Philox4x32-10 addressed by (particle, step, slice[, iteration]),
    generated in registers by the fine kernels (counter_noise.cuh);
    statistically equivalent to the reference's streams, not bitwise."""
    FROZEN = "frozen"
    FRESH = "fresh"
    PHILOX = "philox"
    PHILOX_FRESH = "philox-fresh"


@dataclass(frozen=True)
class NoisePlan:
    """Deterministic Brownian-increment supply keyed by (slice, step[, iteration])."""

    master_seed: int
    mode: NoiseMode = NoiseMode.FROZEN

    def __post_init__(self):
        if not 0 <= int(self.master_seed) < 2 ** 64:
            raise ValueError("master_seed must fit in an unsigned 64-bit integer")
        object.__setattr__(self, "master_seed", int(self.master_seed))
        if isinstance(self.mode, str):
            object.__setattr__(self, "mode", NoiseMode(self.mode))

    @property
    def fresh(self) -> bool:
        return self.mode in (NoiseMode.FRESH, NoiseMode.PHILOX_FRESH)

    @property
    def counter_based(self) -> bool:
        """Increments generated in registers (no materialised stream)."""
        return self.mode in (NoiseMode.PHILOX, NoiseMode.PHILOX_FRESH)

    def counter_noise(self, iteration: int = 0, slice_offset: int = 0):
        return noise.counter_noise(self.master_seed, self.fresh, iteration, slice_offset)

    def device_normals(self, slice_index: int, step_index: int, count: int, iteration: int = 0):
        if self.counter_based:
            return noise.counter_normals(self.master_seed, self.fresh, slice_index, step_index, count,
                                         iteration)[0]
        return noise.normals(self.master_seed, self.fresh, slice_index, step_index, count, iteration)

    def normals(self, slice_index: int, step_index: int, count: int, iteration: int = 0) -> np.ndarray:
        """Standard normal increments for one EM step (generated on the GPU)."""
        return self.device_normals(slice_index, step_index, count, iteration).cpu().numpy()

    def slice_noise(self, n_offset: int, n_slices: int, steps: int, count: int, iteration: int = 0, out=None):
        """Device (n_slices, steps, pitch) increments of consecutive slices."""
        if self.counter_based:
            pitch = noise.row_pitch(count)
            if out is None:
                out = torch.empty((n_slices, steps, pitch), dtype=torch.float64, device=device())
            for a in range(n_slices):
                out[a, :, :count] = noise.counter_normals(self.master_seed, self.fresh, n_offset + a, 0, count,
                                                          iteration, rows=steps)
            return out
        return noise.slice_noise(self.master_seed, n_offset, n_slices, steps, count, iteration, self.fresh, out)

    def init_rng(self) -> np.random.Generator:
        """Host generator of the initial-condition stream (for custom samplers)."""
        return np.random.Generator(np.random.Philox(np.random.SeedSequence((self.master_seed, _DOMAIN_INIT))))

    def derived_seed(self, index: int) -> int:
        ss = np.random.SeedSequence((self.master_seed, _DOMAIN_DERIVED, int(index)))
        words = ss.generate_state(2, dtype=np.uint32)
        return int(words[0]) + (int(words[1]) << 32)


@dataclass(frozen=True)
class StepConfig:
    dt: float
    steps_per_slice: int

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.steps_per_slice < 1:
            raise ValueError("steps_per_slice must be at least 1")

    @property
    def slice_length(self) -> float:
        return self.dt * self.steps_per_slice


class ParticleEnsemble:
    """Immutable snapshot of P particle positions, resident on the GPU.

    ``device_positions`` is the float64 CUDA tensor (treat as read-only);
    ``positions`` is a read-only host copy made on first access.
    """

    __slots__ = ("_dev", "_host")

    def __init__(self, positions):
        t = as_device_f64(positions)
        if t.numel() < 1:
            raise ValueError("an ensemble needs at least one particle")
        self._dev = t
        self._host = None

    @classmethod
    def _wrap(cls, tensor) -> "ParticleEnsemble":
        """Adopt a device row without copying (the engine owns the buffer)."""
        ens = cls.__new__(cls)
        ens._dev = tensor
        ens._host = None
        return ens

    @property
    def device_positions(self):
        return self._dev

    @property
    def positions(self) -> np.ndarray:
        if self._host is None:
            h = self._dev.cpu().numpy().copy()
            h.flags.writeable = False
            self._host = h
        return self._host

    @property
    def size(self) -> int:
        return self._dev.numel()

    def __len__(self) -> int:
        return self.size

    def __repr__(self) -> str:
        return f"ParticleEnsemble(P={self.size}, device={self._dev.device})"


def _blowup_check(bad, slice_index, message=None):
    b = int(bad.cpu()[0])
    if b != _lib.STAT_OK:
        if message is not None:
            raise NumericalBlowup(message)
        raise NumericalBlowup(f"non-finite particle position in slice {slice_index}, step {b}",
                              slice_index=slice_index, step_index=b)


def em_step(model: McKeanVlasovModel, ens: ParticleEnsemble, t: float, dt: float, noise_values) -> ParticleEnsemble:
    """Single Euler-Maruyama step of a whole ensemble (particles.py:134-143)."""
    desc = device_model(model)
    P = ens.size
    if isinstance(noise_values, torch.Tensor):
        xi_flat = noise_values.detach().to(device=device(), dtype=torch.float64).reshape(-1)
        shape_ok = noise_values.numel() == P and noise_values.dim() == 1
    else:
        arr = np.asarray(noise_values, dtype=float)
        shape_ok = arr.shape == (P,)
        xi_flat = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).to(device()) if shape_ok else None
    if not shape_ok:
        raise ValueError("noise must supply one increment per particle")
    xi = kernels.noise_buffer(1, 1, P)
    xi[0, 0, :P] = xi_flat
    out = torch.empty((1, P), dtype=torch.float64, device=device())
    bad = torch.empty(1, dtype=torch.int32, device=device())
    t0 = torch.tensor([float(t)], dtype=torch.float64, device=device())
    kernels.fine_sweep(desc, ens.device_positions.reshape(1, P), out, t0, 1, float(dt), xi, bad)
    _blowup_check(bad, None, "non-finite particle position after step")
    return ParticleEnsemble._wrap(out[0])


def propagate_fine(model: McKeanVlasovModel, ens: ParticleEnsemble, slice_index: int, t0: float, cfg: StepConfig,
                   plan: NoisePlan, iteration: int = 0, increments=None) -> ParticleEnsemble:
    """EM propagation of one ensemble across one slice (particles.py:146-159).

    ``increments`` (optional, (S, P) array/tensor) injects the Brownian
    increments instead of drawing the plan's addressed stream."""
    desc = device_model(model)
    P, S = ens.size, cfg.steps_per_slice
    if increments is None and plan.counter_based:
        out = torch.empty((1, P), dtype=torch.float64, device=device())
        bad = torch.empty(1, dtype=torch.int32, device=device())
        t0d = torch.tensor([float(t0)], dtype=torch.float64, device=device())
        kernels.fine_sweep(desc, ens.device_positions.reshape(1, P), out, t0d, S, cfg.dt, None, bad,
                           counter=plan.counter_noise(iteration, slice_index))
        _blowup_check(bad, slice_index)
        return ParticleEnsemble._wrap(out[0])
    if increments is None:
        xi = plan.slice_noise(slice_index, 1, S, P, iteration)
    else:
        xi = kernels.noise_buffer(1, S, P)
        inc = increments if isinstance(increments, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(increments, dtype=float)))
        if tuple(inc.shape) != (S, P):
            raise ValueError("increments must have shape (steps_per_slice, P)")
        xi[0, :, :P] = inc.to(device=device(), dtype=torch.float64)
    out = torch.empty((1, P), dtype=torch.float64, device=device())
    bad = torch.empty(1, dtype=torch.int32, device=device())
    t0d = torch.tensor([float(t0)], dtype=torch.float64, device=device())
    kernels.fine_sweep(desc, ens.device_positions.reshape(1, P), out, t0d, S, cfg.dt, xi, bad)
    _blowup_check(bad, slice_index)
    return ParticleEnsemble._wrap(out[0])


def _restrict_one(ens: ParticleEnsemble, partition: RegionPartition):
    part = partition.descriptor()
    I = partition.n_regions
    stats = torch.empty((1, 3 * I), dtype=torch.float64, device=device())
    counts = torch.empty((1, I), dtype=torch.int64, device=device())
    kernels.restrict(part, ens.device_positions.reshape(1, -1), stats, counts)
    return stats, counts


def region_statistics(ens: ParticleEnsemble, partition: RegionPartition) -> MacroState:
    """Per-region mean, population variance and fraction (particles.py:176-205)."""
    stats, counts = _restrict_one(ens, partition)
    c = counts.cpu().numpy()[0]
    return MacroState.from_packed(stats.cpu().numpy()[0], partition.n_regions, tuple(c < 2))


def empirical_mean(ens: ParticleEnsemble) -> float:
    return region_statistics(ens, RegionPartition()).means[0]


def empirical_variance(ens: ParticleEnsemble) -> float:
    """Population variance (1/P normalisation)."""
    return region_statistics(ens, RegionPartition()).variances[0]


def estimate_qoi(ens: ParticleEnsemble, phi) -> float:
    """Monte Carlo estimate of E[phi(X)] (phi is an arbitrary host callable)."""
    return float(np.mean(phi(ens.positions)))


def sample_initial(dist, plan: NoisePlan, count: int) -> ParticleEnsemble:
    """Initial ensemble from the plan's dedicated stream (particles.py:208-210).
    Normal and Dirac laws are sampled on the GPU; custom samplers are user
    host code and run on the host before the upload."""
    require_cuda()
    if count < 1:
        raise ValueError("particle count must be at least 1")
    if dist.kind == "normal":
        return ParticleEnsemble._wrap(noise.initial_normal(plan.master_seed, dist.mean, math.sqrt(dist.variance),
                                                           count))
    if dist.kind == "dirac":
        return ParticleEnsemble._wrap(torch.full((count,), float(dist.mean), dtype=torch.float64, device=device()))
    return ParticleEnsemble(dist.sample(plan.init_rng(), count))
