"""Restriction / matching / lifting (drop-in for mcparareal.coupling,
/root/reference/pkg/src/mcparareal/coupling.py:26-95), on the GPU.

``match`` consumes the restriction of its source ensemble computed by the
same kernel as ``restrict``, so ``match(restrict(u), u)`` keeps every bit of
``u`` (the identity shortcut, coupling.py:82-83) exactly as the reference.
"""

from __future__ import annotations

import logging

from . import kernels
from ._device import device, torch
from .errors import DegenerateMatch
from .particles import ParticleEnsemble, _restrict_one, region_statistics
from .state import SINGLE_REGION, MacroState, RegionPartition

logger = logging.getLogger("mcparareal.coupling")

POLICIES = {"raise": 0, "collapse": 1}


def restrict(ens: ParticleEnsemble, partition: RegionPartition = SINGLE_REGION) -> MacroState:
    """Per-region mean, population variance and particle fraction."""
    return region_statistics(ens, partition)


def match(target: MacroState, ens: ParticleEnsemble, partition: RegionPartition = SINGLE_REGION,
          degenerate_policy: str = "raise") -> ParticleEnsemble:
    """Affinely map each region's particles onto the target mean/variance."""
    if degenerate_policy not in POLICIES:
        raise ValueError(f"unknown degenerate policy {degenerate_policy!r}")
    if target.n_regions != partition.n_regions:
        raise ValueError(f"target has {target.n_regions} regions, partition has {partition.n_regions}")
    for i, v in enumerate(target.variances):
        if v < 0.0:
            logger.warning("match: clamping negative target variance %.3e in region %d", v, i)
    P = ens.size
    part = partition.descriptor()
    cur, counts = _restrict_one(ens, partition)
    tgt = torch.from_numpy(target.packed().reshape(1, -1)).to(device())
    out = torch.empty((1, P), dtype=torch.float64, device=device())
    status = torch.empty(1, dtype=torch.int32, device=device())
    kernels.match(part, tgt, cur, counts, ens.device_positions.reshape(1, P), out, POLICIES[degenerate_policy],
                  status)
    region = int(status.cpu()[0])
    if region >= 0:
        var_t = max(target.variances[region], 0.0)
        raise DegenerateMatch(f"region {region}: cannot scale a zero-variance group to variance {var_t:.3e}",
                              region=region)
    return ParticleEnsemble._wrap(out[0])


def lift(target: MacroState, initial: ParticleEnsemble, partition: RegionPartition = SINGLE_REGION,
         degenerate_policy: str = "raise") -> ParticleEnsemble:
    """Micro state with the initial ensemble's shape and the target's moments."""
    return match(target, initial, partition, degenerate_policy)


def restrict_batch(ensembles, partition: RegionPartition = SINGLE_REGION) -> list[MacroState]:
    """Restriction of several equal-size ensembles in one launch."""
    x = torch.stack([e.device_positions for e in ensembles])
    I = partition.n_regions
    stats = torch.empty((x.shape[0], 3 * I), dtype=torch.float64, device=device())
    counts = torch.empty((x.shape[0], I), dtype=torch.int64, device=device())
    kernels.restrict(partition.descriptor(), x, stats, counts)
    s, c = stats.cpu().numpy(), counts.cpu().numpy()
    return [MacroState.from_packed(s[e], I, tuple(c[e] < 2)) for e in range(x.shape[0])]

