"""Multi-GPU mM-Parareal: slices sharded across ranks (one process per GPU).

Partition: rank r owns the contiguous slices [r*Ng, (r+1)*Ng).
Per iteration the only traffic is
  1. an all-gather of the owned slices' restricted fine moments
     (Ng * 3I float64 per rank -- the coarse row needs all of them), and
  2. a ring shift of ONE ensemble: rank r's last matched ensemble u_{b} is
     the next iteration's input of rank r+1's first slice (engine.py:232-235).
Every rank integrates the (cheap, serial) coarse row redundantly, so all
ranks hold bit-identical macro rows; increments are generated per rank for
its own global slice indices, so the sharded run is bit-identical to the
single-GPU run of the same N.  Micro statistics and status arrays are
gathered once, after the last iteration.

The orchestration is written against a small backend interface so the same
code runs the sm_100a kernels (``GpuBackend``, NCCL) and, in the CPU tests,
the oracle (gloo).  Production uses ``GpuBackend`` only.
"""

from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, kernels
from .engine import PararealConfig, PararealTrace, _build_trace, _raise_first_error, _StageTimer
from .models import device_model
from .moments import device_ode
from .noise import row_pitch, slice_noise
from .particles import NoisePlan, ParticleEnsemble, sample_initial
from .rk54 import integrator_descriptor
from .state import SINGLE_REGION


class GpuBackend:
    """sm_100a kernels on the rank's current CUDA device."""

    def __init__(self, model, coarse, cfg: PararealConfig):
        self.model_d = device_model(model)
        self.ode_d, self.ode_model_d = device_ode(coarse)
        self.integ_d = integrator_descriptor(cfg.integrator)
        self.part_d = cfg.partition.descriptor()
        self.device = torch.device("cuda", torch.cuda.current_device())

    def empty(self, shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def noise(self, seed, n_offset, n_slices, steps, P, iteration, fresh, out):
        slice_noise(seed, n_offset, n_slices, steps, P, iteration, fresh, out=out)

    @staticmethod
    def _noise_args(xi):
        """xi is an increment buffer, or a CounterNoise (NoiseMode.PHILOX*:
        increments generated in registers)."""
        return (None, xi) if isinstance(xi, _lib.CounterNoise) else (xi, None)

    def fine(self, x_in, x_out, t0, steps, dt, xi, bad):
        xi, counter = self._noise_args(xi)
        kernels.fine_sweep(self.model_d, x_in, x_out, t0, steps, dt, xi, bad, counter=counter)

    def fine_restrict(self, x_in, x_out, t0, steps, dt, xi, bad, stats, counts):
        """Sweep plus the single-region restriction of its outputs, fused
        (MEAN_OF_F models; the restriction kernel otherwise)."""
        if self.model_d.stat_kind == _lib.STAT_MEAN_OF_F:
            xi, counter = self._noise_args(xi)
            kernels.fine_sweep(self.model_d, x_in, x_out, t0, steps, dt, xi, bad, stats=stats, counts=counts,
                               counter=counter)
        else:
            kernels.fine_sweep(self.model_d, x_in, x_out, t0, steps, dt, xi, bad)
            kernels.restrict(SINGLE_REGION.descriptor(), x_out, stats, counts)

    def restrict(self, x, stats, counts, scratch):
        kernels.restrict(self.part_d, x, stats, counts, scratch)

    def restrict_scratch(self, n_ens, P, I):
        return kernels.restrict_scratch(n_ens, P, I)

    def coarse_row(self, times, iteration, rho0, fine_stats, cache_in, macro_out, cache_out, raw_out, status,
                   skip_until):
        kernels.coarse_row(self.ode_d, self.ode_model_d, self.integ_d, times, iteration, rho0, fine_stats,
                           cache_in, macro_out, cache_out, raw_out, status, skip_until)

    def match(self, targets, cur, counts, src, out, policy, status):
        kernels.match(self.part_d, targets, cur, counts, src, out, policy, status)

    def restrict_single(self, x, stats, counts):
        kernels.restrict(SINGLE_REGION.descriptor(), x, stats, counts)

    def w1_rows(self, a, b):
        """Per-row W1 = mean|sort(a) - sort(b)| (engine.py:244-253), device tensor."""
        return kernels.mean_abs_diff(kernels.sort_rows(a), kernels.sort_rows(b))

    def synchronize(self):
        torch.cuda.synchronize()


class TorchComm:
    """torch.distributed collectives (NCCL on GPU ranks, gloo in CPU tests)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_rows(self, local):
        out = torch.empty((self.world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)
        return out

    def shift_right(self, send, recv):
        """rank r -> r+1; rank 0 receives nothing, the last rank sends nothing."""
        ops = []
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, send.contiguous(), self.rank + 1, group=self.group))
        if self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, recv, self.rank - 1, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def _device(self):
        return "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"

    def all_min_int(self, value: int) -> int:
        t = torch.tensor([int(value)], dtype=torch.int64, device=self._device())
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def all_gather_bytes(self, payload: bytes) -> list:
        """Fixed-size byte strings from every rank (IPC handles)."""
        t = torch.tensor(list(payload), dtype=torch.uint8, device=self._device()).reshape(1, -1)
        out = self.all_gather_rows(t).cpu().numpy()
        return [bytes(row) for row in out]

    def all_max(self, value: float) -> float:
        t = torch.tensor([value], dtype=torch.float64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


_PIPE_STATE: dict = {}
last_run_info: dict = {"pipeline": False}


def _pipeline_sharded_ok(be, cfg: PararealConfig, plan: NoisePlan, comm) -> bool:
    """Every rank agrees to run the multi-GPU iteration pipeline: GPU
    backend, an instantiated single-region configuration (the two-region
    units run on one rank only), FROZEN noise, no Wasserstein stop, N
    divisible by the world size, at most 8 ranks."""
    if (not isinstance(be, GpuBackend) or os.environ.get("MMPR_PIPELINE", "1") == "0"
            or not hasattr(comm, "all_min_int")):
        return False
    # opt-in above one rank: the cross-GPU form is verified by the one-GPU
    # emulation of its scheduling only (Multi-GPU)
    if comm.world > 1 and os.environ.get("MMPR_SHARDED_PIPELINE", "0") != "1":
        return False
    G = comm.world
    ok = (G <= 8 and cfg.n_slices % G == 0 and cfg.iterations >= 1 and not plan.fresh and not plan.counter_based
          and cfg.stop_wasserstein_tol is None and cfg.partition.n_regions == 1
          and kernels.pipeline_supported(be.model_d, be.ode_d, be.ode_model_d, be.integ_d, cfg.particles,
                                            n_ranks=G))
    return comm.all_min_int(1 if ok else 0) == 1


def _pipeline_state(be, cfg: PararealConfig, comm):
    """Per-configuration rank buffers with an IPC-exportable exchange block,
    and the previous rank's exchange block mapped into this process (the
    only peer memory a rank touches: it reads rank r-1's outputs for its first
    slice and adds its "consumed" signals to rank r-1's flags)."""
    from . import sharded_pipeline as SP
    R, G = comm.rank, comm.world
    key = (cfg.n_slices, cfg.iterations, cfg.particles, cfg.step.steps_per_slice, cfg.retain_snapshots, R, G,
           torch.cuda.current_device())
    st = _PIPE_STATE.get(key)
    if st is not None:
        return st
    for old in list(_PIPE_STATE.values()):  # one configuration at a time
        old["rb"].free()
    _PIPE_STATE.clear()
    rb = SP.RankBuffers(R, G, cfg.n_slices, cfg.iterations, cfg.particles, cfg.step.steps_per_slice,
                        cfg.retain_snapshots, raw_exchange=G > 1)
    prev_base = None
    if G > 1:
        handle = (ctypes.c_ubyte * 64)()
        _lib.call("mmpr_ipc_handle", ctypes.c_void_p(rb.block.ptr), handle)
        handles = comm.all_gather_bytes(bytes(handle))
        ok = 1
        if R > 0:
            ptr = ctypes.c_void_p()
            st_open = _lib.load().mmpr_ipc_open((ctypes.c_ubyte * 64).from_buffer_copy(handles[R - 1]),
                                                ctypes.byref(ptr))
            ok = 1 if st_open == 0 else 0
            prev_base = int(ptr.value) if ok else None
        if comm.all_min_int(ok) != 1:
            if prev_base is not None:
                _lib.load().mmpr_ipc_close(ctypes.c_void_p(prev_base))
            rb.free()
            return None
    st = {"rb": rb, "prev_base": prev_base}
    _PIPE_STATE[key] = st
    return st


def _run_pipeline_sharded(be, initial, cfg: PararealConfig, plan: NoisePlan, comm, reuse: bool,
                          record_timings: bool, st) -> PararealTrace:
    """Iterations 1..K as one persistent kernel per GPU; the first slice of
    rank r waits on rank r-1's flags and reads its last fine output, its
    restriction and macro value through the mapped exchange block
    (mmpr_parareal_pipeline_ranks).  One all-gather at the end merges the
    per-slice trace arrays."""
    from . import sharded_pipeline as SP
    R, G = comm.rank, comm.world
    N, K, P, S = cfg.n_slices, cfg.iterations, cfg.particles, cfg.step.steps_per_slice
    Ng = N // G
    rb = st["rb"]
    times = tuple(cfg.t_start + n * cfg.slice_length for n in range(N + 1))
    times_d = torch.tensor(times, dtype=torch.float64, device=be.device)
    if isinstance(initial, ParticleEnsemble):
        x0 = initial.device_positions.to(be.device)
    else:
        x0 = sample_initial(initial, plan, P).device_positions
    timer = _StageTimer(record_timings)
    ev = timer.start()
    rb.prologue(be.ode_d, be.ode_model_d, be.integ_d, times_d, x0, plan.master_seed)
    timer.stop("prologue", ev)
    own = rb.io(times_d)
    ios = [own] * G
    if R > 0:
        ios[R - 1] = rb.peer_io(st["prev_base"], own)
    rb.epoch += 1
    ev = timer.start()
    SP.launch(be.model_d, be.ode_d, be.ode_model_d, be.integ_d, cfg.step.dt, S, reuse, ios, R, 1, rb.epoch,
              False, G > 1, N, K, P)
    timer.stop("iterations", ev)
    # ---- one gather of the per-slice arrays, merged by ownership -------------------
    names = (("macro", "boundary"), ("micro", "boundary"), ("micro_counts", "boundary"), ("fine_stats", "slice"),
             ("fine_counts", "slice"), ("bad", "slice"), ("raw", "shifted"), ("coarse_status", "shifted"),
             ("match_status", "shifted"))
    h = {}
    by_dtype = {}
    for name, kind in names:
        by_dtype.setdefault(getattr(rb, name).dtype, []).append((name, kind))
    for dtype, items in by_dtype.items():  # one gather and one read-back per dtype
        flat = torch.cat([getattr(rb, name).reshape(-1) for name, _ in items]).reshape(1, -1)
        rows = (comm.all_gather_rows(flat) if G > 1 else flat).cpu().numpy()
        off = 0
        for name, kind in items:
            shape = tuple(getattr(rb, name).shape)
            size = int(np.prod(shape))
            parts = [rows[g, off:off + size].reshape(shape) for g in range(G)]
            h[name] = SP.merge_rows(parts, Ng, G, N, kind)
            off += size
    h["rho0"] = rb.rho0.cpu().numpy()
    h["counts0"] = rb.counts0.cpu().numpy()
    _raise_first_error(h, N, K, 1)
    trace = _build_trace(h, None, dataclasses.replace(cfg, retain_snapshots=False), plan, times, K, 1,
                         _StageTimer(False), None)
    own_b = SP.owned_boundaries(R, Ng, G, N)
    if cfg.retain_snapshots:
        trace.snapshots = [[ParticleEnsemble._wrap(rb.snap[k, n]) for n in own_b] for k in range(K + 1)]
    trace.timings = timer.resolve()
    trace.timings["slice_offset"] = own_b.start
    trace.timings["slices_per_rank"] = Ng
    trace.d2h_bytes = int(sum(v.nbytes for v in h.values()))
    return trace


def run_micro_macro_sharded(model, coarse, initial, cfg: PararealConfig, plan: NoisePlan, comm=None,
                            backend=None, reuse_converged_coarse: bool = True,
                            record_timings: bool = True) -> PararealTrace:
    """mM-Parareal over ``comm.world`` ranks; every rank returns the full
    macro/micro trace, snapshots hold the rank's own slices only
    (``trace.snapshots[k][m]`` is global slice boundary ``offset + m``).

    With MMPR_SHARDED_PIPELINE=1 (and always at world size 1),
    configurations the iteration pipeline covers run it on every GPU
    (cross-rank dependencies through peer memory, one gather at the end);
    otherwise the per-iteration kernels run with NCCL collectives."""
    comm = comm if comm is not None else TorchComm()
    reuse_converged_coarse = reuse_converged_coarse and not plan.fresh  # see engine.run_micro_macro
    be = backend if backend is not None else GpuBackend(model, coarse, cfg)
    if _pipeline_sharded_ok(be, cfg, plan, comm):
        st = _pipeline_state(be, cfg, comm)
        if st is not None:
            last_run_info["pipeline"] = True
            return _run_pipeline_sharded(be, initial, cfg, plan, comm, reuse_converged_coarse, record_timings, st)
    last_run_info["pipeline"] = False
    R, G = comm.rank, comm.world
    N, K, P, S, I = cfg.n_slices, cfg.iterations, cfg.particles, cfg.step.steps_per_slice, cfg.partition.n_regions
    if N % G:
        raise ValueError(f"n_slices={N} must be divisible by the world size {G}")
    Ng = N // G
    a = R * Ng
    nv = 3 * I
    dt = cfg.step.dt
    times = tuple(cfg.t_start + n * cfg.slice_length for n in range(N + 1))
    times_d = torch.tensor(times, dtype=torch.float64, device=be.device)
    retain = cfg.retain_snapshots
    i32, i64 = torch.int32, torch.int64

    if isinstance(initial, ParticleEnsemble):
        x0 = initial.device_positions.to(be.device).reshape(1, P)
    elif hasattr(initial, "kind") and be.device.type == "cuda":
        x0 = sample_initial(initial, plan, P).device_positions.reshape(1, P)
    else:
        x0 = torch.as_tensor(np.asarray(initial.sample(plan.init_rng(), P), dtype=float)).to(be.device).reshape(1, P)

    snap = be.empty((K + 1 if retain else 2, Ng + 1, P))
    fine = be.empty((Ng, P))
    counter_mode = getattr(plan, "counter_based", False)
    xi = be.empty((1, 1, 2) if counter_mode else (Ng, S, row_pitch(P)))
    macro = be.empty((K + 1, N + 1, nv))
    cache = be.empty((K + 1, N, nv))
    raw = be.empty((max(K, 1), N, nv))
    fine_all = be.empty((max(K, 1), N, nv))
    fine_local = be.empty((Ng, nv))
    fine_counts = be.empty((Ng, I), i64)
    micro_local = be.empty((K + 1, Ng + 1, nv))
    micro_counts_local = be.empty((K + 1, Ng + 1, I), i64)
    bad_local = torch.full((max(K, 1), Ng), _lib.STAT_OK, dtype=i32, device=be.device)
    coarse_status = torch.full((K + 1, N), _lib.STAT_OK, dtype=i32, device=be.device)
    match_local = torch.full((K + 1, Ng), _lib.STAT_OK, dtype=i32, device=be.device)
    lift_first = torch.full((1,), _lib.STAT_OK, dtype=i32, device=be.device)
    rho0 = be.empty((1, nv))
    counts0 = be.empty((1, I), i64)
    scratch = be.empty((be.restrict_scratch(Ng + 1, P, I),)) if I > 1 else None

    def sn(k):
        return snap[k if retain else k % 2]

    # iteration 0: redundant coarse cascade; each rank lifts its own boundaries
    be.restrict(x0, rho0, counts0, scratch)
    be.coarse_row(times_d, 0, rho0, None, None, macro[0], cache[0], None, coarse_status[0], 0)
    be.match(macro[0, a + 1:a + Ng + 1], rho0, counts0, x0, sn(0)[1:], 1, match_local[0])
    if a == 0:
        sn(0)[0].copy_(x0[0])
    else:
        be.match(macro[0, a:a + 1], rho0, counts0, x0, sn(0)[0:1], 1, lift_first)
    be.restrict(sn(0), micro_local[0], micro_counts_local[0], scratch)
    if not plan.fresh and not counter_mode:
        be.noise(plan.master_seed, a, Ng, S, P, 0, False, xi)

    timer = _StageTimer(record_timings and be.device.type == "cuda")
    stopped_at = None
    done = 0
    for k in range(K):
        if plan.fresh and not counter_mode:
            be.noise(plan.master_seed, a, Ng, S, P, k, True, xi)
        xk = plan.counter_noise(k, a) if counter_mode else xi
        cur, nxt = sn(k), sn(k + 1)
        ev = timer.start()
        if I == 1:
            be.fine_restrict(cur[:Ng], fine, times_d[a:a + Ng], S, dt, xk, bad_local[k], fine_local, fine_counts)
            timer.stop("fine", ev)
        else:
            be.fine(cur[:Ng], fine, times_d[a:a + Ng], S, dt, xk, bad_local[k])
            timer.stop("fine", ev)
            be.restrict(fine, fine_local, fine_counts, scratch)
        fine_all[k].copy_(comm.all_gather_rows(fine_local))
        be.coarse_row(times_d, k + 1, rho0, fine_all[k], cache[k], macro[k + 1], cache[k + 1], raw[k],
                      coarse_status[k + 1], (k + 1) if reuse_converged_coarse else 0)
        be.match(macro[k + 1, a + 1:a + Ng + 1], fine_local, fine_counts, fine, nxt[1:], 0, match_local[k + 1])
        if a == 0:
            nxt[0].copy_(x0[0])
        comm.shift_right(nxt[Ng], nxt[0])
        be.restrict(nxt, micro_local[k + 1], micro_counts_local[k + 1], scratch)
        done = k + 1
        if cfg.stop_wasserstein_tol is not None:
            delta = comm.all_max(float(be.w1_rows(nxt[1:], cur[1:]).max()))
            if delta <= cfg.stop_wasserstein_tol:
                stopped_at = k + 1
                break

    # gather micro statistics and per-slice statuses once
    Kd = done
    micro = be.empty((Kd + 1, N + 1, nv))
    micro_counts = be.empty((Kd + 1, N + 1, I), i64)
    for k in range(Kd + 1):
        rows = comm.all_gather_rows(micro_local[k, 1:])
        micro[k, 1:].copy_(rows)
        micro[k, 0].copy_(rho0[0])
        micro_counts[k, 1:].copy_(comm.all_gather_rows(micro_counts_local[k, 1:]))
        micro_counts[k, 0].copy_(counts0[0])
    bad = comm.all_gather_rows(bad_local.t().contiguous()).t() if K > 0 else bad_local
    match_status = comm.all_gather_rows(match_local.t().contiguous()).t()
    be.synchronize()
    h = {"macro": macro[:Kd + 1].cpu().numpy(), "micro": micro.cpu().numpy(),
         "micro_counts": micro_counts.cpu().numpy(), "fine_stats": fine_all[:max(Kd, 1)].cpu().numpy(),
         "raw": raw[:max(Kd, 1)].cpu().numpy(), "bad": bad.cpu().numpy(),
         "coarse_status": coarse_status.cpu().numpy(), "match_status": match_status.cpu().numpy(),
         "rho0": rho0.cpu().numpy(), "counts0": counts0.cpu().numpy()}
    _raise_first_error(h, N, Kd, I)

    trace = _build_trace(h, None, dataclasses.replace(cfg, retain_snapshots=False), plan, times, Kd, I,
                         _StageTimer(False), stopped_at)
    if retain:
        trace.snapshots = [[ParticleEnsemble._wrap(snap[k, m]) for m in range(Ng + 1)] for k in range(Kd + 1)]
    trace.timings = timer.resolve()
    trace.timings["slice_offset"] = a
    trace.timings["slices_per_rank"] = Ng
    trace.d2h_bytes = int(sum(v.nbytes for v in h.values()))
    return trace


