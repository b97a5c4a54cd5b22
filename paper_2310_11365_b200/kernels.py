"""Thin, shape-checked wrappers of the libmmpr entry points over torch
device tensors.  Stream-ordered; nothing here synchronises the host.

All ensembles are float64 rows: a batch of E ensembles of P particles is a
(E, P) tensor (row pitch = stride(0)); packed macro states are (E, 3I).
"""

from __future__ import annotations

import ctypes
import math

from . import _lib
from ._device import device, require_cuda, torch
from .noise import row_pitch


def _f64(t, name):
    if t.dtype != torch.float64 or t.device.type != "cuda":
        raise ValueError(f"{name} must be a float64 CUDA tensor")


def _rows(t, name):
    _f64(t, name)
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be a 2-D row-contiguous tensor")
    return t.stride(0)


def fine_sweep(model: _lib.Model, x_in, x_out, t0, steps: int, dt: float, xi, bad_step, final_mean=None,
               stats=None, counts=None, stream=None, counter: _lib.CounterNoise | None = None, times=None) -> None:
    """EM over ``steps`` steps for every row of x_in (E, P) -> x_out (E, P).
    xi: (E, steps, pitch) increments; t0: (E,) float64; bad_step: (E,) int32.
    stats (E, 3) / counts (E, 1): single-region restriction of x_out fused
    into the sweep (MEAN_OF_F models).  ``counter`` (NoiseMode.PHILOX*):
    increments generated in registers by counter-based Philox; xi unused.
    ``times`` (E, 2) int64: globaltimer ns at each slice's start and end."""
    require_cuda()
    if times is not None:
        if times.dtype != torch.int64 or tuple(times.shape) != (x_in.shape[0], 2) or not times.is_contiguous():
            raise ValueError("times must be contiguous int64 (E, 2)")
        _lib.call("mmpr_set_fine_times", times.data_ptr())
        try:
            fine_sweep(model, x_in, x_out, t0, steps, dt, xi, bad_step, final_mean, stats, counts, stream, counter)
        finally:
            _lib.call("mmpr_set_fine_times", None)
        return
    E, P = x_in.shape
    in_pitch = _rows(x_in, "x_in")
    out_pitch = _rows(x_out, "x_out")
    if x_out.shape != x_in.shape:
        raise ValueError("x_out must match x_in")
    if counter is not None:
        if model.stat_kind != _lib.STAT_MEAN_OF_F:
            raise _lib.MmprError("counter-based noise runs the MEAN_OF_F fine kernels only")
        if bad_step.dtype != torch.int32 or bad_step.numel() < E:
            raise ValueError("bad_step must be int32 (E,)")
        if stats is not None:
            _f64(stats, "stats")
            if stats.numel() < 3 * E or not stats.is_contiguous():
                raise ValueError("stats must be contiguous float64 (E, 3)")
        _lib.call("mmpr_fine_sweep_counter", ctypes.byref(model), int(E), int(P), int(steps), float(dt),
                  float(math.sqrt(dt)), t0.data_ptr(), x_in.data_ptr(), int(in_pitch), x_out.data_ptr(),
                  int(out_pitch), ctypes.byref(counter), bad_step.data_ptr(), _lib.ptr(stats), _lib.ptr(counts),
                  _lib.stream_handle(stream))
        return
    _f64(xi, "xi")
    if xi.dim() != 3 or xi.shape[0] != E or xi.shape[1] < steps or xi.stride(2) != 1:
        raise ValueError("xi must be (E, >=steps, pitch)")
    pitch = xi.stride(1)
    if pitch < P or pitch % 2:
        raise ValueError("xi row pitch must be even and >= P")
    if bad_step.dtype != torch.int32 or bad_step.numel() < E:
        raise ValueError("bad_step must be int32 (E,)")
    if model.stat_kind != _lib.STAT_MEAN_OF_F:  # plane rotator / Burgers
        if final_mean is not None:
            raise ValueError("final_mean is defined for MEAN_OF_F models only")
        nbytes = ctypes.c_uint64(0)
        args = (ctypes.byref(model), int(E), int(P), int(steps), float(dt), float(math.sqrt(dt)), x_in.data_ptr(),
                int(in_pitch), x_out.data_ptr(), int(out_pitch), xi.data_ptr(), int(xi.stride(0)), int(pitch),
                bad_step.data_ptr())
        _lib.call("mmpr_fine_sweep_stepwise", *args, None, ctypes.byref(nbytes), _lib.stream_handle(stream))
        work = torch.empty(max(1, nbytes.value), dtype=torch.uint8, device=x_in.device)
        _lib.call("mmpr_fine_sweep_stepwise", *args, work.data_ptr(), ctypes.byref(nbytes),
                  _lib.stream_handle(stream))
        if stats is not None:
            restrict(_single_region(), x_out, stats, counts)
        return
    if stats is not None:
        _f64(stats, "stats")
        if stats.numel() < 3 * E or not stats.is_contiguous():
            raise ValueError("stats must be contiguous float64 (E, 3)")
        if counts is not None and (counts.dtype != torch.int64 or counts.numel() < E):
            raise ValueError("counts must be int64 (E, 1)")
        _lib.call("mmpr_fine_sweep_restrict", ctypes.byref(model), int(E), int(P), int(steps), float(dt),
                  float(math.sqrt(dt)), t0.data_ptr(), x_in.data_ptr(), int(in_pitch), x_out.data_ptr(),
                  int(out_pitch), xi.data_ptr(), int(xi.stride(0)), int(pitch), bad_step.data_ptr(),
                  stats.data_ptr(), _lib.ptr(counts), _lib.stream_handle(stream))
        return
    _lib.call("mmpr_fine_sweep", ctypes.byref(model), int(E), int(P), int(steps), float(dt),
              float(math.sqrt(dt)), t0.data_ptr(), x_in.data_ptr(), int(in_pitch), x_out.data_ptr(),
              int(out_pitch), xi.data_ptr(), int(xi.stride(0)), int(pitch), bad_step.data_ptr(),
              _lib.ptr(final_mean), _lib.stream_handle(stream))


def restrict_scratch(n_ens: int, P: int, n_regions: int) -> int:
    """Doubles of scratch mmpr_restrict needs (0 for one region)."""
    return int(_lib.load().mmpr_restrict_scratch_doubles(int(n_ens), int(P), int(n_regions)))


def restrict(part: _lib.Partition, x, stats, counts, scratch=None, stream=None) -> None:
    """stats (E, 3I) and counts (E, I) int64 of every row of x (E, P)."""
    require_cuda()
    E, P = x.shape
    pitch = _rows(x, "x")
    I = part.n_regions
    _f64(stats, "stats")
    if stats.shape != (E, 3 * I) or not stats.is_contiguous():
        raise ValueError("stats must be contiguous (E, 3I)")
    if counts.dtype != torch.int64 or counts.shape != (E, I) or not counts.is_contiguous():
        raise ValueError("counts must be contiguous int64 (E, I)")
    if I > 1:
        need = restrict_scratch(E, P, I)
        if scratch is None:
            scratch = torch.empty(need, dtype=torch.float64, device=device())
        elif scratch.numel() < need:
            raise ValueError("scratch too small")
    _lib.call("mmpr_restrict", ctypes.byref(part), int(E), int(P), x.data_ptr(), int(pitch), stats.data_ptr(),
              counts.data_ptr(), _lib.ptr(scratch) if I > 1 else None, _lib.stream_handle(stream))


def match(part: _lib.Partition, targets, cur_stats, cur_counts, x_src, x_out, policy: int, status, clamped=None,
          stream=None) -> None:
    """Affine per-region match of E ensembles.  x_src may have one row (shared
    source, e.g. lift from ens0), as may cur_stats / cur_counts."""
    require_cuda()
    E, P = x_out.shape
    out_pitch = _rows(x_out, "x_out")
    src_pitch = _rows(x_src, "x_src") if x_src.shape[0] > 1 else 0
    if x_src.shape[1] != P or x_src.shape[0] not in (1, E):
        raise ValueError("x_src must be (1 or E, P)")
    I = part.n_regions
    for t, name in ((targets, "targets"), (cur_stats, "cur_stats")):
        _f64(t, name)
        if t.dim() != 2 or t.shape[1] != 3 * I or t.stride(1) != 1 or t.shape[0] not in (1, E):
            raise ValueError(f"{name} must be (1 or E, 3I)")
    tgt_stride = targets.stride(0) if targets.shape[0] > 1 else 0
    cur_stride = cur_stats.stride(0) if cur_stats.shape[0] > 1 else 0
    if cur_counts.dtype != torch.int64 or cur_counts.shape[1] != I or cur_counts.shape[0] not in (1, E):
        raise ValueError("cur_counts must be int64 (1 or E, I)")
    cnt_stride = cur_counts.stride(0) if cur_counts.shape[0] > 1 else 0
    if status.dtype != torch.int32 or status.numel() < E:
        raise ValueError("status must be int32 (E,)")
    _lib.call("mmpr_match", ctypes.byref(part), int(E), int(P), targets.data_ptr(), int(tgt_stride),
              cur_stats.data_ptr(), int(cur_stride), cur_counts.data_ptr(), int(cnt_stride), x_src.data_ptr(),
              int(src_pitch), x_out.data_ptr(), int(out_pitch), int(policy), status.data_ptr(),
              _lib.ptr(clamped), _lib.stream_handle(stream))


def match_restrict_regions(part: _lib.Partition, targets, cur_stats, cur_counts, x_src, x_out, policy: int, status,
                           stats, counts, scratch, clamped=None, stream=None) -> None:
    """Per-region match of E ensembles and the per-region restriction of the
    matched ensembles in one pass (one cluster per ensemble; the separate
    passes beyond one cluster).  stats (E, 3I), counts (E, I) int64,
    scratch: >= E*I*P doubles."""
    require_cuda()
    E, P = x_out.shape
    out_pitch = _rows(x_out, "x_out")
    src_pitch = _rows(x_src, "x_src") if x_src.shape[0] > 1 else 0
    if x_src.shape[1] != P or x_src.shape[0] not in (1, E):
        raise ValueError("x_src must be (1 or E, P)")
    I = part.n_regions
    for t, name in ((targets, "targets"), (cur_stats, "cur_stats")):
        _f64(t, name)
        if t.dim() != 2 or t.shape[1] != 3 * I or t.stride(1) != 1 or t.shape[0] not in (1, E):
            raise ValueError(f"{name} must be (1 or E, 3I)")
    tgt_stride = targets.stride(0) if targets.shape[0] > 1 else 0
    cur_stride = cur_stats.stride(0) if cur_stats.shape[0] > 1 else 0
    if cur_counts.dtype != torch.int64 or cur_counts.shape[1] != I or cur_counts.shape[0] not in (1, E):
        raise ValueError("cur_counts must be int64 (1 or E, I)")
    cnt_stride = cur_counts.stride(0) if cur_counts.shape[0] > 1 else 0
    if status.dtype != torch.int32 or status.numel() < E:
        raise ValueError("status must be int32 (E,)")
    _f64(stats, "stats")
    if stats.shape != (E, 3 * I) or not stats.is_contiguous():
        raise ValueError("stats must be contiguous float64 (E, 3I)")
    if counts.dtype != torch.int64 or tuple(counts.shape) != (E, I) or not counts.is_contiguous():
        raise ValueError("counts must be contiguous int64 (E, I)")
    if scratch is None or scratch.numel() < E * I * P:
        raise ValueError("scratch must hold E*I*P doubles")
    _lib.call("mmpr_match_restrict_regions", ctypes.byref(part), int(E), int(P), targets.data_ptr(), int(tgt_stride),
              cur_stats.data_ptr(), int(cur_stride), cur_counts.data_ptr(), int(cnt_stride), x_src.data_ptr(),
              int(src_pitch), x_out.data_ptr(), int(out_pitch), int(policy), status.data_ptr(), _lib.ptr(clamped),
              stats.data_ptr(), counts.data_ptr(), scratch.data_ptr(), _lib.stream_handle(stream))


def match_restrict(targets, cur_stats, cur_counts, x_src, x_out, policy: int, status, stats, counts=None,
                   clamped=None, stream=None) -> None:
    """Single-region match of E ensembles and the restriction of the matched
    ensembles in one pass (stats (E, 3), counts (E, 1))."""
    require_cuda()
    E, P = x_out.shape
    out_pitch = _rows(x_out, "x_out")
    src_pitch = _rows(x_src, "x_src") if x_src.shape[0] > 1 else 0
    if x_src.shape[1] != P or x_src.shape[0] not in (1, E):
        raise ValueError("x_src must be (1 or E, P)")
    for t, name in ((targets, "targets"), (cur_stats, "cur_stats")):
        _f64(t, name)
        if t.dim() != 2 or t.shape[1] != 3 or t.stride(1) != 1 or t.shape[0] not in (1, E):
            raise ValueError(f"{name} must be (1 or E, 3)")
    tgt_stride = targets.stride(0) if targets.shape[0] > 1 else 0
    cur_stride = cur_stats.stride(0) if cur_stats.shape[0] > 1 else 0
    if cur_counts.dtype != torch.int64 or cur_counts.shape[1] != 1 or cur_counts.shape[0] not in (1, E):
        raise ValueError("cur_counts must be int64 (1 or E, 1)")
    cnt_stride = cur_counts.stride(0) if cur_counts.shape[0] > 1 else 0
    if status.dtype != torch.int32 or status.numel() < E:
        raise ValueError("status must be int32 (E,)")
    _f64(stats, "stats")
    if stats.shape != (E, 3) or not stats.is_contiguous():
        raise ValueError("stats must be contiguous float64 (E, 3)")
    if counts is not None and (counts.dtype != torch.int64 or counts.numel() < E or not counts.is_contiguous()):
        raise ValueError("counts must be contiguous int64 (E, 1)")
    _lib.call("mmpr_match_restrict", int(E), int(P), targets.data_ptr(), int(tgt_stride), cur_stats.data_ptr(),
              int(cur_stride), cur_counts.data_ptr(), int(cnt_stride), x_src.data_ptr(), int(src_pitch),
              x_out.data_ptr(), int(out_pitch), int(policy), status.data_ptr(), _lib.ptr(clamped),
              stats.data_ptr(), _lib.ptr(counts), _lib.stream_handle(stream))


def coarse_row(ode: _lib.MomentOde, model: _lib.Model, integ: _lib.Integrator, times, iteration: int, rho0,
               fine_stats, cache_in, macro_out, cache_out, raw_out, status, skip_until: int = 0,
               stream=None) -> None:
    """One macro row of the mM iteration on the device (one warp)."""
    require_cuda()
    n = times.numel() - 1
    _lib.call("mmpr_coarse_row", ctypes.byref(ode), ctypes.byref(model), ctypes.byref(integ), int(n),
              times.data_ptr(), int(iteration), rho0.data_ptr(), _lib.ptr(fine_stats), _lib.ptr(cache_in),
              macro_out.data_ptr(), cache_out.data_ptr(), _lib.ptr(raw_out), status.data_ptr(), int(skip_until),
              _lib.stream_handle(stream))


def pipeline_supported(model: _lib.Model, ode: _lib.MomentOde, ode_model: _lib.Model, integ: _lib.Integrator,
                       particles: int, counter_noise: bool = False, n_ranks: int = 1) -> bool:
    """True when iterations 1..K of this configuration run as one persistent
    kernel (mmpr_parareal_pipeline) with this noise supply on this many
    ranks.  Host-only query."""
    return _lib.load().mmpr_pipeline_supported_ex(ctypes.byref(model), ctypes.byref(ode), ctypes.byref(ode_model),
                                                  ctypes.byref(integ), int(particles), int(bool(counter_noise)),
                                                  int(n_ranks)) == 0


# persistent clusters a multi-region pipeline launch may use (its scratch
# rows): at least the co-resident 16-CTA clusters of a B200 (148 SMs x 2 / 16)
PIPELINE_SCRATCH_ROWS = 24


def pipeline_flags_size(n_slices: int, iterations: int) -> int:
    return int(_lib.load().mmpr_pipeline_flags_size(int(n_slices), int(iterations)))


def parareal_pipeline(model: _lib.Model, ode: _lib.MomentOde, ode_model: _lib.Model, integ: _lib.Integrator,
                      dt: float, steps: int,
                      reuse: bool, times, x0, rho0, counts0, xi, snap, fine, macro, micro, micro_counts,
                      fine_stats, fine_counts, raw, cache, bad, coarse_status, match_status, flags,
                      stream=None, counter: _lib.CounterNoise | None = None,
                      partition: _lib.Partition | None = None, region_scratch=None, fine_times=None) -> None:
    """Iterations 1..K of run_micro_macro in one launch (after the prologue).

    With I regions: snap: (K+1 or 2, N+1, P); fine: (2, N, P); macro/micro:
    (K+1, N+1, 3I); micro_counts (K+1, N+1, I); fine_stats/raw: (K, N, 3I);
    fine_counts (K, N, I); cache (K+1, N, 3I); bad (K, N);
    coarse_status/match_status (K+1, N) int32; flags: int32 scratch of
    pipeline_flags_size(N, K).  I > 1 also takes the partition and a float64
    region_scratch of shape (rows, I, P), rows >= 1 (one per persistent
    cluster the launch may use; pipeline_scratch_rows())."""
    require_cuda()
    K1, N1, NV = macro.shape
    K, N = K1 - 1, N1 - 1
    I = NV // 3
    P = x0.shape[-1]
    _f64(snap, "snap")
    if snap.dim() != 3 or snap.shape[1:] != (N + 1, P) or snap.shape[0] not in (K + 1, 2) or snap.stride(2) != 1:
        raise ValueError("snap must be (K+1 or 2, N+1, P)")
    _f64(fine, "fine")
    if fine.shape != (2, N, P) or fine.stride(2) != 1 or fine.stride(0) != N * fine.stride(1):
        raise ValueError("fine must be (2, N, P) with uniform row pitch")
    if counter is None:
        _f64(xi, "xi")
        if xi.dim() != 3 or xi.shape[0] < N or xi.shape[1] < steps or xi.stride(2) != 1:
            raise ValueError("xi must be (N, >=steps, pitch)")
    for t, shape, dtype, name in ((macro, (K + 1, N + 1, 3 * I), torch.float64, "macro"),
                                  (micro, (K + 1, N + 1, 3 * I), torch.float64, "micro"),
                                  (micro_counts, (K + 1, N + 1, I), torch.int64, "micro_counts"),
                                  (fine_stats, (K, N, 3 * I), torch.float64, "fine_stats"),
                                  (fine_counts, (K, N, I), torch.int64, "fine_counts"),
                                  (raw, (K, N, 3 * I), torch.float64, "raw"),
                                  (cache, (K + 1, N, 3 * I), torch.float64, "cache"),
                                  (bad, (K, N), torch.int32, "bad"),
                                  (coarse_status, (K + 1, N), torch.int32, "coarse_status"),
                                  (match_status, (K + 1, N), torch.int32, "match_status")):
        if tuple(t.shape) != shape or t.dtype != dtype or not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous {dtype} {shape}")
    if flags.dtype != torch.int32 or flags.numel() < pipeline_flags_size(N, K):
        raise ValueError("flags must be int32 of pipeline_flags_size(N, K)")
    io = _lib.PipelineIO(times=times.data_ptr(), x0=x0.data_ptr(), rho0=rho0.data_ptr(), counts0=counts0.data_ptr(),
                         xi=xi.data_ptr() if counter is None else None,
                         xi_slice_pitch=xi.stride(0) if counter is None else 0,
                         xi_row_pitch=xi.stride(1) if counter is None else 0,
                         snap=snap.data_ptr(), snap_iter_stride=snap.stride(0), snap_slice_pitch=snap.stride(1),
                         snap_rows=snap.shape[0], fine=fine.data_ptr(), fine_pitch=fine.stride(1),
                         macro=macro.data_ptr(), micro=micro.data_ptr(), micro_counts=micro_counts.data_ptr(),
                         fine_stats=fine_stats.data_ptr(), fine_counts=fine_counts.data_ptr(), raw=raw.data_ptr(),
                         cache=cache.data_ptr(), bad=bad.data_ptr(), coarse_status=coarse_status.data_ptr(),
                         match_status=match_status.data_ptr(), flags=flags.data_ptr())
    if counter is not None:
        io.counter_noise = 1
        io.counter_key[0], io.counter_key[1] = counter.key[0], counter.key[1]
        io.counter_kfield = counter.kfield
    if fine_times is not None:
        if fine_times.dtype != torch.int64 or tuple(fine_times.shape) != (K, N, 2) or not fine_times.is_contiguous():
            raise ValueError("fine_times must be contiguous int64 (K, N, 2)")
        io.fine_times = fine_times.data_ptr()
    if I > 1:
        if partition is None or region_scratch is None:
            raise ValueError("a multi-region pipeline needs the partition and region_scratch")
        _f64(region_scratch, "region_scratch")
        if region_scratch.dim() != 3 or region_scratch.shape[1:] != (I, P) or not region_scratch.is_contiguous():
            raise ValueError("region_scratch must be contiguous (rows, I, P)")
        io.partition = partition
        io.region_scratch = region_scratch.data_ptr()
        io.region_scratch_rows = region_scratch.shape[0]
    _lib.call("mmpr_parareal_pipeline", ctypes.byref(model), ctypes.byref(ode), ctypes.byref(ode_model),
              ctypes.byref(integ), int(N), int(K),
              int(P), int(steps), float(dt), float(math.sqrt(dt)), 1 if reuse else 0, ctypes.byref(io),
              _lib.stream_handle(stream))


def integrate_macro(ode: _lib.MomentOde, model: _lib.Model, integ: _lib.Integrator, t0, t1, state_in, state_out,
                    status, stream=None) -> None:
    require_cuda()
    n = state_in.shape[0]
    _lib.call("mmpr_integrate_macro", ctypes.byref(ode), ctypes.byref(model), ctypes.byref(integ), int(n),
              t0.data_ptr(), t1.data_ptr(), state_in.data_ptr(), state_out.data_ptr(), status.data_ptr(),
              _lib.stream_handle(stream))


def sort_rows(x, out=None, stream=None):
    """Ascending sort of every row of x (R, P) into out (same shape and row
    pitch): np.sort per row."""
    require_cuda()
    _f64(x, "x")
    R, P = x.shape
    pitch = _rows(x, "x")
    if out is None:
        out = torch.empty_strided(x.shape, x.stride(), dtype=torch.float64, device=x.device)
    if out.shape != x.shape or _rows(out, "out") != pitch:
        raise ValueError("out must match x in shape and row pitch")
    nbytes = ctypes.c_uint64(0)
    _lib.call("mmpr_sort_rows", int(R), int(P), None, None, int(pitch), None, ctypes.byref(nbytes),
              _lib.stream_handle(stream))
    temp = torch.empty(max(1, nbytes.value), dtype=torch.uint8, device=x.device)
    _lib.call("mmpr_sort_rows", int(R), int(P), x.data_ptr(), out.data_ptr(), int(pitch), temp.data_ptr(),
              ctypes.byref(nbytes), _lib.stream_handle(stream))
    return out


def mean_abs_diff(a, b, out=None, stream=None):
    """out[r] = np.mean(np.abs(a[r] - b[r])) (numpy pairwise order)."""
    require_cuda()
    _f64(a, "a")
    _f64(b, "b")
    if a.shape != b.shape:
        raise ValueError("a and b must have the same shape")
    R, P = a.shape
    if out is None:
        out = torch.empty(R, dtype=torch.float64, device=a.device)
    _lib.call("mmpr_mean_abs_diff", int(R), int(P), a.data_ptr(), _rows(a, "a"), b.data_ptr(), _rows(b, "b"),
              out.data_ptr(), _lib.stream_handle(stream))
    return out


def _single_region() -> _lib.Partition:
    d = _lib.Partition()
    d.n_regions = 1
    return d


def histogram_sorted(sorted_rows, edges, stream=None):
    """Cumulative counts (R, E) int64 of every sorted row below each edge
    (the last edge inclusive)."""
    require_cuda()
    R, P = sorted_rows.shape
    pitch = _rows(sorted_rows, "sorted_rows")
    _f64(edges, "edges")
    E = edges.numel()
    cum = torch.empty((R, E), dtype=torch.int64, device=sorted_rows.device)
    _lib.call("mmpr_histogram_sorted", int(R), int(P), sorted_rows.data_ptr(), int(pitch),
              edges.contiguous().data_ptr(), int(E), cum.data_ptr(), _lib.stream_handle(stream))
    return cum


def noise_buffer(n_slices: int, steps: int, P: int):
    return torch.empty((n_slices, steps, row_pitch(P)), dtype=torch.float64, device=device())
