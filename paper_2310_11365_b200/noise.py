"""Device noise: the reference's addressed numpy streams, generated on the GPU.

Mirrors the addressing of NoisePlan (particles.py:22-71): FROZEN step noise is
stream (seed, 1, n, j), FRESH is (seed, 2, n, j, k), the initial ensemble is
(seed, 0).  ``libmmpr`` derives the Philox key of each address with numpy's
SeedSequence and replays numpy's ziggurat over Philox4x64-10 bit for bit, so
``slice_noise`` equals stacking ``NoisePlan.normals(n, j, P, k)``.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import device, require_cuda, torch

DOMAIN_INIT = 0
DOMAIN_STEP_FROZEN = 1
DOMAIN_STEP_FRESH = 2
DOMAIN_DERIVED = 3
DOMAIN_COUNTER = 4  # key of the counter-based Philox mode (NoiseMode.PHILOX*)


def entropy_words(entropy) -> np.ndarray:
    """numpy's coercion of a tuple of non-negative ints to uint32 words."""
    words = []
    for v in entropy:
        v = int(v)
        if v < 0:
            raise ValueError("entropy values must be non-negative")
        if v == 0:
            words.append(0)
        while v > 0:
            words.append(v & 0xFFFFFFFF)
            v >>= 32
    return np.array(words, dtype=np.uint32)


def row_pitch(P: int) -> int:
    """Increment rows are padded to an even length (16-byte aligned rows for
    the bulk copies of the fine sweep)."""
    return P + (P & 1)


def entropy_key(entropy, stream=None):
    """Device uint64[2] Philox key of SeedSequence(entropy)."""
    require_cuda()
    w = entropy_words(entropy)
    if len(w) > 16:
        raise ValueError("entropy tuple too long")
    key = torch.empty(2, dtype=torch.int64, device=device())
    _lib.call("mmpr_entropy_key", w.ctypes.data, len(w), key.data_ptr(), _lib.stream_handle(stream))
    return key


def step_keys(seed: int, fresh: bool, iteration: int, n_offset: int, n_slices: int, steps: int, stream=None):
    """Device uint64[n_slices][steps][2] keys of the step-noise addresses."""
    require_cuda()
    keys = torch.empty((n_slices, steps, 2), dtype=torch.int64, device=device())
    _lib.call("mmpr_noise_keys", int(seed), int(bool(fresh)), int(iteration), int(n_offset), int(n_slices),
              int(steps), keys.data_ptr(), _lib.stream_handle(stream))
    return keys


def fill_normals(keys, count: int, out, pitch: int, loc: float | None = None, scale: float | None = None,
                 stream=None):
    """out[r*pitch + i] = (loc + scale*) z_i of stream r, for every key row."""
    n_streams = keys.numel() // 2
    affine = loc is not None
    _lib.call("mmpr_normals_fill", keys.data_ptr(), int(n_streams), int(count), out.data_ptr(), int(pitch),
              int(affine), float(loc or 0.0), float(scale if scale is not None else 1.0),
              _lib.stream_handle(stream))


def slice_noise(seed: int, n_offset: int, n_slices: int, steps: int, P: int, iteration: int = 0,
                fresh: bool = False, out=None, stream=None):
    """Increments of slices [n_offset, n_offset+n_slices): device tensor
    (n_slices, steps, row_pitch(P)); row j of slice n equals
    NoisePlan(seed, mode).normals(n, j, P, iteration)."""
    pitch = row_pitch(P)
    if out is None:
        out = torch.empty((n_slices, steps, pitch), dtype=torch.float64, device=device())
    if n_slices * steps == 0:
        return out
    keys = step_keys(seed, fresh, iteration, n_offset, n_slices, steps, stream)
    fill_normals(keys, P, out, pitch, stream=stream)
    return out


def normals(seed: int, fresh: bool, slice_index: int, step_index: int, count: int, iteration: int = 0,
            stream=None):
    """Device version of NoisePlan.normals: tensor of ``count`` normals."""
    if fresh:
        ent = (seed, DOMAIN_STEP_FRESH, slice_index, step_index, iteration)
    else:
        ent = (seed, DOMAIN_STEP_FROZEN, slice_index, step_index)
    key = entropy_key(ent, stream)
    out = torch.empty(count, dtype=torch.float64, device=device())
    fill_normals(key, count, out, count, stream=stream)
    return out


def initial_normal(seed: int, mean: float, sd: float, count: int, stream=None):
    """Generator(Philox(SeedSequence((seed, 0)))).normal(mean, sd, count) on the device."""
    key = entropy_key((seed, DOMAIN_INIT), stream)
    out = torch.empty(count, dtype=torch.float64, device=device())
    fill_normals(key, count, out, count, loc=mean, scale=sd, stream=stream)
    return out


def exp_ambiguous(reset: bool = False) -> int:
    """Wedge tests decided inside the band where CUDA's exp and the host
    libm's exp could disagree (0: every ziggurat decision equals numpy's)."""
    import ctypes
    require_cuda()
    torch.cuda.synchronize()
    out = ctypes.c_uint64(0)
    _lib.call("mmpr_noise_exp_ambiguous", ctypes.addressof(out), int(bool(reset)))
    return int(out.value)


def log1p_libm(x):
    """Device log1p equal to the host C library's (numpy's tail draws)."""
    require_cuda()
    x = torch.as_tensor(x, dtype=torch.float64, device=device()).contiguous()
    out = torch.empty_like(x)
    _lib.call("mmpr_log1p_libm", x.data_ptr(), out.data_ptr(), int(x.numel()), _lib.stream_handle())
    return out


def counter_key(seed: int) -> tuple[int, int]:
    """Philox2x32-10 key word of the counter-based mode,
    SeedSequence((seed, 4)).generate_state(1, uint32), and the unused
    second word of mmpr_counter_noise.key."""
    w = np.random.SeedSequence((int(seed), DOMAIN_COUNTER)).generate_state(1, np.uint32)
    return int(w[0]), 0


def counter_noise(seed: int, fresh: bool, iteration: int = 0, slice_offset: int = 0) -> _lib.CounterNoise:
    """mmpr_counter_noise of a plan: frozen (kfield 0) or fresh (iteration + 1)."""
    c = _lib.CounterNoise()
    c.key[0], c.key[1] = counter_key(seed)
    c.kfield = (int(iteration) + 1) if fresh else 0
    if c.kfield >= 1 << 12:
        raise ValueError("iteration index too large for the counter layout")
    c.slice_offset = int(slice_offset)
    return c


def counter_normals(seed: int, fresh: bool, slice_index: int, step_index: int, count: int, iteration: int = 0,
                    rows: int = 1, first_particle: int = 0, stream=None):
    """Device (rows, count) increments of particles first_particle.. at steps
    step_index.. of slice slice_index in the counter-based mode."""
    require_cuda()
    c = counter_noise(seed, fresh, iteration)
    out = torch.empty((rows, count), dtype=torch.float64, device=device())
    import ctypes
    _lib.call("mmpr_counter_normals_fill", ctypes.byref(c), int(slice_index), int(step_index), int(rows),
              int(first_particle), int(count), out.data_ptr(), int(count), _lib.stream_handle(stream))
    return out
