"""Per-rank buffers, prologue and merge of the multi-rank iteration pipeline
(mmpr_parareal_pipeline_ranks, include/mmpr.h).

Rank r owns the contiguous slices [r*Ng, (r+1)*Ng) (the last rank also
boundary N) and runs the (k, n) units of those slices
(engine.run_micro_macro, /root/reference/pkg/src/mcparareal/engine.py:
197-238).  Every per-slice array is indexed by GLOBAL slice/boundary; a rank
writes only its own entries.  The five arrays another rank reads -- the flag
words, macro, fine_stats, fine_counts and the two parity rows of fine
outputs -- live in one "exchange" block, so on several GPUs a single CUDA IPC
handle per rank maps them into its neighbour's address space.

Used by the multi-GPU driver (distributed.py: one process per GPU, peer
pointers) and by the one-GPU emulation of several ranks (one launch over all
ranks' buffers, tests/test_gpu_pipeline.py).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, kernels
from ._device import device, torch
from .noise import row_pitch, slice_noise

_ALIGN = 256


def exchange_layout(N: int, K: int, P: int) -> dict:
    """name -> (byte offset, element count, dtype) inside the exchange block."""
    items = (("flags", kernels.pipeline_flags_size(N, K), torch.int32),
             ("macro", (K + 1) * (N + 1) * 3, torch.float64),
             ("fine_stats", K * N * 3, torch.float64),
             ("fine_counts", K * N, torch.int64),
             ("fine", 2 * N * P, torch.float64))
    out, off = {}, 0
    for name, count, dtype in items:
        out[name] = (off, count, dtype)
        off += -(-count * torch.empty((), dtype=dtype).element_size() // _ALIGN) * _ALIGN
    out["_bytes"] = off
    return out


def owner(n: int, Ng: int, G: int) -> int:
    """Rank owning slice n / the match unit of boundary n."""
    return min(n // Ng, G - 1)


def owned_boundaries(r: int, Ng: int, G: int, N: int) -> range:
    """Boundaries whose (k, n) units rank r runs: [r*Ng, (r+1)*Ng), plus N
    for the last rank."""
    return range(r * Ng, N + 1 if r == G - 1 else (r + 1) * Ng)


class _RawBlock:
    """A cudaMalloc'd block (mmpr_exchange_alloc) viewed as a torch tensor."""

    def __init__(self, nbytes: int):
        ptr = ctypes.c_void_p()
        _lib.call("mmpr_exchange_alloc", int(nbytes), ctypes.byref(ptr))
        self.ptr = int(ptr.value)
        self.nbytes = int(nbytes)
        self.__cuda_array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                         "version": 2}
        self.tensor = torch.as_tensor(self, device=device())

    def free(self):
        if self.ptr:
            self.tensor = None
            _lib.load().mmpr_exchange_free(ctypes.c_void_p(self.ptr))
            self.ptr = 0


class RankBuffers:
    """Everything one rank's units write, for the (N, K, P, S) run."""

    def __init__(self, r: int, G: int, N: int, K: int, P: int, S: int, retain: bool, raw_exchange: bool = False):
        if N % G:
            raise ValueError(f"n_slices={N} must be divisible by the number of ranks {G}")
        self.r, self.G, self.N, self.K, self.P, self.S = r, G, N, K, P, S
        self.Ng = N // G
        dev = device()
        f64, i64, i32 = torch.float64, torch.int64, torch.int32
        self.layout = exchange_layout(N, K, P)
        nbytes = self.layout["_bytes"]
        if raw_exchange:  # IPC-exportable: its own cudaMalloc
            self.block = _RawBlock(nbytes)
            raw = self.block.tensor
        else:
            self.block = None
            raw = torch.empty((nbytes,), dtype=torch.uint8, device=dev)
        self.exchange = raw
        for name, spec in self.layout.items():
            if name.startswith("_"):
                continue
            off, count, dtype = spec
            nb = count * torch.empty((), dtype=dtype).element_size()
            setattr(self, name, raw[off:off + nb].view(dtype))
        self.flags.zero_()
        self.macro = self.macro.view(K + 1, N + 1, 3)
        self.fine_stats = self.fine_stats.view(K, N, 3)
        self.fine_counts = self.fine_counts.view(K, N, 1)
        self.fine = self.fine.view(2, N, P)
        self.micro = torch.zeros((K + 1, N + 1, 3), dtype=f64, device=dev)
        self.micro_counts = torch.zeros((K + 1, N + 1, 1), dtype=i64, device=dev)
        self.raw = torch.zeros((K, N, 3), dtype=f64, device=dev)
        self.cache = torch.zeros((K + 1, N, 3), dtype=f64, device=dev)
        self.bad = torch.full((K, N), _lib.STAT_OK, dtype=i32, device=dev)
        self.coarse_status = torch.full((K + 1, N), _lib.STAT_OK, dtype=i32, device=dev)
        self.match_status = torch.full((K + 1, N), _lib.STAT_OK, dtype=i32, device=dev)
        self.snap = torch.empty((K + 1 if retain else 2, N + 1, P), dtype=f64, device=dev)
        self.xi = torch.empty((self.Ng, S, row_pitch(P)), dtype=f64, device=dev)
        self.x0 = torch.empty((1, P), dtype=f64, device=dev)
        self.rho0 = torch.empty((1, 3), dtype=f64, device=dev)
        self.counts0 = torch.empty((1, 1), dtype=i64, device=dev)
        self.epoch = 0

    def free(self):
        if self.block is not None:
            self.block.free()

    # ---- C-ABI views --------------------------------------------------------------
    def io(self, times) -> _lib.PipelineIO:
        return _lib.PipelineIO(
            times=times.data_ptr(), x0=self.x0.data_ptr(), rho0=self.rho0.data_ptr(), counts0=self.counts0.data_ptr(),
            xi=self.xi.data_ptr(), xi_slice_pitch=self.xi.stride(0), xi_row_pitch=self.xi.stride(1),
            snap=self.snap.data_ptr(), snap_iter_stride=self.snap.stride(0), snap_slice_pitch=self.snap.stride(1),
            snap_rows=self.snap.shape[0], fine=self.fine.data_ptr(), fine_pitch=self.fine.stride(1),
            macro=self.macro.data_ptr(), micro=self.micro.data_ptr(), micro_counts=self.micro_counts.data_ptr(),
            fine_stats=self.fine_stats.data_ptr(), fine_counts=self.fine_counts.data_ptr(), raw=self.raw.data_ptr(),
            cache=self.cache.data_ptr(), bad=self.bad.data_ptr(), coarse_status=self.coarse_status.data_ptr(),
            match_status=self.match_status.data_ptr(), flags=self.flags.data_ptr())

    def peer_io(self, base: int, template: _lib.PipelineIO) -> _lib.PipelineIO:
        """Another rank's view seen through its exchange block mapped at
        `base` (only the exchange arrays are ever touched; the rest are
        placeholders from `template`)."""
        io = _lib.PipelineIO()
        ctypes.memmove(ctypes.byref(io), ctypes.byref(template), ctypes.sizeof(io))
        L = self.layout
        io.flags = base + L["flags"][0]
        io.macro = base + L["macro"][0]
        io.fine_stats = base + L["fine_stats"][0]
        io.fine_counts = base + L["fine_counts"][0]
        io.fine = base + L["fine"][0]
        return io

    # ---- iteration 0 for this rank's boundaries ---------------------------------------
    def prologue(self, ode_d, ode_model_d, integ_d, times, x0, seed: int, fresh: bool = False):
        """rho0 = R(ens0); the coarse cascade (row 0, every slice,
        redundantly); the lift of the owned boundaries (collapse policy) with
        their micro restriction; the owned slices' FROZEN increments
        (engine.py:153-195)."""
        N, Ng, r, G = self.N, self.Ng, self.r, self.G
        single = kernels._single_region()
        self.x0.copy_(x0.reshape(1, -1))
        kernels.restrict(single, self.x0, self.rho0, self.counts0)
        kernels.coarse_row(ode_d, ode_model_d, integ_d, times, 0, self.rho0, None, None, self.macro[0],
                           self.cache[0], None, self.coarse_status[0])
        lo, hi = r * Ng, (N if r == G - 1 else (r + 1) * Ng - 1)
        a = max(lo, 1)
        snap0 = self.snap[0]
        if hi >= a:
            kernels.match_restrict(self.macro[0, a:hi + 1], self.rho0, self.counts0, self.x0, snap0[a:hi + 1], 1,
                                   self.match_status[0, a - 1:hi], self.micro[0, a:hi + 1],
                                   self.micro_counts[0, a:hi + 1])
        if lo == 0:
            snap0[0].copy_(self.x0[0])
            self.micro[0, 0].copy_(self.rho0[0])
            self.micro_counts[0, 0].copy_(self.counts0[0])
        slice_noise(seed, lo, Ng, self.S, self.P, 0, fresh, out=self.xi)


def launch(model_d, ode_d, ode_model_d, integ_d, dt: float, S: int, reuse: bool, ios, first: int, count: int,
           epoch: int, reset: bool, multi_gpu: bool, N: int, K: int, P: int) -> None:
    arr = (_lib.PipelineIO * len(ios))(*ios)
    _lib.call("mmpr_parareal_pipeline_ranks", ctypes.byref(model_d), ctypes.byref(ode_d), ctypes.byref(ode_model_d),
              ctypes.byref(integ_d), int(N), int(K), int(P), int(S), float(dt), float(np.sqrt(dt)),
              1 if reuse else 0, len(ios), arr, int(first), int(count), int(epoch), 1 if reset else 0,
              1 if multi_gpu else 0, _lib.stream_handle())


# ---- merge of the per-rank results (host, numpy) ---------------------------------------
def merge_rows(parts: list, Ng: int, G: int, N: int, kind: str) -> np.ndarray:
    """Assemble global arrays from per-rank copies (each written only at its
    owned entries; axis 1 indexes slices/boundaries).  kind: "boundary"
    (index n in [0, N]: macro, micro; owner(n), boundary 0 from rank 0 and N
    from the last), "slice" (fine_stats/fine_counts/bad at slice n,
    owner(n)), or "shifted" (cache/raw/coarse_status/match_status at n-1 for
    the match unit of boundary n: index m is owned by owner(m + 1))."""
    stacked = np.stack(parts)  # (G, rows, length, ...)
    length = stacked.shape[2]
    idx = np.arange(length)
    if kind in ("boundary", "slice"):
        src = np.minimum(idx // Ng, G - 1)
    elif kind == "shifted":
        src = np.minimum((idx + 1) // Ng, G - 1)
    else:
        raise ValueError(kind)
    picked = stacked[src, :, idx]  # (length, rows, ...)
    return np.moveaxis(picked, 0, 1).copy()
