"""ctypes binding of libmmpr.so (the C-ABI declared in include/mmpr.h).

The library is built in-tree (``paper_2310_11365_b200/libmmpr.so``) by
``__graft_entry__.build()`` / ``make -C paper_2310_11365_b200/csrc``.  There is
no CPU fallback: every device entry point raises ``MmprError`` when the
library or a CUDA device is unavailable.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmmpr.so")

MAX_REGIONS = 4
MAX_PARAMS = 8
MAX_ODE_PARAMS = 16

# model families (include/mmpr.h)
MODEL_OU = 1
MODEL_LINEAR = 2
MODEL_DOUBLE_WELL = 3
MODEL_CUBIC_MF = 4
MODEL_DW_MULT = 5
MODEL_ROTATOR = 6
MODEL_BURGERS = 7

STAT_MEAN_OF_F = 0
STAT_EMPIRICAL_CDF = 1
STAT_ROTATOR_SUM = 2

ODE_UNIMODAL = 1
ODE_PERTURBED_OU = 2
ODE_MULTIMODAL = 3
ODE_GAUSSIAN_CUBIC = 4
ODE_TAYLOR = 5
ODE_ROTATOR_TAYLOR = 6
ODE_BURGERS = 7

INTEG_EULER = 1
INTEG_DP54 = 2

STAT_OK = -1
STAT_WATCHDOG = -2
STAT_INTEG_FAILED = 1
STAT_SINGULAR = 2

STATUS_TEXT = {0: "ok", 1: "invalid argument", 2: "CUDA error", 3: "unsupported"}


class MmprError(RuntimeError):
    """A libmmpr call failed (bad argument, CUDA error or unsupported case)."""


class Model(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("stat_kind", ctypes.c_int32),
                ("p", ctypes.c_double * MAX_PARAMS)]


class Partition(ctypes.Structure):
    _fields_ = [("n_regions", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("seps", ctypes.c_double * (MAX_REGIONS - 1)),
                ("centers", ctypes.c_double * MAX_REGIONS)]


class MomentOde(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_regions", ctypes.c_int32),
                ("p", ctypes.c_double * MAX_ODE_PARAMS)]


class Integrator(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("max_steps", ctypes.c_int32),
                ("dt", ctypes.c_double), ("rel_tol", ctypes.c_double),
                ("abs_tol", ctypes.c_double), ("first_step", ctypes.c_double)]


COUNTER_FRESH = 0xFFFFFFFF  # mmpr_pipeline_io.counter_kfield: fresh counter noise


class PipelineIO(ctypes.Structure):
    """mmpr_pipeline_io: device buffers of one run of the iteration pipeline."""
    _fields_ = [("times", ctypes.c_void_p), ("x0", ctypes.c_void_p), ("rho0", ctypes.c_void_p),
                ("counts0", ctypes.c_void_p), ("xi", ctypes.c_void_p), ("xi_slice_pitch", ctypes.c_int64),
                ("xi_row_pitch", ctypes.c_int64), ("snap", ctypes.c_void_p), ("snap_iter_stride", ctypes.c_int64),
                ("snap_slice_pitch", ctypes.c_int64), ("snap_rows", ctypes.c_int32), ("fine", ctypes.c_void_p),
                ("fine_pitch", ctypes.c_int64), ("macro", ctypes.c_void_p), ("micro", ctypes.c_void_p),
                ("micro_counts", ctypes.c_void_p), ("fine_stats", ctypes.c_void_p),
                ("fine_counts", ctypes.c_void_p), ("raw", ctypes.c_void_p), ("cache", ctypes.c_void_p),
                ("bad", ctypes.c_void_p), ("coarse_status", ctypes.c_void_p), ("match_status", ctypes.c_void_p),
                ("flags", ctypes.c_void_p), ("counter_noise", ctypes.c_int32),
                ("counter_key", ctypes.c_uint32 * 2), ("counter_kfield", ctypes.c_uint32),
                ("partition", Partition), ("region_scratch", ctypes.c_void_p),
                ("region_scratch_rows", ctypes.c_int64), ("fine_times", ctypes.c_void_p)]


class CounterNoise(ctypes.Structure):
    """mmpr_counter_noise: counter-based Philox increments (NoiseMode.PHILOX*)."""
    _fields_ = [("key", ctypes.c_uint32 * 2), ("kfield", ctypes.c_uint32), ("slice_offset", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_D = ctypes.c_double

# name -> (restype, argtypes); every symbol include/mmpr.h declares
SIGNATURES = {
    "mmpr_version": (ctypes.c_char_p, []),
    "mmpr_last_error": (ctypes.c_char_p, []),
    "mmpr_kernel_launches": (ctypes.c_uint64, []),
    "mmpr_fine_sweep_occupancy": (ctypes.c_int, [_I64, _P, _P]),
    "mmpr_set_fine_times": (ctypes.c_int, [_P]),
    "mmpr_noise_keys": (ctypes.c_int, [_U64, _I32, _I32, _I32, _I32, _I32, _P, _P]),
    "mmpr_entropy_key": (ctypes.c_int, [_P, _I32, _P, _P]),
    "mmpr_normals_fill": (ctypes.c_int, [_P, _I32, _I64, _P, _I64, _I32, _D, _D, _P]),
    "mmpr_noise_exp_ambiguous": (ctypes.c_int, [_P, _I32]),
    "mmpr_fine_sweep_counter": (ctypes.c_int, [_P, _I32, _I64, _I32, _D, _D, _P, _P, _I64, _P, _I64, _P, _P, _P,
                                                _P, _P]),
    "mmpr_counter_normals_fill": (ctypes.c_int, [_P, _I32, _I32, _I32, _I64, _I64, _P, _I64, _P]),
    "mmpr_log1p_libm": (ctypes.c_int, [_P, _P, _I64, _P]),
    "mmpr_fine_sweep": (ctypes.c_int, [_P, _I32, _I64, _I32, _D, _D, _P, _P, _I64, _P, _I64,
                                        _P, _I64, _I64, _P, _P, _P]),
    "mmpr_restrict": (ctypes.c_int, [_P, _I32, _I64, _P, _I64, _P, _P, _P, _P]),
    "mmpr_restrict_scratch_doubles": (ctypes.c_int64, [_I32, _I64, _I32]),
    "mmpr_match": (ctypes.c_int, [_P, _I32, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _P,
                                   _I64, _I32, _P, _P, _P]),
    "mmpr_match_restrict": (ctypes.c_int, [_I32, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _I32,
                                            _P, _P, _P, _P, _P]),
    "mmpr_match_restrict_regions": (ctypes.c_int, [_P, _I32, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64,
                                                    _I32, _P, _P, _P, _P, _P, _P]),
    "mmpr_coarse_row": (ctypes.c_int, [_P, _P, _P, _I32, _P, _I32, _P, _P, _P, _P, _P, _P, _P,
                                        _I32, _P]),
    "mmpr_integrate_macro": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P, _P, _P, _P, _P]),
    "mmpr_fine_sweep_restrict": (ctypes.c_int, [_P, _I32, _I64, _I32, _D, _D, _P, _P, _I64, _P, _I64,
                                                 _P, _I64, _I64, _P, _P, _P, _P]),
    "mmpr_fine_sweep_stepwise": (ctypes.c_int, [_P, _I32, _I64, _I32, _D, _D, _P, _I64, _P, _I64, _P, _I64,
                                                 _I64, _P, _P, _P, _P]),
    "mmpr_ensemble_statistic": (ctypes.c_int, [_P, _I32, _I64, _P, _I64, _P, _P, _P, _P]),
    "mmpr_sort_rows": (ctypes.c_int, [_I32, _I64, _P, _P, _I64, _P, _P, _P]),
    "mmpr_mean_abs_diff": (ctypes.c_int, [_I32, _I64, _P, _I64, _P, _I64, _P, _P]),
    "mmpr_histogram_sorted": (ctypes.c_int, [_I32, _I64, _P, _I64, _P, _I32, _P, _P]),
    "mmpr_pipeline_flags_size": (ctypes.c_int64, [_I32, _I32]),
    "mmpr_pipeline_supported": (ctypes.c_int, [_P, _P, _P, _P, _I64]),
    "mmpr_pipeline_supported_ex": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _I32]),
    "mmpr_parareal_pipeline": (ctypes.c_int, [_P, _P, _P, _P, _I32, _I32, _I64, _I32, _D, _D, _I32, _P, _P]),
    "mmpr_parareal_pipeline_ranks": (ctypes.c_int, [_P, _P, _P, _P, _I32, _I32, _I64, _I32, _D, _D, _I32, _I32, _P,
                                                     _I32, _I32, _I32, _I32, _I32, _P]),
    "mmpr_exchange_alloc": (ctypes.c_int, [_I64, _P]),
    "mmpr_exchange_free": (ctypes.c_int, [_P]),
    "mmpr_ipc_handle": (ctypes.c_int, [_P, _P]),
    "mmpr_ipc_open": (ctypes.c_int, [_P, _P]),
    "mmpr_ipc_close": (ctypes.c_int, [_P]),
    "mmpr_device_can_access_peer": (ctypes.c_int, [_I32, _I32, _P]),
}

_lib = None
_lock = threading.Lock()


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libmmpr.so once and bind every declared symbol (MMPR_LIB
    overrides the in-tree path, for A/B kernel experiments)."""
    global _lib
    path = path or os.environ.get("MMPR_LIB") or LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise MmprError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if path != LIB_PATH and not hasattr(lib, name):
                continue  # an older build loaded for an A/B experiment
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


# entry points that launch exactly one kernel each (bench.py counts them)
LAUNCHING = frozenset({"mmpr_noise_keys", "mmpr_entropy_key", "mmpr_normals_fill", "mmpr_fine_sweep",
                       "mmpr_fine_sweep_counter", "mmpr_counter_normals_fill",
                       "mmpr_fine_sweep_restrict", "mmpr_match_restrict", "mmpr_match_restrict_regions",
                       "mmpr_restrict", "mmpr_match", "mmpr_coarse_row", "mmpr_integrate_macro",
                       "mmpr_mean_abs_diff", "mmpr_parareal_pipeline", "mmpr_parareal_pipeline_ranks"})
launch_count = {"total": 0}


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise MmprError on failure."""
    lib = load()
    if name in LAUNCHING:  # kernels the call launched (libmmpr's own counter: a call may launch several)
        before = lib.mmpr_kernel_launches()
        status = getattr(lib, name)(*args)
        launch_count["total"] += int(lib.mmpr_kernel_launches() - before)
    else:
        status = getattr(lib, name)(*args)
    if status != 0:
        detail = lib.mmpr_last_error().decode(errors="replace")
        raise MmprError(f"{name} failed: {STATUS_TEXT.get(status, status)}"
                        + (f" ({detail})" if detail else ""))


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
