"""Shared pytest configuration.

Markers: ``gpu`` -- needs a CUDA device and the in-tree libmmpr.so; run on the
B200 box with ``pytest -m gpu``.  Everything else runs on CPU here.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and libmmpr.so (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name + ".npz"))
    return load


@pytest.fixture(scope="session")
def npstream_lib():
    """oracle/libnpstream.so: the C restatement of numpy's stream (checker)."""
    import ctypes
    import subprocess
    path = os.path.join(ROOT, "oracle", "libnpstream.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    lib.nps_seedseq_pool.argtypes = [P, ctypes.c_int, P]
    lib.nps_seedseq_key.argtypes = [P, ctypes.c_int, P]
    lib.nps_standard_normal_fill.argtypes = [P, ctypes.c_int, ctypes.c_int64, P]
    lib.nps_standard_normal_fill.restype = ctypes.c_uint64
    lib.nps_standard_normal_fill_key.argtypes = [P, ctypes.c_int64, P]
    lib.nps_standard_normal_fill_key.restype = ctypes.c_uint64
    lib.nps_word.argtypes = [P, ctypes.c_uint64]
    lib.nps_word.restype = ctypes.c_uint64
    lib.nps_libm_log1p_fill.argtypes = [P, ctypes.c_int64, P]
    lib.nps_log1p_restated_fill.argtypes = [P, ctypes.c_int64, P]
    return lib
