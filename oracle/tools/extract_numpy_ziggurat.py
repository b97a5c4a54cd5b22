"""Recover numpy's ziggurat tables for ``Generator.standard_normal``.

Test/build infrastructure, not product code.  numpy (the reference's only
third-party dependency, pinned here at numpy 2.3.5) draws every standard
normal of ``mcparareal.particles.NoisePlan.normals``
(/root/reference/pkg/src/mcparareal/particles.py:49-61) with a 256-layer
ziggurat over 64-bit Philox words.  Reproducing that stream bit-for-bit on the
GPU needs the three 256-entry tables (layer widths ``wi``, fast-accept
thresholds ``ki``, layer heights ``fi``) and the tail constants.

How they are recovered (no numpy source is read):

* ``wi`` and ``ki`` are *probed*: a custom bit generator (a PyCapsule
  exposing a ``bitgen_t`` whose ``next_uint64`` returns chosen words) feeds
  ``Generator.standard_normal``.  A word with 52-bit mantissa field 1 and
  layer index i returns exactly ``wi[i]``; a binary search on the mantissa
  field for the first word that consumes a second word gives ``ki[i]``.
* ``fi`` is read from numpy's ``_generator`` extension next to the probed
  ``wi`` bytes (the byte pattern occurs exactly once) and validated against
  ``exp(-x_i^2/2)`` (<= 1 ulp) and monotonicity; ``ki`` read from the same
  place must equal the probed values.
* the tail start ``r`` is probed (tail branch with a zero uniform), and
  ``1/r`` is validated by reproducing probed tail outputs exactly.

Run: ``python oracle/tools/extract_numpy_ziggurat.py`` (writes
``paper_2310_11365_b200/csrc/np_ziggurat_tables.h``).
"""

from __future__ import annotations

import ctypes
import glob
import math
import os
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "paper_2310_11365_b200", "csrc", "np_ziggurat_tables.h")

MANT52 = (1 << 52) - 1
HALF_WORD = (1 << 52) << 11        # next_double() == 0.5


class _BitGenT(ctypes.Structure):
    _fields_ = [("state", ctypes.c_void_p), ("next_uint64", ctypes.c_void_p),
                ("next_uint32", ctypes.c_void_p), ("next_double", ctypes.c_void_p),
                ("next_raw", ctypes.c_void_p)]


class ScriptedBitGenerator:
    """Duck-typed numpy BitGenerator replaying a scripted list of words."""

    def __init__(self):
        self.words: list[int] = []
        self.pos = 0

        def next64(_):
            w = self.words[self.pos] if self.pos < len(self.words) else HALF_WORD
            self.pos += 1
            return w

        f64 = ctypes.CFUNCTYPE(ctypes.c_uint64, ctypes.c_void_p)
        f32 = ctypes.CFUNCTYPE(ctypes.c_uint32, ctypes.c_void_p)
        fdb = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_void_p)
        self._keep = (f64(next64), f32(lambda s: next64(s) & 0xFFFFFFFF),
                      fdb(lambda s: (next64(s) >> 11) * (1.0 / 9007199254740992.0)))
        ptr = [ctypes.cast(f, ctypes.c_void_p) for f in self._keep]
        self._bg = _BitGenT(None, ptr[0], ptr[1], ptr[2], ptr[0])
        new = ctypes.pythonapi.PyCapsule_New
        new.restype = ctypes.py_object
        new.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
        self.capsule = new(ctypes.addressof(self._bg), b"BitGenerator", None)
        self.lock = threading.Lock()


def _word(layer: int, mant: int, sign: int = 0) -> int:
    return layer | (sign << 8) | (mant << 9)


def probe():
    src = ScriptedBitGenerator()
    gen = np.random.Generator(src)

    def draw(words):
        src.words, src.pos = list(words), 0
        return float(gen.standard_normal()), src.pos

    wi = np.array([draw([_word(i, 1)])[0] for i in range(256)])

    def fast(layer, mant):
        return draw([_word(layer, mant), 0])[1] == 1

    ki = np.zeros(256, dtype=np.uint64)
    for i in range(256):
        if fast(i, MANT52):
            ki[i] = 1 << 52
            continue
        lo, hi = 0, 1 << 52
        while lo < hi:
            mid = (lo + hi) // 2
            if fast(i, mid):
                lo = mid + 1
            else:
                hi = mid
        ki[i] = lo
    r, used = draw([_word(0, MANT52 ^ (1 << 8)), 0, HALF_WORD])
    assert used == 3 and r > 3.0, (r, used)
    return wi, ki, r, draw


def locate_fi(wi, ki):
    pattern = wi.astype("<f8").tobytes()
    libdir = os.path.dirname(np.random.__file__)
    for path in sorted(glob.glob(os.path.join(libdir, "_generator*.so"))):
        blob = open(path, "rb").read()
        if blob.count(pattern) != 1:
            continue
        at = blob.find(pattern)
        ki_bin = np.frombuffer(blob[at + 2048: at + 4096], dtype="<u8")
        fi = np.frombuffer(blob[at - 2048: at], dtype="<f8").copy()
        assert np.array_equal(ki_bin, ki), "probed ki disagrees with library bytes"
        return fi
    raise RuntimeError("numpy ziggurat tables not found")


def validate_fi(fi, wi):
    x = wi * 2.0 ** 52
    assert fi[0] == 1.0
    assert np.all(np.diff(fi) < 0)
    ulps = np.abs(np.exp(-0.5 * x[1:] * x[1:]) - fi[1:]) / np.spacing(fi[1:])
    assert ulps.max() <= 1.0, ulps.max()


def validate_inv_r(r, draw):
    inv_r = float("0.27366123732975827203338247596")
    for u_bits in (1 << 50, 3 << 49, 12345 << 30, (1 << 52) + 77):
        u = u_bits * 2.0 ** -53
        out, _ = draw([_word(0, MANT52 ^ (1 << 8)), u_bits << 11, ((1 << 53) - 3) << 11])
        xx = -inv_r * math.log1p(-u)
        assert out == r + xx, (out, r + xx)
    return inv_r


def _hex(v: float) -> str:
    return float(v).hex()


def main():
    wi, ki, r, draw = probe()
    fi = locate_fi(wi, ki)
    validate_fi(fi, wi)
    inv_r = validate_inv_r(r, draw)
    assert wi[255] * 2.0 ** 52 == r
    lines = [
        "// GENERATED by oracle/tools/extract_numpy_ziggurat.py from numpy "
        f"{np.__version__} -- do not edit.",
        "// numpy Generator.standard_normal ziggurat (256 layers, 52-bit mantissa):",
        "// wi = layer widths / 2^52, ki = fast-accept mantissa thresholds,",
        "// fi = layer heights exp(-x^2/2); tail start r and 1/r.",
        "#pragma once",
        "#include <stdint.h>",
        f"#define NPZ_R {_hex(r)}",
        f"#define NPZ_INV_R {_hex(inv_r)}",
        "#define NPZ_KI_VALUES \\",
    ]
    def block(values, fmt):
        rows = [", ".join(fmt(v) for v in values[i:i + 4]) for i in range(0, 256, 4)]
        return ["  " + r + (", \\" if i < len(rows) - 1 else "") for i, r in enumerate(rows)]

    lines += block(ki, lambda v: f"0x{int(v):016x}ULL")
    lines += ["", "#define NPZ_WI_VALUES \\"] + block(wi, _hex)
    lines += ["", "#define NPZ_FI_VALUES \\"] + block(fi, _hex)
    lines += [""]
    with open(OUT, "w") as fh:
        fh.write("\n".join(lines))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
