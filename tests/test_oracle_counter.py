"""CPU: the counter-based Philox mode's restatement (oracle/npstream.c
section 5) -- the checker of the device's in-register generator.

* Philox2x32-10 core against the Random123 known-answer vectors (Salmon et
  al., SC'11; kat_vectors of the Random123 distribution).
* The ziggurat transform on top is numpy's (same tables and rules as the
  numpy-exact stream, section 3): a counter normal equals numpy's ziggurat
  applied to the same 64-bit words, checked through a scripted bit source.
* Distribution sanity of the generated increments.
"""

import ctypes
import math

import numpy as np
import pytest

from oracle import mm_oracle as O

KAT = [((0, 0), 0, (0xff1dae59, 0x6cd10df2)),
       ((0xffffffff, 0xffffffff), 0xffffffff, (0x2c3f628b, 0xab4fd7ad)),
       ((0x243f6a88, 0x85a308d3), 0x13198a2e, (0xdd7ce038, 0xf62a4c12))]


def _philox(ctr, key):
    c = np.array(ctr, dtype=np.uint32)
    o = np.zeros(2, np.uint32)
    O._nps().nps_philox2x32_10(c.ctypes.data, key, o.ctypes.data)
    return tuple(int(v) for v in o)


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox2x32_10_known_answers(ctr, key, want):
    assert _philox(ctr, key) == want


def test_fast_path_is_numpys_ziggurat_on_the_counter_word():
    """A counter normal whose first word (draw 0) is fast-accepted equals
    numpy's ziggurat value of that word (layer = low 8 bits, sign = bit 8,
    52-bit magnitude times wi[layer]); ~98.8% of draws."""
    seed, n, j = 7, 3, 11
    key = int(O.counter_key(seed)[0]) ^ n
    z = O.counter_normals(seed, n, j, 4000)
    fast = 0
    for p in range(4000):
        o = _philox((p, j), key)
        w = o[0] | (o[1] << 32)
        idx, rabs = w & 0xff, (w >> 9) & 0x000fffffffffffff
        if rabs < _KI[idx]:
            x = float(rabs) * _WI[idx]
            assert z[p] == (-x if (w >> 8) & 1 else x), p
            fast += 1
    assert fast > 0.97 * 4000


def test_counter_normals_distribution():
    z = np.concatenate([O.counter_normals(123, n, j, 50_000) for n in range(4) for j in range(5)])
    N = z.size
    assert abs(z.mean()) < 5 / math.sqrt(N)
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2 / N)
    tail = np.mean(np.abs(z) > 3.6541528853610087)
    assert abs(tail - 2.58e-4) < 5 * math.sqrt(2.58e-4 / N)
    # fresh mode and other slices/steps give other numbers
    assert not np.array_equal(O.counter_normals(123, 0, 0, 100), O.counter_normals(123, 0, 0, 100, 1, True))
    assert not np.array_equal(O.counter_normals(123, 0, 0, 100), O.counter_normals(123, 1, 0, 100))
    assert np.array_equal(O.counter_normals(123, 2, 4, 100)[50:], O.counter_normals(123, 2, 4, 50, first_particle=50))


def _tables():
    import re
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2310_11365_b200", "csrc",
                        "np_ziggurat_tables.h")
    src = open(path).read()

    def grab(name):
        body = src.split(f"#define {name}")[1].split("#define")[0]
        return [v for v in re.findall(r"(0x[0-9a-fA-F.p+\-]+|[-+]?[0-9][0-9.eE+\-]*)", body.replace("\\\n", " "))]
    ki = [int(v.rstrip("ULul"), 16) if v.startswith("0x") and "p" not in v else int(float(v)) for v in grab("NPZ_KI_VALUES")]
    wi = [float.fromhex(v) if v.startswith("0x") else float(v) for v in grab("NPZ_WI_VALUES")]
    return ki, wi


_KI, _WI = _tables()
