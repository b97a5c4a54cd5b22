"""Pin oracle/npstream.c (the CPU restatement of numpy's SeedSequence +
Philox4x64-10 + ziggurat stream, the checker for the GPU generator) against
numpy itself and the reference's golden noise vectors.  CPU only."""

import numpy as np
import pytest

from paper_2310_11365_b200.noise import entropy_words


def _fill(lib, entropy, count):
    w = entropy_words(entropy)
    out = np.zeros(count)
    used = lib.nps_standard_normal_fill(w.ctypes.data, len(w), count, out.ctypes.data)
    return out, used


@pytest.mark.parametrize("entropy", [(0, 1, 0, 0), (0, 1, 3, 5), (2 ** 40 + 5, 1, 3, 5),
                                     (20240601, 2, 7, 99, 3), (0, 0), (2 ** 64 - 1, 3, 12)])
def test_seedsequence_pool_and_key(npstream_lib, entropy):
    w = entropy_words(entropy)
    pool = np.zeros(4, np.uint32)
    key = np.zeros(2, np.uint64)
    npstream_lib.nps_seedseq_pool(w.ctypes.data, len(w), pool.ctypes.data)
    npstream_lib.nps_seedseq_key(w.ctypes.data, len(w), key.ctypes.data)
    ss = np.random.SeedSequence(entropy)
    assert np.array_equal(pool, ss.pool)
    assert np.array_equal(key, ss.generate_state(2, np.uint64))
    assert np.array_equal(key, np.random.Philox(ss).state["state"]["key"])


def test_philox_words_match_numpy_raw(npstream_lib):
    key = np.array([0x0123456789ABCDEF, 0xFEDCBA9876543210], dtype=np.uint64)
    raw = np.random.Philox(key=key).random_raw(64)
    got = np.array([npstream_lib.nps_word(key.ctypes.data, i) for i in range(64)], dtype=np.uint64)
    assert np.array_equal(got, raw)


@pytest.mark.parametrize("entropy,count", [((0, 1, 0, 0), 200_000), ((7, 2, 1, 2, 3), 100_000),
                                           ((20240601, 1, 63, 99), 300_000), ((5, 0), 1)])
def test_standard_normal_stream_bitwise(npstream_lib, entropy, count):
    got, used = _fill(npstream_lib, entropy, count)
    ref = np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy))).standard_normal(count)
    assert np.array_equal(got, ref)
    assert used >= count
    if count > 1000:
        # the stream contains wedge and tail draws (every code path exercised)
        assert used > count
        assert np.any(np.abs(ref) > 3.6541528853610087)


def test_golden_noise_vectors(npstream_lib, golden):
    g = golden("noise")
    for c in range(5):
        seed, fresh, n, j, P, k = (int(v) for v in g[f"case{c}_meta"])
        ent = (seed, 2, n, j, k) if fresh else (seed, 1, n, j)
        got, _ = _fill(npstream_lib, ent, P)
        assert np.array_equal(got, g[f"case{c}_normals"]), c
