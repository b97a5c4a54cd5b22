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


def _log1p_inputs(n, seed=3):
    """-u for numpy's unit doubles u (the tail draws' arguments), plus
    tiny/near-one/edge values that reach every branch of log1p."""
    rng = np.random.default_rng(seed)
    u = (rng.integers(0, 2 ** 53, n, dtype=np.uint64) * 2.0 ** -53)
    extra = np.concatenate([u[: n // 8] * 1e-9, 1.0 - u[: n // 8] * 1e-7, u[: n // 16] * 2.0 ** -60,
                            -u[: n // 16] * 10, [0.0, -0.0, -1.0, 2.0 ** -54, -2.0 ** -29, 1e300, -0.2929,
                                                  0.41422, 3.0, 1e17]])
    return np.ascontiguousarray(np.concatenate([-u, extra]))


def test_log1p_restatement_matches_host_libm(npstream_lib):
    """numpy's Marsaglia tail calls the C library's log1p; the device restates
    glibc's FMA build of it (npstream.cuh np::glibc_log1p).  The same
    restatement in C must equal this host's libm bit for bit."""
    import platform
    x = _log1p_inputs(4_000_000)
    libm = np.empty_like(x)
    mine = np.empty_like(x)
    npstream_lib.nps_libm_log1p_fill(x.ctypes.data, len(x), libm.ctypes.data)
    npstream_lib.nps_log1p_restated_fill(x.ctypes.data, len(x), mine.ctypes.data)
    if platform.machine() != "x86_64":
        pytest.skip("restatement is of the x86-64 glibc FMA build")
    same = (mine.view(np.uint64) == libm.view(np.uint64)) | (np.isnan(mine) & np.isnan(libm))
    assert same.all(), f"{(~same).sum()} mismatches, first at {x[~same][:3]}"
