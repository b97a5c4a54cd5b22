"""GPU parity: numpy-exact noise streams (noise.cu) against numpy itself,
the C restatement (oracle/npstream.c) and the reference's golden vectors."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TAIL = 3.6541528853610087  # ziggurat tail start (numpy's r)


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_2310_11365_b200 import _lib
    _lib.load()
    assert torch.cuda.is_available()
    return torch.device("cuda")


def _np_stream(entropy, count):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy))).standard_normal(count)


def _assert_stream_equal(got, ref):
    """Bit for bit, tail draws included (the device restates the host libm's
    log1p), and no wedge decision fell in the exp ambiguity band."""
    from paper_2310_11365_b200 import noise
    diff = got != ref
    assert not diff.any(), (f"{int(diff.sum())} draws differ (tail draws among them: "
                            f"{int((np.abs(ref[diff]) > TAIL).sum())})")
    assert noise.exp_ambiguous() == 0
    return 0


def test_step_keys_match_seedsequence(dev):
    from paper_2310_11365_b200 import noise
    for fresh in (False, True):
        keys = noise.step_keys(20240601, fresh, 7, 5, 3, 4).cpu().numpy().view(np.uint64)
        for a in range(3):
            for j in range(4):
                ent = (20240601, 2, 5 + a, j, 7) if fresh else (20240601, 1, 5 + a, j)
                assert np.array_equal(keys[a, j], np.random.SeedSequence(ent).generate_state(2, np.uint64))


@pytest.mark.parametrize("seed", [0, 1, 2 ** 40 + 5, 2 ** 64 - 1])
def test_entropy_key(dev, seed):
    from paper_2310_11365_b200 import noise
    key = noise.entropy_key((seed, 0)).cpu().numpy().view(np.uint64)
    assert np.array_equal(key, np.random.SeedSequence((seed, 0)).generate_state(2, np.uint64))


@pytest.mark.parametrize("P", [1, 2, 7, 1000, 1023, 1024, 1025, 100_000, 262_147])
def test_slice_noise_matches_numpy(dev, P):
    from paper_2310_11365_b200 import noise
    S = 3 if P < 200_000 else 2
    xi = noise.slice_noise(11, 4, 2, S, P).cpu().numpy()
    mismatches = 0
    for a in range(2):
        for j in range(S):
            mismatches += _assert_stream_equal(xi[a, j, :P], _np_stream((11, 1, 4 + a, j), P))
    assert mismatches == 0


def test_fresh_noise_keys_iteration(dev):
    from paper_2310_11365_b200 import NoisePlan
    fresh = NoisePlan(123, "fresh")
    a = fresh.normals(1, 1, 5000, iteration=0)
    b = fresh.normals(1, 1, 5000, iteration=7)
    assert not np.array_equal(a, b)
    _assert_stream_equal(b, _np_stream((123, 2, 1, 1, 7), 5000))
    frozen = NoisePlan(123)
    assert np.array_equal(frozen.normals(1, 1, 50, iteration=0), frozen.normals(1, 1, 50, iteration=7))


def test_golden_noise_vectors(dev, golden):
    from paper_2310_11365_b200 import NoisePlan
    g = golden("noise")
    for c in range(5):
        seed, fresh, n, j, P, k = (int(v) for v in g[f"case{c}_meta"])
        got = NoisePlan(seed, "fresh" if fresh else "frozen").normals(n, j, P, k)
        _assert_stream_equal(got, g[f"case{c}_normals"])


def test_sample_initial_normal_matches_reference(dev, golden):
    from paper_2310_11365_b200 import InitialDistribution, NoisePlan, sample_initial
    g = golden("noise")
    for c in range(2):
        seed, mean, var, P = g[f"init{c}_meta"]
        ens = sample_initial(InitialDistribution.normal(mean, var), NoisePlan(int(seed)), int(P))
        _assert_stream_equal(ens.positions, g[f"init{c}"])


def test_stream_against_c_oracle_many_streams(dev, npstream_lib):
    """200 streams of 5000 draws: GPU vs the C restatement (which is bitwise numpy)."""
    from paper_2310_11365_b200 import noise
    P, N, S = 5000, 20, 10
    xi = noise.slice_noise(99, 0, N, S, P).cpu().numpy()
    total = 0
    for n in range(N):
        for j in range(S):
            w = noise.entropy_words((99, 1, n, j))
            ref = np.zeros(P)
            npstream_lib.nps_standard_normal_fill(w.ctypes.data, len(w), P, ref.ctypes.data)
            total += _assert_stream_equal(xi[n, j, :P], ref)
    assert total == 0


def test_normals_distribution_sanity(dev):
    from paper_2310_11365_b200 import noise
    x = noise.slice_noise(5, 0, 1, 1, 2_000_000).cpu().numpy()[0, 0, :2_000_000]
    assert abs(x.mean()) < 5 / math.sqrt(2e6)
    assert abs(x.var() - 1.0) < 5 * math.sqrt(2 / 2e6)


def test_device_log1p_equals_host_libm(dev, npstream_lib):
    """np::glibc_log1p (the tail draws' log1p) against this host's libm on
    the tail draws' arguments -u and every branch's edge values."""
    from paper_2310_11365_b200 import noise
    from test_oracle_npstream import _log1p_inputs
    x = _log1p_inputs(8_000_000, seed=11)
    ref = np.empty_like(x)
    npstream_lib.nps_libm_log1p_fill(x.ctypes.data, len(x), ref.ctypes.data)
    got = noise.log1p_libm(x).cpu().numpy()
    same = (got.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(got) & np.isnan(ref))
    assert same.all(), f"{(~same).sum()} mismatches, first at {x[~same][:3]}"


def test_tail_heavy_streams_bitwise(dev):
    """Many tail draws (|z| > r): 400 streams x 50k draws hold ~5000 tail
    draws; every one equals numpy's bit for bit."""
    from paper_2310_11365_b200 import noise
    P, N, S = 50_000, 40, 10
    xi = noise.slice_noise(2024, 0, N, S, P).cpu().numpy()
    tails = 0
    for n in range(N):
        for j in range(S):
            ref = _np_stream((2024, 1, n, j), P)
            _assert_stream_equal(xi[n, j, :P], ref)
            tails += int((np.abs(ref) > TAIL).sum())
    assert tails > 2000


@pytest.mark.parametrize("segs", ["2", "3", "8", "13"])
def test_segmented_streams_equal_unsegmented_and_numpy(dev, monkeypatch, segs):
    """Streams cut into segments chained through the mailbox in their last
    output slot (the many-streams launch shape, forced here for 320 streams):
    bit for bit the unsegmented fill, and numpy's streams -- ragged counts,
    so carries, tails and the final partial sub-chunk cross segment ends."""
    from paper_2310_11365_b200 import noise
    for P in (20_000, 33_333):
        N, S = 16, 20  # 320 streams: the warp-per-stream kernel
        monkeypatch.setenv("MMPR_NOISE_SEGS", "1")
        base = noise.slice_noise(5, 3, N, S, P).cpu().numpy()[:, :, :P]
        monkeypatch.setenv("MMPR_NOISE_SEGS", segs)
        got = noise.slice_noise(5, 3, N, S, P).cpu().numpy()[:, :, :P]
        assert np.array_equal(got, base)
        for n, j in ((0, 0), (7, 13), (15, 19)):
            _assert_stream_equal(got[n, j], _np_stream((5, 1, 3 + n, j), P))


def test_segmented_launch_shape_is_the_default_above_the_resident_warps(dev, monkeypatch):
    """More streams than resident warps (2368 on a B200) take the segmented
    shape without a switch; the result is the unsegmented one."""
    from paper_2310_11365_b200 import noise
    N, S, P = 30, 100, 12_000  # 3000 streams
    monkeypatch.delenv("MMPR_NOISE_SEGS", raising=False)
    got = noise.slice_noise(1, 0, N, S, P).cpu().numpy()[:, :, :P]
    monkeypatch.setenv("MMPR_NOISE_SEGS", "1")
    base = noise.slice_noise(1, 0, N, S, P).cpu().numpy()[:, :, :P]
    assert np.array_equal(got, base)
    _assert_stream_equal(got[29, 99], _np_stream((1, 1, 29, 99), P))
