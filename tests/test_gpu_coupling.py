"""GPU parity: restriction and matching (coupling.cu) against the reference's
golden vectors (bit-identical required: both are exact integer bookkeeping
plus numpy's pairwise reductions and IEEE elementwise arithmetic)."""

import logging

import numpy as np
import pytest

from oracle import mm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import paper_2310_11365_b200 as mm
    mm._lib.load()
    return mm


def _parts(mm):
    return {"single": mm.RegionPartition(),
            "two": mm.RegionPartition(separatrices=(0.0,), peaks=(-1.5, 1.5)),
            "three": mm.RegionPartition(separatrices=(0.0, 2.0), peaks=(-1.0, 1.0, 3.0))}


def test_restrict_matches_reference_golden(mm, golden):
    g = golden("coupling")
    parts = _parts(mm)
    for en in g["ens_names"]:
        ens = mm.ParticleEnsemble(g[f"ens_{en}"])
        for pn, part in parts.items():
            st = mm.restrict(ens, part)
            ref = g[f"restrict_{pn}_{en}"]
            assert np.array_equal(st.packed(), ref), (pn, en)
            assert st.degenerate == tuple(g[f"restrict_{pn}_{en}_deg"]), (pn, en)


def test_match_matches_reference_golden(mm, golden):
    g = golden("coupling")
    names = list(g["ens_names"])
    parts = list(_parts(mm).values())
    hp = g["hyp_part"]
    parts.append(mm.RegionPartition(separatrices=(hp[0],), peaks=(hp[1], hp[2])))
    for c in range(10):
        pi, ei, collapse, status = (int(v) for v in g[f"match{c}_meta"])
        part = parts[pi]
        I = part.n_regions
        t = g[f"match{c}_target"]
        target = mm.MacroState(tuple(t[:I]), tuple(t[I:]), (1.0 / I,) * I)
        ens = mm.ParticleEnsemble(g[f"ens_{names[ei]}"])
        policy = "collapse" if collapse else "raise"
        if status >= 0:
            with pytest.raises(mm.DegenerateMatch) as err:
                mm.match(target, ens, part, policy)
            assert err.value.region == status
        else:
            out = mm.match(target, ens, part, policy)
            assert np.array_equal(out.positions, g[f"match{c}_out"]), c


def test_known_answers(mm):
    out = mm.match(mm.MacroState((3.0,), (4.0,), (1.0,)), mm.ParticleEnsemble([-1.0, 1.0]))
    np.testing.assert_allclose(out.positions, [1.0, 5.0])
    part = mm.RegionPartition(separatrices=(0.0,), peaks=(-1.0, 1.0))
    st = mm.region_statistics(mm.ParticleEnsemble([0.0, -1.0]), part)
    assert st.fractions == (0.5, 0.5) and st.means[1] == 0.0
    st = mm.region_statistics(mm.ParticleEnsemble([1.0, 2.0, 3.0]), part)
    assert st.fractions == (0.0, 1.0) and st.means[0] == -1.0 and st.degenerate == (True, False)
    assert mm.empirical_mean(mm.ParticleEnsemble([1.0, 2.0, 3.0, 4.0])) == 2.5
    assert mm.empirical_variance(mm.ParticleEnsemble([1.0, 2.0, 3.0, 4.0])) == 1.25


def test_negative_target_variance_clamped_with_warning(mm, caplog):
    with caplog.at_level(logging.WARNING, logger="mcparareal.coupling"):
        out = mm.match(mm.MacroState((2.0,), (-0.5,), (1.0,)), mm.ParticleEnsemble([-1.0, 0.0, 1.0]))
    assert "clamping negative target variance" in caplog.text
    np.testing.assert_array_equal(out.positions, np.full(3, 2.0))


def test_degenerate_policies(mm):
    ens = mm.ParticleEnsemble([2.0, 2.0])
    target = mm.MacroState((5.0,), (1.0,), (1.0,))
    with pytest.raises(mm.DegenerateMatch) as err:
        mm.match(target, ens)
    assert err.value.region == 0
    np.testing.assert_array_equal(mm.match(target, ens, degenerate_policy="collapse").positions, [5.0, 5.0])
    np.testing.assert_array_equal(mm.match(mm.MacroState((5.0,), (0.0,), (1.0,)), ens).positions, [5.0, 5.0])
    with pytest.raises(ValueError):
        mm.match(target, ens, degenerate_policy="typo")
    with pytest.raises(ValueError):
        mm.match(mm.MacroState((0.0, 1.0), (1.0, 1.0), (0.5, 0.5)), mm.ParticleEnsemble([0.0, 1.0]))


@pytest.mark.parametrize("P", [2, 9, 129, 4097, 100_000])
def test_match_restrict_identity_is_bitwise(mm, P):
    rng = np.random.default_rng(P)
    for part in _parts(mm).values():
        x = rng.normal(0.5, 2.0, P)
        ens = mm.ParticleEnsemble(x)
        out = mm.match(mm.restrict(ens, part), ens, part, "collapse")
        assert np.array_equal(out.positions, x)


@pytest.mark.parametrize("seed", range(40))
def test_random_match_against_oracle(mm, seed):
    rng = np.random.default_rng(1000 + seed)
    P = int(rng.integers(2, 3000))
    sep = float(rng.uniform(-1, 1))
    part_m = mm.RegionPartition(separatrices=(sep,), peaks=(sep - 1.0, sep + 1.0))
    part_o = O.Partition((sep,), (sep - 1.0, sep + 1.0))
    x = rng.normal(0.0, float(rng.uniform(0.1, 3.0)), P)
    if seed % 5 == 0:
        x = np.round(x, 1)  # ties and repeated values
    target = np.array([sep - 0.5, sep + 0.5, rng.uniform(1e-4, 2.0), rng.uniform(1e-4, 2.0), 0.5, 0.5])
    st_ref, _ = O.restrict(x, part_o)
    st = mm.restrict(mm.ParticleEnsemble(x), part_m)
    assert np.array_equal(st.packed(), st_ref)
    try:
        ref, _ = O.match(target, x, part_o, "raise")
    except O.OracleDegenerateMatch as e:
        with pytest.raises(mm.DegenerateMatch) as err:
            mm.match(mm.MacroState.from_packed(target, 2), mm.ParticleEnsemble(x), part_m)
        assert err.value.region == e.region
        return
    out = mm.match(mm.MacroState.from_packed(target, 2), mm.ParticleEnsemble(x), part_m)
    assert np.array_equal(out.positions, ref)


def test_restrict_large_bimodal_against_oracle(mm):
    rng = np.random.default_rng(9)
    P = 1 << 20
    x = np.where(rng.random(P) < 0.5, -1.0, 1.0) + 0.2 * rng.standard_normal(P)
    part_m = mm.RegionPartition(separatrices=(0.0,), peaks=(-0.894427, 0.894427))
    part_o = O.Partition((0.0,), (-0.894427, 0.894427))
    assert np.array_equal(mm.restrict(mm.ParticleEnsemble(x), part_m).packed(), O.restrict(x, part_o)[0])


@pytest.mark.parametrize("P", [1, 2, 7, 8, 9, 100, 1000, 1001, 4097, 65_537, 100_000, 131_072, 200_003, 1 << 20])
def test_restrict_single_region_sizes_bitwise(mm, P):
    """Single-region restriction (cluster kernel up to 16 CTAs, one-CTA
    kernel beyond) against np.mean / np.var, batched over ensembles."""
    from paper_2310_11365_b200 import kernels
    import torch
    rng = np.random.default_rng(P)
    E = 3
    x = rng.normal(0.3, 1.7, (E, P))
    x[1] *= 1e-3
    x[2] = np.round(x[2], 2)  # ties and cancellations
    xd = torch.from_numpy(x).cuda()
    stats = torch.empty((E, 3), dtype=torch.float64, device="cuda")
    counts = torch.empty((E, 1), dtype=torch.int64, device="cuda")
    kernels.restrict(mm.SINGLE_REGION.descriptor(), xd, stats, counts)
    got = stats.cpu().numpy()
    for e in range(E):
        ref, cnt = O.restrict(x[e], O.SINGLE)
        assert np.array_equal(got[e], ref), (e, got[e], ref)
        assert counts[e, 0].item() == P
    # non-finite members propagate like numpy's
    x[0, P // 2] = np.inf
    xd = torch.from_numpy(x).cuda()
    kernels.restrict(mm.SINGLE_REGION.descriptor(), xd, stats, counts)
    with np.errstate(invalid="ignore"):
        ref, _ = O.restrict(x[0], O.SINGLE)
    np.testing.assert_array_equal(stats[0].cpu().numpy(), ref)


@pytest.mark.parametrize("P", [1, 9, 1000, 100_000, 200_003, 1 << 20])
@pytest.mark.parametrize("policy", [0, 1])
def test_match_restrict_fused_equals_separate(mm, P, policy):
    """mmpr_match_restrict == mmpr_match then mmpr_restrict, bit for bit,
    including the identity shortcut, a degenerate (zero-variance) source,
    a negative target variance and a shared source (lift)."""
    from paper_2310_11365_b200 import kernels
    import torch
    rng = np.random.default_rng(P + policy)
    E = 5
    x = rng.normal(0.2, 1.3, (E, P))
    x[3] = 0.7  # zero variance: SET (collapse) or status 0 (raise)
    xd = torch.from_numpy(x).cuda()
    part = mm.SINGLE_REGION.descriptor()
    cur = torch.empty((E, 3), dtype=torch.float64, device="cuda")
    cnt = torch.empty((E, 1), dtype=torch.int64, device="cuda")
    kernels.restrict(part, xd, cur, cnt)
    tg = cur.clone()
    tg[0, 0] += 0.25
    tg[1, 1] *= 1.7
    tg[4, 1] = -0.5  # clamped to 0
    # row 2: identity (target == current) keeps the bits
    for src, s_cur, s_cnt in ((xd, cur, cnt), (xd[:1], cur[:1], cnt[:1])):
        out_a = torch.empty_like(xd)
        st_a = torch.empty(E, dtype=torch.int32, device="cuda")
        kernels.match(part, tg, s_cur, s_cnt, src, out_a, policy, st_a)
        stats_a = torch.empty((E, 3), dtype=torch.float64, device="cuda")
        cnt_a = torch.empty((E, 1), dtype=torch.int64, device="cuda")
        kernels.restrict(part, out_a, stats_a, cnt_a)
        out_b = torch.empty_like(xd)
        st_b = torch.empty(E, dtype=torch.int32, device="cuda")
        stats_b = torch.empty((E, 3), dtype=torch.float64, device="cuda")
        cnt_b = torch.empty((E, 1), dtype=torch.int64, device="cuda")
        kernels.match_restrict(tg, s_cur, s_cnt, src, out_b, policy, st_b, stats_b, cnt_b)
        assert torch.equal(out_a, out_b)
        assert torch.equal(st_a, st_b)
        assert torch.equal(stats_a.nan_to_num(7.0), stats_b.nan_to_num(7.0))
        assert torch.equal(cnt_a, cnt_b)
    assert torch.equal(out_b[2], xd[0]) or src.shape[0] == 1


def test_multi_region_restrict_random_sizes(mm):
    """The multi-CTA multi-region restriction against the oracle, bitwise:
    random sizes, 2-4 regions, empty and one-member regions, many ensembles."""
    from paper_2310_11365_b200 import kernels
    import torch
    rng = np.random.default_rng(77)
    parts = [((0.0,), (-1.0, 1.0)), ((-0.5, 0.5), (-1.0, 0.0, 1.0)), ((-2.0, 0.0, 2.0), (-3.0, -1.0, 1.0, 3.0)),
             ((50.0,), (0.0, 60.0))]  # second region empty
    for P in sorted(set(int(v) for v in np.exp(rng.uniform(0, np.log(3e5), 12))) | {1, 2, 9}):
        for seps, peaks in parts:
            E = 3
            x = rng.normal(0.0, 1.5, (E, P))
            if P > 3:
                x[1, : P - 1] = -9.0  # region 0 takes all but one particle
                x[1, -1] = 9.0
            xd = torch.from_numpy(x).cuda()
            part_m = mm.RegionPartition(separatrices=seps, peaks=peaks)
            I = len(peaks)
            stats = torch.empty((E, 3 * I), dtype=torch.float64, device="cuda")
            counts = torch.empty((E, I), dtype=torch.int64, device="cuda")
            kernels.restrict(part_m.descriptor(), xd, stats, counts)
            got, gc = stats.cpu().numpy(), counts.cpu().numpy()
            part_o = O.Partition(seps, peaks)
            for e in range(E):
                ref, rc = O.restrict(x[e], part_o)
                assert np.array_equal(got[e], ref), (P, seps, e)
                assert np.array_equal(gc[e], rc), (P, seps, e)


# ---- hypothesis: coupling operators against the oracle (test_coupling.py:180-248) ----
from hypothesis import given, settings, strategies as hst  # noqa: E402

_positions = hst.lists(hst.floats(min_value=-50.0, max_value=50.0, allow_nan=False, allow_infinity=False),
                       min_size=2, max_size=40).filter(lambda xs: max(xs) - min(xs) > 1e-3)
_targets = hst.tuples(hst.floats(min_value=-100.0, max_value=100.0), hst.floats(min_value=1e-6, max_value=1e4))


@settings(max_examples=300, deadline=None, derandomize=True)
@given(_positions, _targets)
def test_hypothesis_match_restrict_bitwise_oracle(mm, xs, target):
    """Random small ensembles and targets: match, restrict and their
    composition equal the oracle (the reference's arithmetic) bit for bit;
    matching an ensemble to its own restriction is the identity."""
    mu, var = target
    x = np.array(xs)
    ens = mm.ParticleEnsemble(x)
    out = mm.match(mm.MacroState((mu,), (var,), (1.0,)), ens)
    ref = O.match(np.array([mu, var, 1.0]), x)[0]
    assert np.array_equal(out.positions, ref, equal_nan=True)
    assert np.array_equal(mm.restrict(out).packed(), O.restrict(ref)[0], equal_nan=True)
    assert np.array_equal(mm.match(mm.restrict(ens), ens).positions, x, equal_nan=True)


@settings(max_examples=200, deadline=None, derandomize=True)
@given(hst.lists(hst.floats(min_value=-20.0, max_value=20.0, allow_nan=False, allow_infinity=False),
                 min_size=4, max_size=40), hst.floats(min_value=-5.0, max_value=5.0))
def test_hypothesis_two_region_match_bitwise_oracle(mm, xs, sep):
    x = np.array(xs)
    part_m = mm.RegionPartition(separatrices=(sep,), peaks=(sep - 1.0, sep + 1.0))
    part_o = O.Partition((sep,), (sep - 1.0, sep + 1.0))
    target = mm.MacroState((sep - 0.5, sep + 0.5), (0.01, 0.01), (0.5, 0.5))
    try:
        ref = O.match(np.array(target.packed()), x, part_o)[0]
    except O.OracleDegenerateMatch as e:
        with pytest.raises(mm.DegenerateMatch) as err:
            mm.match(target, mm.ParticleEnsemble(x), part_m)
        assert err.value.region == e.region
        return
    out = mm.match(target, mm.ParticleEnsemble(x), part_m)
    assert np.array_equal(out.positions, ref, equal_nan=True)
    assert np.array_equal(mm.restrict(out, part_m).packed(), O.restrict(ref, part_o)[0], equal_nan=True)
