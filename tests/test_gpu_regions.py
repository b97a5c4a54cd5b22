"""GPU parity of the one-pass multi-region coupling (restrict_regions.cu:
per-region match and restriction with one cluster per ensemble) against the
separate multi-kernel passes (MMPR_RESTRICT_CLUSTER=0) and the oracle."""

import numpy as np
import pytest

from oracle import mm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import paper_2310_11365_b200 as mm
    mm._lib.load()
    return mm


def _restrict(mm, part, xd, monkeypatch, cluster):
    import torch
    from paper_2310_11365_b200 import kernels
    monkeypatch.setenv("MMPR_RESTRICT_CLUSTER", "1" if cluster else "0")
    E, I = xd.shape[0], part.n_regions
    stats = torch.empty((E, 3 * I), dtype=torch.float64, device="cuda")
    counts = torch.empty((E, I), dtype=torch.int64, device="cuda")
    kernels.restrict(part.descriptor(), xd, stats, counts)
    return stats.cpu().numpy(), counts.cpu().numpy()


@pytest.mark.parametrize("P", [100_000, 98_307, 40_000, 3_001, 129, 17, 2])
def test_cluster_restriction_equals_multi_kernel_and_oracle(mm, monkeypatch, P):
    import torch
    rng = np.random.default_rng(P)
    part = mm.RegionPartition(separatrices=(0.0,), peaks=(-1.0, 1.0))
    E = 5
    x = np.concatenate([rng.normal(-1.0, 0.3, (E, P // 2)), rng.normal(1.0, 0.3, (E, P - P // 2))], axis=1)
    rng.permuted(x, axis=1, out=x)
    if P > 3:
        x[1] = -5.0  # region 1 empty
        x[2, :-1] = -5.0  # one member in region 1
        x[2, -1] = 5.0
        x[3, : P // 3] = 0.0  # on the separatrix: goes right
    xd = torch.from_numpy(x).cuda()
    a, ac = _restrict(mm, part, xd, monkeypatch, True)
    b, bc = _restrict(mm, part, xd, monkeypatch, False)
    assert np.array_equal(a, b) and np.array_equal(ac, bc)
    for e in range(E):
        ref, rc = O.restrict(x[e], O.Partition((0.0,), (-1.0, 1.0)))
        assert np.array_equal(a[e], ref), e
        assert np.array_equal(ac[e], rc), e


@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("P", [100_000, 5_000])
def test_match_restrict_regions_equals_separate_passes(mm, monkeypatch, policy, P):
    """One pass (match by pre-transform membership, restriction of the
    matched positions) against mmpr_match + mmpr_restrict, bit for bit,
    including a degenerate region (zero variance) and a negative target
    variance (clamped)."""
    import torch
    from paper_2310_11365_b200 import kernels
    rng = np.random.default_rng(P + policy)
    part = mm.RegionPartition(separatrices=(0.0,), peaks=(-1.0, 1.0))
    E, I = 4, 2
    x = np.where(rng.random((E, P)) < 0.45, rng.normal(-1.0, 0.25, (E, P)), rng.normal(1.0, 0.25, (E, P)))
    x[2, x[2] >= 0.0] = 0.75  # region 1 degenerate (variance 0)
    xd = torch.from_numpy(x).cuda()
    cur = torch.empty((E, 3 * I), dtype=torch.float64, device="cuda")
    cur_counts = torch.empty((E, I), dtype=torch.int64, device="cuda")
    kernels.restrict(part.descriptor(), xd, cur, cur_counts)
    tgt = cur.clone()
    tgt[:, 0] += 0.05
    tgt[:, 1] -= 0.1
    tgt[:, 2] *= 1.3
    tgt[:, 3] *= 0.7
    tgt[3, 3] = -0.01  # clamped to 0
    tgt[2, 3] = 0.5  # positive target for the zero-variance region: DegenerateMatch(1) when raising
    outs = []
    for cluster in (True, False):
        monkeypatch.setenv("MMPR_RESTRICT_CLUSTER", "1" if cluster else "0")
        out = torch.empty_like(xd)
        st = torch.empty(E, dtype=torch.int32, device="cuda")
        cl = torch.empty(E, dtype=torch.int32, device="cuda")
        stats = torch.empty((E, 3 * I), dtype=torch.float64, device="cuda")
        counts = torch.empty((E, I), dtype=torch.int64, device="cuda")
        scratch = torch.empty((E * I * P,), dtype=torch.float64, device="cuda")
        kernels.match_restrict_regions(part.descriptor(), tgt, cur, cur_counts, xd, out, policy, st, stats, counts,
                                       scratch, clamped=cl)
        outs.append([t.cpu().numpy() for t in (out, st, cl, stats, counts)])
    for u, v in zip(*outs):
        assert np.array_equal(u, v)
    out, st, cl = outs[0][:3]
    assert st[2] == (1 if policy == 0 else mm._lib.STAT_OK) and cl[3] == 2
    for e in range(E):
        if e == 2 and policy == 0:
            continue
        ref, rc = O.match(tgt[e].cpu().numpy(), x[e], O.Partition((0.0,), (-1.0, 1.0)),
                          "raise" if policy == 0 else "collapse")
        assert np.array_equal(out[e], ref), e


def test_bimodal_run_fused_equals_separate(mm, monkeypatch):
    """BASELINE config 3's model at reduced N / K: the engine's one-pass
    multi-region coupling against the separate kernels, bit for bit."""
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    model = mm.make_double_well(dw)
    part = dw.default_partition()
    ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
    cfg = mm.PararealConfig(n_slices=8, iterations=4, slice_length=0.0625, particles=100_000,
                            step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6))
    res = []
    for cluster in ("1", "0"):  # the engine's opt-in one-pass coupling vs its default
        monkeypatch.setenv("MMPR_RESTRICT_CLUSTER", cluster)
        mm.engine.clear_graph_cache()
        tr = mm.run_micro_macro(model, ode, mm.bimodal_initial(-1.0, 1.0, 0.2), cfg, mm.NoisePlan(0))
        res.append((np.array([[s.packed() for s in row] for row in tr.macro]),
                    np.array([[s.packed() for s in row] for row in tr.micro_stats]),
                    np.array([[e.positions for e in row] for row in tr.snapshots])))
    mm.engine.clear_graph_cache()
    for u, v in zip(*res):
        assert np.array_equal(u, v)
