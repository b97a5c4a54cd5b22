"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/mmpr.h declares, the ctypes descriptors match the C
struct layouts, and the host-side API mirrors the reference's validation."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mmpr.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:const char \*|int |int64_t )(mmpr_\w+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_functions()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.mmpr_version().decode().startswith("mmpr ")


def test_struct_layouts_match_header():
    # sizes implied by include/mmpr.h (natural alignment, x86-64)
    assert ctypes.sizeof(_lib.Model) == 8 + 8 * _lib.MAX_PARAMS
    assert ctypes.sizeof(_lib.Partition) == 8 + 8 * (_lib.MAX_REGIONS - 1) + 8 * _lib.MAX_REGIONS
    assert ctypes.sizeof(_lib.MomentOde) == 8 + 8 * _lib.MAX_ODE_PARAMS
    assert ctypes.sizeof(_lib.Integrator) == 8 + 4 * 8
    # 21 pointers / int64 + snap_rows padded to 8, then counter_noise, counter_key[2], counter_kfield,
    # the partition, region_scratch, region_scratch_rows, fine_times
    assert ctypes.sizeof(_lib.PipelineIO) == 24 * 8 + 16 + ctypes.sizeof(_lib.Partition) + 24
    assert ctypes.sizeof(_lib.CounterNoise) == 16


def test_pipeline_support_query_without_a_gpu():
    """mmpr_pipeline_supported / mmpr_pipeline_flags_size are host-only."""
    from paper_2310_11365_b200 import engine, kernels, moments
    m = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    ode, ode_model = moments.device_ode(mm.unimodal_rhs(m))
    euler = engine.integrator_descriptor(mm.EulerConfig(1e-2))
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 100_000)
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 98_307)
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 10_000)  # 10 elements per lane (config 1)
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 50_000)  # 13 per lane, 8-CTA cluster
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 10_000, counter_noise=True)
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 10_000, n_ranks=2)
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 100_000, counter_noise=True, n_ranks=2)
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 2 ** 17)  # 16 per lane, 16-CTA cluster
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 2 ** 13)
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 2 ** 17, counter_noise=True)
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 9_999)  # any-size form (16 per lane, >= 8)
    assert kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 30_000)
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 30_000, counter_noise=True)
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 4_096)  # fewer than 64 leaf slots
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 2 ** 17 + 8)  # beyond one cluster
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, euler, 2 ** 20)
    dp54 = engine.integrator_descriptor(mm.IntegratorConfig())
    assert not kernels.pipeline_supported(m.descriptor, ode, ode_model, dp54, 100_000)
    spec = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
    cub = mm.make_cubic_meanfield(spec)
    ode_c, odm_c = moments.device_ode(mm.gaussian_closure_rhs(spec))
    assert kernels.pipeline_supported(cub.descriptor, ode_c, odm_c, euler, 100_000)
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    dwm = mm.make_double_well(dw)
    ode_m, odm_m = moments.device_ode(mm.multimodal_rhs(dwm, dw.default_partition(), dw.potential, dw.sigma))
    assert kernels.pipeline_supported(dwm.descriptor, ode_m, odm_m, euler, 100_000)  # two regions (config 3)
    assert not kernels.pipeline_supported(dwm.descriptor, ode_m, odm_m, euler, 100_000, counter_noise=True)
    assert not kernels.pipeline_supported(dwm.descriptor, ode_m, odm_m, euler, 10_000)
    assert kernels.pipeline_supported(dwm.descriptor, ode_m, odm_m, euler, 99_999)  # 12-13 per lane + a tail element
    assert not kernels.pipeline_supported(dwm.descriptor, ode_m, odm_m, euler, 90_000)  # two regions: 13 per lane only
    assert not kernels.pipeline_supported(dwm.descriptor, ode_m, odm_m, dp54, 100_000)
    three = mm.RegionPartition(separatrices=(-0.5, 0.5), peaks=(-1.0, 0.0, 1.0))
    ode_3, odm_3 = moments.device_ode(mm.multimodal_rhs(dwm, three, dw.potential, dw.sigma))
    assert not kernels.pipeline_supported(dwm.descriptor, ode_3, odm_3, euler, 100_000)  # three regions
    assert kernels.pipeline_flags_size(64, 5) == 1 + 5 * 64 + 2 * 6 * 65 + 6 + 1  # ..., abort word
    lib = _lib.load()
    assert lib.mmpr_pipeline_supported(None, None, None, None, 100_000) == 1
    assert lib.mmpr_parareal_pipeline(None, None, None, None, 4, 2, 100_000, 10, 1e-3, 0.03, 1, None, None) == 1


def test_invalid_arguments_are_rejected_without_a_gpu():
    lib = _lib.load()
    # NULL model / negative sizes fail argument checks before any CUDA call
    assert lib.mmpr_fine_sweep(None, 1, 10, 1, 1e-3, 0.03, None, None, 10, None, 10, None, 10, 10, None, None,
                               None) == 1
    assert lib.mmpr_restrict(None, 1, 10, None, 10, None, None, None, None) == 1
    assert lib.mmpr_normals_fill(None, 1, 10, None, 10, 0, 0.0, 1.0, None) == 1


def test_descriptors_follow_factory_closures():
    m = mm.make_double_well(mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.1, sigma=0.5))
    d = m.descriptor
    assert d.kind == _lib.MODEL_DOUBLE_WELL
    tilt = 0.1 * math.sqrt(0.25 / 0.8)
    assert list(d.p)[:6] == [1.0, 0.8, 0.2, tilt, 0.5, 3.0]
    # closures and descriptor describe the same drift
    x = np.linspace(-2, 2, 9)
    ref = -(4 * 0.25 * x ** 3 - 2 * 0.4 * x - 0.2 * 0.3 + tilt)
    assert np.allclose(m.drift(x, 0.3, 0.0), ref)
    ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    assert (ou.descriptor.kind, list(ou.descriptor.p)[:3]) == (_lib.MODEL_OU, [-1.0, 0.5, 0.5])
    assert mm.make_linear(mm.LinearMcKVSpec(A=lambda t: -1.0)).descriptor is None


def test_models_without_descriptor_are_rejected():
    from paper_2310_11365_b200.models import device_model
    with pytest.raises(TypeError):
        device_model(mm.make_linear(mm.LinearMcKVSpec(A=lambda t: -1.0 - t)))
    with pytest.raises(TypeError):  # the closure of a closure-built model
        mm.moments.device_ode(mm.taylor_enriched_rhs(mm.make_linear(mm.LinearMcKVSpec(A=lambda t: -t))))
    # the ROTATOR_SUM / EMPIRICAL_CDF models now carry device descriptors
    rot = device_model(mm.make_plane_rotator(mm.PlaneRotatorSpec(K=0.7, kBT=0.2)))
    assert (rot.kind, rot.stat_kind, list(rot.p)[:4]) == (6, 2, [0.7, math.sqrt(0.4), 1.0, 0.4])
    assert mm.moments.device_ode(mm.burgers_rhs(0.4))[0].kind == 7


def test_partition_and_state_semantics():
    part = mm.RegionPartition(separatrices=(0.0, 2.0), peaks=(-1.0, 1.0, 3.0))
    assert part.center(1) == 1.0 and part.center(0) == -1.0
    np.testing.assert_array_equal(part.assign(np.array([-0.1, 0.0, 2.0, 5.0])), [0, 1, 2, 2])
    d = part.descriptor()
    assert d.n_regions == 3 and list(d.seps)[:2] == [0.0, 2.0] and list(d.centers)[:3] == [-1.0, 1.0, 3.0]
    with pytest.raises(mm.InvalidPartition):
        mm.RegionPartition(separatrices=(0.0,))
    a = mm.MacroState((1.0, 2.0), (0.5, 0.5), (0.4, 0.6))
    b = mm.MacroState((0.5, 0.5), (0.25, 0.25), (0.1, -0.1))
    assert (a - b).fractions == (0.30000000000000004, 0.7)
    assert a.mixture_variance() == pytest.approx(0.74)
    assert mm.MacroState.from_packed(a.packed(), 2) == a


def test_parareal_config_validation_matches_reference():
    step = mm.StepConfig(dt=1e-3, steps_per_slice=100)
    mm.PararealConfig(n_slices=10, iterations=5, slice_length=0.1, particles=10, step=step)
    with pytest.raises(mm.ConfigError):
        mm.PararealConfig(n_slices=10, iterations=11, slice_length=0.1, particles=10, step=step)
    with pytest.raises(mm.ConfigError):  # 62.5 fine steps do not cover a 0.0625 slice at dt=1e-3
        mm.PararealConfig(n_slices=32, iterations=8, slice_length=0.0625, particles=10,
                          step=mm.StepConfig(dt=1e-3, steps_per_slice=62))
    with pytest.raises(ValueError):
        mm.NoisePlan(-1)
    with pytest.raises(ValueError):
        mm.EulerConfig(0.0)


def test_multimodal_ode_descriptor_targets_and_rates():
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    part = dw.default_partition()
    ode = mm.multimodal_rhs(mm.make_double_well(dw), part, dw.potential, dw.sigma)
    p = list(ode.descriptor.p)[:4]
    w = np.exp(-dw.potential(np.array(part.peaks)))
    assert p[:2] == list(w / w.sum())
    gap = abs(part.peaks[1] - part.peaks[0])
    assert p[2:] == [0.25 / (2 * gap)] * 2
    y = np.array([-0.8, 0.9, 0.05, 0.04, 0.5, 0.5])
    assert np.all(np.isfinite(ode.rhs(0.0, y)))


def test_device_calls_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(mm.MmprError):
        mm.ParticleEnsemble([1.0, 2.0])
