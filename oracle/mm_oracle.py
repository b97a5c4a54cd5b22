"""CPU restatement of the reference's mM-Parareal hot path -- TEST INFRASTRUCTURE.

This module is the *checker* for the sm_100a path in paper_2310_11365_b200:
only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline/reference
legs may import it.  It is never the thing measured or shipped.

It restates, with the reference's own numpy operation order (so results are
bit-identical to /root/reference on the same inputs -- pinned by
tests/test_oracle_golden.py against fixtures generated from the reference
itself, tests/golden/make_golden.py):

  noise      NoisePlan.normals / init_rng        particles.py:22-71
  model      drift/diffusion of the factories     models.py:265-279, 339-372
  EM step    _em_step_raw / em_step               particles.py:119-143
  fine       propagate_fine                       particles.py:146-159
  restrict   region_statistics / restrict         particles.py:176-205, coupling.py:26-29
  match      match / lift                         coupling.py:32-95
  coarse     unimodal/perturbed-OU/multimodal rhs moments.py:52-68,111-125,145-192
             integrate (DP5(4))                   rk54.py:16-129
  engine     run_micro_macro / sequential_fine    engine.py:127-277
  metrics    wasserstein_1d / relative_errors /   metrics.py:35-218
             statistical_floor / moment_spread /
             floor_from_references

plus the BASELINE-config additions that have no reference counterpart
("parity unpinned" by reference tests, pinned only by this restatement and by
the reference engine run with these pieces plugged in):
  * forward-Euler coarse integrator (BASELINE configs' "forward Euler dt");
  * cubic mean-field model + Gaussian moment closure (BASELINE config 2);
  * double-well drift with multiplicative noise b = s0*sqrt(1+x^2) (config 5).

Macro states are packed float64 vectors [M_1..M_I, S_1..S_I, a_1..a_I]
(moments.pack_state layout) instead of MacroState objects; arithmetic on
them is the same elementwise IEEE arithmetic MacroState.__add__/__sub__ does.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# errors (errors.py:14-44)
# ---------------------------------------------------------------------------


class OracleBlowup(Exception):
    def __init__(self, slice_index, step_index):
        super().__init__(f"non-finite particle position in slice {slice_index}, step {step_index}")
        self.slice_index = slice_index
        self.step_index = step_index


class OracleDegenerateMatch(Exception):
    def __init__(self, region):
        super().__init__(f"region {region}: cannot scale a zero-variance group")
        self.region = region


class OracleIntegrationFailure(Exception):
    pass


# ---------------------------------------------------------------------------
# noise (particles.py:22-71)
# ---------------------------------------------------------------------------
DOMAIN_INIT, DOMAIN_FROZEN, DOMAIN_FRESH = 0, 1, 2


def _gen(entropy):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy)))


def step_normals(seed, slice_index, step_index, count, iteration=0, fresh=False):
    if fresh:
        ent = (int(seed), DOMAIN_FRESH, int(slice_index), int(step_index), int(iteration))
    else:
        ent = (int(seed), DOMAIN_FROZEN, int(slice_index), int(step_index))
    return _gen(ent).standard_normal(count)


def sample_normal_initial(seed, mean, variance, count):
    """InitialDistribution.normal(mean, variance).sample(plan.init_rng(), P)."""
    return _gen((int(seed), DOMAIN_INIT)).normal(float(mean), math.sqrt(variance), count)


def slice_noise(seed, slice_index, steps, count, iteration=0, fresh=False):
    return np.stack([step_normals(seed, slice_index, j, count, iteration, fresh)
                     for j in range(steps)])


# counter-based Philox mode (NoiseMode.PHILOX*: the device's in-register
# generator, no reference counterpart) -- restated in C in npstream.c
_NPS = None


def _nps():
    global _NPS
    if _NPS is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnpstream.so")
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        lib.nps_counter_normals.argtypes = [P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_int64, P]
        lib.nps_philox2x32_10.argtypes = [P, ctypes.c_uint32, P]
        _NPS = lib
    return _NPS


def counter_key(seed):
    """(SeedSequence((seed, 4)).generate_state(1, uint32), 0) (noise.counter_key)."""
    return np.array([np.random.SeedSequence((int(seed), 4)).generate_state(1, np.uint32)[0], 0], dtype=np.uint32)


def counter_normals(seed, slice_index, step_index, count, iteration=0, fresh=False, first_particle=0):
    key = np.ascontiguousarray(counter_key(seed))
    out = np.empty(count)
    kf = (int(iteration) + 1) if fresh else 0
    _nps().nps_counter_normals(key.ctypes.data, kf, int(slice_index), int(step_index), int(first_particle),
                               int(count), out.ctypes.data)
    return out


def counter_slice_noise(seed, slice_index, steps, count, iteration=0, fresh=False):
    """(steps, P) increments of one slice in the counter-based mode."""
    return np.stack([counter_normals(seed, slice_index, j, count, iteration, fresh) for j in range(steps)])


# ---------------------------------------------------------------------------
# models (descriptor = (kind, params)); factory closures' op order
# ---------------------------------------------------------------------------
OU, LINEAR, DOUBLE_WELL, CUBIC_MF, DW_MULT, ROTATOR, BURGERS = 1, 2, 3, 4, 5, 6, 7
TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class Model:
    kind: int
    p: tuple


def model_ou(a, a_E, B):
    return Model(OU, (float(a), float(a_E), float(B)))


def model_linear(A, A_E, A_0, B, B_E, B_0):
    return Model(LINEAR, tuple(float(v) for v in (A, A_E, A_0, B, B_E, B_0)))


def model_double_well(alpha, gamma, beta, J, sigma):
    tilt = J * math.sqrt(alpha / (2.0 * gamma))
    return Model(DOUBLE_WELL, (4.0 * alpha, 2.0 * gamma, float(beta), tilt, float(sigma), 12.0 * alpha))


def model_cubic(c1, c3, cE, sigma):
    return Model(CUBIC_MF, (float(c1), float(c3), float(cE), float(sigma)))


def model_dw_mult(alpha, gamma, beta, J, s0):
    tilt = J * math.sqrt(alpha / (2.0 * gamma))
    return Model(DW_MULT, (4.0 * alpha, 2.0 * gamma, float(beta), tilt, float(s0), 12.0 * alpha))


def model_rotator(K, kBT, wrap=True):
    """Plane rotator (models.py:286-314): p = (K, sqrt(2 kBT), wrap)."""
    return Model(ROTATOR, (float(K), math.sqrt(2.0 * kBT), 1.0 if wrap else 0.0))


def model_burgers(sigma):
    """Burgers rank interaction (models.py:317-334): p = (0, sigma)."""
    return Model(BURGERS, (0.0, float(sigma)))


def statistic(m: Model, x):
    """ensemble_statistic (models.py:61-83) for every statistic kind."""
    if m.kind == ROTATOR:
        return float(np.mean(np.sin(x))), float(np.mean(np.cos(x)))
    if m.kind == BURGERS:  # mid-rank CDF, ties by index
        order = np.argsort(x, kind="stable")
        ranks = np.empty(len(x), dtype=float)
        ranks[order] = np.arange(len(x), dtype=float)
        return (ranks + 0.5) / len(x)
    return float(np.mean(x))


def drift(m: Model, x, s):
    p = m.p
    if m.kind == ROTATOR:                 # K (cos x S - sin x C) - sin x
        S, C = s
        return p[0] * (np.cos(x) * S - np.sin(x) * C) - np.sin(x)
    if m.kind == BURGERS:                 # 1 - s
        return 1.0 - s
    if m.kind == OU:                      # a * x + a_E * s
        return p[0] * x + p[1] * s
    if m.kind == LINEAR:                  # A x + A_E s + A_0
        return p[0] * x + p[1] * s + p[2]
    if m.kind in (DOUBLE_WELL, DW_MULT):  # -(4 alpha x**3 - 2 gamma x - beta s + tilt)
        return -(p[0] * x ** 3 - p[1] * x - p[2] * s + p[3])
    if m.kind == CUBIC_MF:                # cE s - c1 x - c3 (x x x)
        return p[2] * s - p[0] * x - p[1] * (x * x * x)
    raise ValueError(m.kind)


def diffusion(m: Model, x, s):
    p = m.p
    x = np.asarray(x, dtype=float)
    if m.kind == OU:
        return np.full_like(x, p[2])
    if m.kind == LINEAR:
        return p[3] * x + p[4] * s + p[5]
    if m.kind == DOUBLE_WELL:
        return np.full_like(x, p[4])
    if m.kind == CUBIC_MF:
        return np.full_like(x, p[3])
    if m.kind == DW_MULT:
        return p[4] * np.sqrt(1.0 + x * x)
    if m.kind in (ROTATOR, BURGERS):
        return np.full_like(x, p[1])
    raise ValueError(m.kind)


def coefficients(m: Model, x, s):
    """(a, b, a_x, b_x, b_xx) at scalar x for the moment closures."""
    p = m.p
    a = float(drift(m, x, s))
    b = float(diffusion(m, x, s))
    if m.kind == OU:
        return a, b, p[0], 0.0, 0.0
    if m.kind == LINEAR:
        return a, b, p[0], p[3], 0.0
    if m.kind == DOUBLE_WELL:
        return a, b, float(-(p[5] * x ** 2 - p[1])), 0.0, 0.0
    if m.kind == CUBIC_MF:
        return a, b, float(-p[0] - 3.0 * p[1] * (x * x)), 0.0, 0.0
    if m.kind == DW_MULT:
        q = 1.0 + x * x
        r = np.sqrt(q)
        return a, b, float(-(p[5] * x ** 2 - p[1])), float(p[4] * x / r), float(p[4] / (q * r))
    raise ValueError(m.kind)


# ---------------------------------------------------------------------------
# particles (particles.py:119-205)
# ---------------------------------------------------------------------------


def em_step_raw(m: Model, x, t, dt, noise):
    s = statistic(m, x)
    y = x + drift(m, x, s) * dt + diffusion(m, x, s) * math.sqrt(dt) * noise
    if m.kind == ROTATOR and m.p[2]:      # post_step: np.mod(x, 2 pi)
        y = np.mod(y, TWO_PI)
    return y


def propagate_fine(m: Model, x0, slice_index, t0, dt, steps, noise):
    """noise: (steps, P) increments; returns the slice-end ensemble."""
    x = np.array(x0, dtype=float, copy=True)
    for j in range(steps):
        x = em_step_raw(m, x, t0 + j * dt, dt, noise[j])
        if not np.all(np.isfinite(x)):
            raise OracleBlowup(slice_index, j)
    return x


@dataclass(frozen=True)
class Partition:
    seps: tuple = ()
    peaks: tuple = (0.0,)

    @property
    def n_regions(self):
        return len(self.seps) + 1

    def center(self, i):
        lo = self.seps[i - 1] if i > 0 else -math.inf
        hi = self.seps[i] if i < len(self.seps) else math.inf
        if math.isfinite(lo) and math.isfinite(hi):
            return 0.5 * (lo + hi)
        return self.peaks[i]

    def assign(self, x):
        if not self.seps:
            return np.zeros(len(x), dtype=np.intp)
        return np.searchsorted(np.asarray(self.seps), x, side="right")


SINGLE = Partition()


def restrict(x, part: Partition = SINGLE):
    """Packed [means, variances, fractions] and per-region counts."""
    x = np.asarray(x, dtype=float)
    idx = part.assign(x)
    n = part.n_regions
    out = np.zeros(3 * n)
    counts = np.zeros(n, dtype=np.int64)
    for i in range(n):
        members = x[idx == i]
        c = members.size
        counts[i] = c
        out[2 * n + i] = c / x.size
        if c == 0:
            out[i] = part.center(i)
        elif c == 1:
            out[i] = float(members[0])
        else:
            out[i] = float(np.mean(members))
            out[n + i] = float(np.var(members))
    return out, counts


def match(target, x, part: Partition = SINGLE, policy="raise"):
    """Returns (matched positions, clamped-region bitmask)."""
    n = part.n_regions
    x = np.asarray(x, dtype=float)
    out = x.copy()
    idx = part.assign(x)
    clamped = 0
    for i in range(n):
        mask = idx == i
        members = x[mask]
        if members.size == 0:
            continue
        mu_t = float(target[i])
        var_t = float(target[n + i])
        if var_t < 0.0:
            clamped |= 1 << i
            var_t = 0.0
        cur_mean = float(np.mean(members))
        cur_var = float(np.var(members))
        if cur_var == 0.0:
            if var_t > 0.0 and policy == "raise":
                raise OracleDegenerateMatch(i)
            out[mask] = mu_t
            continue
        scale = math.sqrt(var_t / cur_var)
        if scale == 1.0 and mu_t == cur_mean:
            continue
        out[mask] = scale * (members - cur_mean) + mu_t
    return out, clamped


# ---------------------------------------------------------------------------
# moment ODEs (moments.py) and integrators
# ---------------------------------------------------------------------------
UNIMODAL, PERTURBED_OU, MULTIMODAL, GAUSSIAN_CUBIC, TAYLOR, ROTATOR_TAYLOR, BURGERS_ODE = 1, 2, 3, 4, 5, 6, 7


@dataclass(frozen=True)
class Ode:
    kind: int
    n_regions: int
    p: tuple = ()
    model: Model | None = None


def ode_unimodal(model: Model):
    return Ode(UNIMODAL, 1, (), model)


def ode_perturbed_ou(a, a_E, B, eps_mean=1.0, eps_var=1.0):
    mean_rate = (a + a_E) * (1.0 + eps_mean)
    var_rate = 2.0 * a * (1.0 + eps_mean)
    var_source = B ** 2 * (1.0 + eps_var) ** 2
    return Ode(PERTURBED_OU, 1, (mean_rate, var_rate, var_source))


def ode_multimodal(model: Model, part: Partition, potential, sigma, weight_mode="plain"):
    n = part.n_regions
    peaks = np.asarray(part.peaks, dtype=float)
    if weight_mode == "plain":
        w = np.exp(-np.asarray(potential(peaks), dtype=float))
    else:
        w = np.exp(-np.asarray(potential(peaks), dtype=float) / (2.0 * sigma ** 2))
    targets = w / np.sum(w)
    gaps = np.abs(np.diff(peaks))
    dists = np.empty(n)
    dists[0] = gaps[0]
    dists[1:] = gaps
    rates = sigma ** 2 / (2.0 * dists)
    return Ode(MULTIMODAL, n, tuple(targets) + tuple(rates), model)


def ode_gaussian_cubic(c1, c3, cE, sigma):
    return Ode(GAUSSIAN_CUBIC, 1, (float(c1), float(c3), float(cE), float(sigma)))


def ode_rotator_taylor(K, kBT):
    """The plane rotator's enriched closure (models.py:299-306)."""
    return Ode(ROTATOR_TAYLOR, 1, (float(K), 2.0 * kBT))


def ode_burgers(sigma):
    """burgers_rhs (moments.py:128-142)."""
    return Ode(BURGERS_ODE, 1, (float(sigma) ** 2,))


class OracleSingular(Exception):
    pass


def rhs(ode: Ode, t, y):
    y = np.asarray(y, dtype=float)
    n = ode.n_regions
    if ode.kind == UNIMODAL:
        m, var, _ = y
        if ode.model.kind == ROTATOR:  # point statistic (sin M, cos M)
            K, b = ode.model.p[0], ode.model.p[1]
            S, C = math.sin(m), math.cos(m)
            a = float(K * (np.cos(m) * S - np.sin(m) * C) - np.sin(m))
            a_x = float(K * (-np.sin(m) * S - np.cos(m) * C) - np.cos(m))
            return np.array([a + 0.5 * 0.0, (2.0 * a_x + 0.0 * 0.0) * var + b * b, 0.0])
        a, b, a_x, b_x, b_xx = coefficients(ode.model, m, float(m))
        return np.array([a + 0.5 * b_xx, (2.0 * a_x + b_x * b_x) * var + b * b, 0.0])
    if ode.kind == ROTATOR_TAYLOR:
        m, var, _ = y
        K, sigma_sq = ode.p
        sm, cm = math.sin(m), math.cos(m)
        if abs(sm) < 1e-8 or abs(cm) < 1e-8:
            raise OracleSingular(m)
        return np.array([-sm + var / (2.0 * sm), -2.0 * (-K - cm + var / (2.0 * cm)) * var + sigma_sq, 0.0])
    if ode.kind == BURGERS_ODE:
        _, var, _ = y
        return np.array([0.5, -(2.0 / math.sqrt(2.0 * math.pi)) * math.sqrt(max(var, 0.0)) + ode.p[0], 0.0])
    if ode.kind == PERTURBED_OU:
        m, var, _ = y
        mr, vr, vs = ode.p
        return np.array([mr * m, vr * var + vs, 0.0])
    if ode.kind == MULTIMODAL:
        means, variances, fractions = y[:n], y[n:2 * n], y[2 * n:]
        total = 0.0
        for a_i, m_i in zip(fractions, means):
            total += a_i * float(m_i)
        dm, dv = np.empty(n), np.empty(n)
        for i in range(n):
            a, b, a_x, b_x, b_xx = coefficients(ode.model, means[i], total)
            dm[i] = a + 0.5 * b_xx
            dv[i] = (2.0 * a_x + b_x * b_x) * variances[i] + b * b
        targets = np.asarray(ode.p[:n])
        rates = np.asarray(ode.p[n:2 * n])
        return np.concatenate([dm, dv, -rates * (fractions - targets)])
    if ode.kind == GAUSSIAN_CUBIC:
        c1, c3, cE, sig = ode.p
        m, v, _ = y
        dm = cE * m - c1 * m - c3 * (m * m * m + 3.0 * m * v)
        dv = -2.0 * c1 * v - 6.0 * c3 * v * (m * m + v) + sig * sig
        return np.array([dm, dv, 0.0])
    raise ValueError(ode.kind)


@dataclass(frozen=True)
class Euler:
    """Forward Euler with round((t1-t0)/dt) >= 1 equal steps (BASELINE configs)."""
    dt: float


@dataclass(frozen=True)
class DP54:
    rel_tol: float = 1e-8
    abs_tol: float = 1e-10
    max_steps: int = 100_000
    first_step: float | None = None


def integrate_euler(ode: Ode, y0, t0, t1, dt):
    y = np.atleast_1d(np.asarray(y0, dtype=float)).copy()
    span = t1 - t0
    if span == 0:
        return y
    n = max(1, int(round(span / dt)))
    h = span / n
    for i in range(n):
        y = y + h * rhs(ode, t0 + i * h, y)
    if not np.all(np.isfinite(y)):
        raise OracleIntegrationFailure("non-finite Euler state")
    return y


_C = np.array([0.0, 1 / 5, 3 / 10, 4 / 5, 8 / 9, 1.0, 1.0])
_A = [np.array([]), np.array([1 / 5]), np.array([3 / 40, 9 / 40]),
      np.array([44 / 45, -56 / 15, 32 / 9]),
      np.array([19372 / 6561, -25360 / 2187, 64448 / 6561, -212 / 729]),
      np.array([9017 / 3168, -355 / 33, 46732 / 5247, 49 / 176, -5103 / 18656]),
      np.array([35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84])]
_B5 = np.array([35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84, 0.0])
_B4 = np.array([5179 / 57600, 0.0, 7571 / 16695, 393 / 640, -92097 / 339200, 187 / 2100, 1 / 40])
_E = _B5 - _B4


def integrate_dp54(ode: Ode, y0, t0, t1, cfg: DP54):
    """Dormand-Prince 5(4) with PI control, as rk54.integrate."""
    f = lambda t, y: rhs(ode, t, y)  # noqa: E731
    y = np.atleast_1d(np.asarray(y0, dtype=float)).copy()
    span = t1 - t0
    if span < 0:
        raise ValueError("t1 must not precede t0")
    if span == 0:
        return y
    t = t0
    k1 = np.asarray(f(t, y), dtype=float)
    if not np.all(np.isfinite(k1)):
        raise OracleIntegrationFailure("rhs not finite")
    if cfg.first_step is not None:
        h = cfg.first_step
    else:
        sc = cfg.abs_tol + cfg.rel_tol * np.abs(y)
        d0 = float(np.sqrt(np.mean((y / sc) ** 2)))
        d1 = float(np.sqrt(np.mean((k1 / sc) ** 2)))
        h = 1e-6 if (d0 < 1e-5 or d1 < 1e-5) else 0.01 * d0 / d1
    h = min(h, span)
    err_prev = 1.0
    min_step = 1e-14 * max(abs(t0), abs(t1), 1.0)
    for _ in range(cfg.max_steps):
        h = min(h, t1 - t)
        k = [k1]
        for i in range(1, 7):
            yi = y + h * (np.dot(_A[i], k[:i]) if i > 1 else _A[i][0] * k[0])
            k.append(np.asarray(f(t + _C[i] * h, yi), dtype=float))
        k = np.array(k)
        y_new = y + h * (_B5 @ k)
        err_vec = h * (_E @ k)
        if not np.all(np.isfinite(y_new)):
            raise OracleIntegrationFailure("solution not finite")
        sc = cfg.abs_tol + cfg.rel_tol * np.maximum(np.abs(y), np.abs(y_new))
        err_norm = float(np.sqrt(np.mean((err_vec / sc) ** 2)))
        if err_norm <= 1.0:
            t += h
            y = y_new
            k1 = k[6]
            if t >= t1 - min_step:
                return y
            factor = 0.9 * max(err_norm, 1e-10) ** (-(0.7 / 5.0)) * err_prev ** (0.4 / 5.0)
            err_prev = max(err_norm, 1e-10)
            h *= min(5.0, max(0.2, factor))
        else:
            factor = 0.9 * err_norm ** (-(0.7 / 5.0))
            h *= min(1.0, max(0.2, factor))
        if h < min_step:
            raise OracleIntegrationFailure("step size underflow")
    raise OracleIntegrationFailure("step budget exhausted")


def integrate_macro(ode: Ode, y0, t0, t1, integ):
    if isinstance(integ, Euler):
        return integrate_euler(ode, y0, t0, t1, integ.dt)
    return integrate_dp54(ode, y0, t0, t1, integ)


# ---------------------------------------------------------------------------
# engine (engine.py:127-277)
# ---------------------------------------------------------------------------


@dataclass
class Trace:
    times: tuple
    macro: np.ndarray          # (K+1, N+1, 3I), clamped corrected states
    micro: np.ndarray          # (K+1, N+1, 3I), restriction of matched ensembles
    fine_stats: np.ndarray     # (K, N, 3I) R(F(u_n^k))
    raw: np.ndarray            # (K, N, 3I) corrected states before the clamp
    snapshots: list | None     # [k][n] ensembles
    clamp_events: list = field(default_factory=list)
    fraction_gaps: list = field(default_factory=list)
    lift_collapses: list = field(default_factory=list)


def _fine_task(model, x, n, t0, dt, steps, seed, k, fresh):
    """One slice's F(u_n^k) with its addressed noise (a process-pool task:
    the reference's _fine_sweep map, engine.py:110-124, over processes)."""
    x = np.array(x, dtype=float, copy=True)
    for j in range(steps):  # one step's normals at a time (P = 2^20 slices)
        x = em_step_raw(model, x, t0 + j * dt, dt, step_normals(seed, n, j, x.size, k, fresh))
        if not np.all(np.isfinite(x)):
            raise OracleBlowup(n, j)
    return x


def run_micro_macro(model: Model, ode: Ode, ens0, n_slices, iterations, slice_length, dt, steps,
                    seed, part: Partition = SINGLE, integ=None, t_start=0.0, fresh=False,
                    noise=None, retain_snapshots=True, pool=None):
    """noise: optional callable (n, k) -> (steps, P) array (injected mode);
    default draws the reference's addressed numpy streams.  pool: optional
    multiprocessing pool the fine sweep's slices are mapped over (results are
    identical: every slice's noise is addressed by (n, j[, k]))."""
    integ = integ if integ is not None else DP54()
    ens0 = np.asarray(ens0, dtype=float)
    P = ens0.size
    times = tuple(t_start + n * slice_length for n in range(n_slices + 1))
    I = part.n_regions
    nv = 3 * I

    def C(y, n):
        return integrate_macro(ode, y, times[n], times[n + 1], integ)

    def xi(n, k):
        if noise is not None:
            return noise(n, k)
        return slice_noise(seed, n, steps, P, k, fresh)

    rho0, _ = restrict(ens0, part)
    macro = np.zeros((iterations + 1, n_slices + 1, nv))
    micro = np.zeros((iterations + 1, n_slices + 1, nv))
    fine_stats_all = np.zeros((iterations, n_slices, nv))
    raw_all = np.zeros((iterations, n_slices, nv))
    tr = Trace(times, macro, micro, fine_stats_all, raw_all, [] if retain_snapshots else None)

    row = [rho0]
    ens_row = [ens0]
    cache = []
    for n in range(n_slices):
        pred = C(row[n], n)
        cache.append(pred)
        for i in range(I):
            if rho0[I + i] == 0.0 and pred[I + i] > 0.0 and rho0[2 * I + i] > 0.0:
                tr.lift_collapses.append((0, n + 1, i))
        lifted, _ = match(pred, ens0, part, policy="collapse")
        row.append(pred)
        ens_row.append(lifted)
    macro[0] = np.array(row)
    for n, e in enumerate(ens_row):
        micro[0, n] = restrict(e, part)[0]
    for n in range(1, n_slices + 1):
        tr.fraction_gaps.append((0, n, float(np.max(np.abs(macro[0, n, 2 * I:] - micro[0, n, 2 * I:])))))
    if tr.snapshots is not None:
        tr.snapshots.append(list(ens_row))

    prev = ens_row
    for k in range(iterations):
        if pool is not None and noise is None:
            fine_out = pool.starmap(_fine_task, [(model, prev[n], n, times[n], dt, steps, seed, k, fresh)
                                                 for n in range(n_slices)])
        else:
            fine_out = [propagate_fine(model, prev[n], n, times[n], dt, steps, xi(n, k))
                        for n in range(n_slices)]
        fine_stats = [restrict(f, part)[0] for f in fine_out]
        new_row = [rho0]
        new_ens = [ens0]
        new_cache = []
        for n in range(n_slices):
            pred = C(new_row[n], n)
            new_cache.append(pred)
            corrected = fine_stats[n] + (pred - cache[n])
            raw_all[k, n] = corrected
            fine_stats_all[k, n] = fine_stats[n]
            tr.fraction_gaps.append((k + 1, n + 1, float(np.max(np.abs(
                corrected[2 * I:] - fine_stats[n][2 * I:])))))
            var = corrected[I:2 * I].copy()
            for i in range(I):
                if var[i] < 0.0:
                    tr.clamp_events.append((k + 1, n + 1, i, float(var[i])))
            if var.min() < 0.0:
                var = np.array([max(v, 0.0) for v in var])
            state = np.concatenate([corrected[:I], var, fine_stats[n][2 * I:]])
            matched, _ = match(state, fine_out[n], part, policy="raise")
            new_row.append(state)
            new_ens.append(matched)
        cache = new_cache
        macro[k + 1] = np.array(new_row)
        for n, e in enumerate(new_ens):
            micro[k + 1, n] = restrict(e, part)[0]
        if tr.snapshots is not None:
            tr.snapshots.append(list(new_ens))
        prev = new_ens
    return tr


def sequential_fine(model: Model, ens0, n_slices, slice_length, dt, steps, seed, t_start=0.0,
                    iteration=0, fresh=False, noise=None):
    x = np.asarray(ens0, dtype=float)
    out = [x]
    for n in range(n_slices):
        xi = noise(n, iteration) if noise is not None else slice_noise(seed, n, steps, x.size, iteration, fresh)
        x = propagate_fine(model, x, n, t_start + n * slice_length, dt, steps, xi)
        out.append(x)
    return out


# ---------------------------------------------------------------------------
# error metrics (metrics.py:35-218)
# ---------------------------------------------------------------------------
def w1(a, b):
    """W1 of two equally sized samples: mean |sort(a) - sort(b)| (metrics.py:35-47)."""
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.mean(np.abs(np.sort(a) - np.sort(b))))


def l2(v):
    return float(np.sqrt(np.sum(np.asarray(v) ** 2)))


def relative_errors(snapshots, k, ref_k, var_denominator="variance"):
    """(e_mean, e_var, e_wass, norm_mean, norm_var, norm_wass), per-slice
    |mean err|, |var err|, W1 of iterate k against iterate ref_k over the
    interior boundaries n = 1..N (metrics.py:73-130)."""
    cur, ref = snapshots[k], snapshots[ref_k]
    N = len(cur) - 1
    me = np.array([np.mean(cur[n]) - np.mean(ref[n]) for n in range(1, N + 1)])
    ve = np.array([np.var(cur[n]) - np.var(ref[n]) for n in range(1, N + 1)])
    wa = np.array([w1(cur[n], ref[n]) for n in range(1, N + 1)])
    rm = l2([np.mean(ref[n]) for n in range(1, N + 1)])
    rv = l2([np.var(ref[n]) for n in range(1, N + 1)]) if var_denominator == "variance" else rm
    q = math.sqrt(N)
    scal = np.array([l2(me) / rm, l2(ve) / rv, l2(wa) / rm, l2(me) / q, l2(ve) / q, l2(wa) / q])
    return scal, np.array([np.abs(me), np.abs(ve), wa])


def statistical_floor(finals):
    pairs = [(i, j) for i in range(len(finals)) for j in range(i + 1, len(finals))]
    tot = 0.0
    for i, j in pairs:
        tot += w1(finals[i], finals[j])
    return tot / len(pairs)


def moment_spread(finals):
    pairs = [(i, j) for i in range(len(finals)) for j in range(i + 1, len(finals))]
    m = [float(np.mean(f)) for f in finals]
    v = [float(np.var(f)) for f in finals]
    return (sum(abs(m[i] - m[j]) for i, j in pairs) / len(pairs),
            sum(abs(v[i] - v[j]) for i, j in pairs) / len(pairs))


def floor_from_references(paths, var_denominator="variance"):
    """(e_mean, e_var, e_wass, replicas) from >= 2 serial fine trajectories
    (metrics.py:165-218): moments of the SORTED ensembles, W1 between them."""
    N = len(paths[0]) - 1
    srt = [[np.sort(np.asarray(p[n], dtype=float)) for n in range(1, N + 1)] for p in paths]
    means = np.array([[float(np.mean(x)) for x in s] for s in srt])
    varis = np.array([[float(np.var(x)) for x in s] for s in srt])
    dm = float(np.mean([l2(m) for m in means]))
    dv = float(np.mean([l2(v) for v in varis])) if var_denominator == "variance" else dm
    pairs = [(i, j) for i in range(len(paths)) for j in range(i + 1, len(paths))]
    nm = nv = nw = 0.0
    for i, j in pairs:
        nm += l2(means[i] - means[j])
        nv += l2(varis[i] - varis[j])
        nw += l2(np.array([float(np.mean(np.abs(srt[i][n] - srt[j][n]))) for n in range(N)]))
    c = len(pairs)
    return np.array([nm / c / dm, nv / c / dv, nw / c / dm, len(paths)])
