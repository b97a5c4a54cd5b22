// Coarse-propagator device pieces shared by the row kernel (coarse.cu) and
// the iteration pipeline (pipeline.cu): moment-ODE right-hand sides and the
// forward-Euler integrator, in the reference's numpy operation order
// (/root/reference/pkg/src/mcparareal/moments.py:52-68, 111-125, 145-203).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mmpr_device.cuh"

namespace mmpr {

#define CS_MAXV (3 * MMPR_MAX_REGIONS)
#define MMPR_COARSE_SINGULAR 2

// numpy pairwise sum for n <= 128 (short vectors: sequential from 0 when
// n < 8, else 8 accumulators)
static __device__ double small_pairwise(const double *a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = add(r, a[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = add(r[j], a[i + j]);
  double res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
  for (; i < n; ++i) res = add(res, a[i]);
  return res;
}

// OK / MK: ODE and model kinds as compile-time constants, so the serial
// chain is straight-line code with the parameters in registers.
// Returns 0, or MMPR_COARSE_SINGULAR when a closure is evaluated at its
// removable singularity (the reference raises SingularityError).
template <int NV, int OK, int MK>
__device__ __forceinline__ int ode_rhs(const mmpr_moment_ode &ode, const mmpr_model &model_in, double t,
                                       const double *y, double *dy) {
  (void)t;
  constexpr int I = NV / 3;
  mmpr_model model = model_in;
  model.kind = MK;  // folds the family switch in coeffs()
  switch (OK) {
    case MMPR_ODE_UNIMODAL: {  // first-order closure with point statistic s = M
      const double m = y[0], var = y[1];
      const ModelCoeffs c = coeffs(model, m, m);
      dy[0] = add(c.drift, mul(0.5, c.diff_dxx));
      dy[1] = add(mul(add(mul(2.0, c.drift_dx), mul(c.diff_dx, c.diff_dx)), var), mul(c.diff, c.diff));
      dy[2] = 0.0;
      break;
    }
    case MMPR_ODE_PERTURBED_OU: {
      const double *p = ode.p;
      dy[0] = mul(p[0], y[0]);
      dy[1] = add(mul(p[1], y[1]), p[2]);
      dy[2] = 0.0;
      break;
    }
    case MMPR_ODE_MULTIMODAL: {  // mixture statistic sum_i a_i M_i (from 0.0)
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < I; ++i) s = add(s, mul(y[2 * I + i], y[i]));
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const ModelCoeffs c = coeffs(model, y[i], s);
        dy[i] = add(c.drift, mul(0.5, c.diff_dxx));
        dy[I + i] = add(mul(add(mul(2.0, c.drift_dx), mul(c.diff_dx, c.diff_dx)), y[I + i]), mul(c.diff, c.diff));
        // -rates * (fractions - targets)
        dy[2 * I + i] = mul(-ode.p[I + i], sub(y[2 * I + i], ode.p[i]));
      }
      break;
    }
    case MMPR_ODE_GAUSSIAN_CUBIC: {
      // dM = cE*M - c1*M - c3*(M*M*M + 3*M*S)
      // dS = -2*c1*S - 6*c3*S*(M*M + S) + sigma*sigma
      const double *p = ode.p;
      const double m = y[0], v = y[1];
      dy[0] = sub(sub(mul(p[2], m), mul(p[0], m)), mul(p[1], add(mul(mul(m, m), m), mul(mul(3.0, m), v))));
      dy[1] = add(sub(mul(mul(-2.0, p[0]), v), mul(mul(mul(6.0, p[1]), v), add(mul(m, m), v))),
                  mul(p[3], p[3]));
      dy[2] = 0.0;
      break;
    }
    case MMPR_ODE_TAYLOR: {  // first-order closure at the enriched statistic s = M + (S/2) f''(M), f'' = 0
      const double m = y[0], var = y[1];
      const double s = add(m, mul(mul(0.5, var), 0.0));
      const ModelCoeffs c = coeffs(model, m, s);
      dy[0] = add(c.drift, mul(0.5, c.diff_dxx));
      dy[1] = add(mul(add(mul(2.0, c.drift_dx), mul(c.diff_dx, c.diff_dx)), var), mul(c.diff, c.diff));
      dy[2] = 0.0;
      break;
    }
    case MMPR_ODE_ROTATOR_TAYLOR: {  // the rotator's enriched closure (models.py:299-306)
      const double m = y[0], var = y[1];
      double sm, cm;
      sincos(m, &sm, &cm);
      if (fabs(sm) < 1e-8 || fabs(cm) < 1e-8) return MMPR_COARSE_SINGULAR;
      const double K = ode.p[0], sigma_sq = ode.p[1];
      dy[0] = add(-sm, div(var, mul(2.0, sm)));
      dy[1] = add(mul(mul(-2.0, add(sub(-K, cm), div(var, mul(2.0, cm)))), var), sigma_sq);
      dy[2] = 0.0;
      break;
    }
    case MMPR_ODE_BURGERS: {  // dM = 1/2, dS = -(2/sqrt(2 pi)) sqrt(max(S, 0)) + sigma^2
      const double var = y[1];
      const double v = (0.0 > var) ? 0.0 : var;  // Python max(var, 0.0)
      dy[0] = 0.5;
      dy[1] = add(mul(ode.p[1], __dsqrt_rn(v)), ode.p[0]);
      dy[2] = 0.0;
      break;
    }
    default:
#pragma unroll
      for (int i = 0; i < NV; ++i) dy[i] = __longlong_as_double(0x7ff8000000000000ULL);
  }
  return 0;
}

template <int NV>
__device__ __forceinline__ bool all_finite(const double *v) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < NV; ++i) ok &= (bool)isfinite(v[i]);
  return ok;
}

// Forward-Euler step count and size over [t0, t1]: n = round((t1 - t0)/dt) >= 1.
__device__ __forceinline__ void euler_grid(double dt, double t0, double t1, long long *n_out, double *h_out) {
  const double span = sub(t1, t0);
  long long n = llrint(div(span, dt));
  if (n < 1) n = 1;
  *n_out = span == 0.0 ? 0 : n;
  *h_out = div(span, (double)n);
}

// Forward Euler with n equal steps of size h from t0.
template <int NV, int OK, int MK>
__device__ int integrate_euler_n(const mmpr_moment_ode &ode, const mmpr_model &model, long long n, double h,
                                 double t0, double *y) {
  if (n == 0) return MMPR_STAT_OK;
  if constexpr (OK == MMPR_ODE_UNIMODAL && MK == MMPR_MODEL_OU) {
    // the OU closure's coefficients do not depend on the state: the same
    // products the generic path forms every step, formed once
    const double a = model.p[0], aE = model.p[1], B = model.p[2];
    const double c0 = mul(0.5, 0.0);                    // 0.5 * b_xx
    const double c1 = add(mul(2.0, a), mul(0.0, 0.0));  // 2 a_x + b_x^2
    const double c2 = mul(B, B);                        // b^2
    // fractions: f + h*0 repeated n times equals one addition of +0.0 (it
    // only turns -0.0 into +0.0), so it leaves the serial loop
    const double z = mul(h, 0.0);
    double m = y[0], v = y[1];
    const int steps = (int)n;
#pragma unroll 2
    for (int i = 0; i < steps; ++i) {
      const double dm = add(add(mul(a, m), mul(aE, m)), c0);
      const double dv = add(mul(c1, v), c2);
      m = add(m, mul(h, dm));
      v = add(v, mul(h, dv));
    }
    y[0] = m;
    y[1] = v;
    y[2] = add(y[2], z);
    return all_finite<NV>(y) ? MMPR_STAT_OK : 1;
  } else {
    double k[NV];
    for (long long i = 0; i < n; ++i) {
      const double t = add(t0, mul((double)i, h));
      if (ode_rhs<NV, OK, MK>(ode, model, t, y, k)) return MMPR_COARSE_SINGULAR;
#pragma unroll
      for (int v = 0; v < NV; ++v) y[v] = add(y[v], mul(h, k[v]));
    }
    return all_finite<NV>(y) ? MMPR_STAT_OK : 1;
  }
}

}  // namespace mmpr
