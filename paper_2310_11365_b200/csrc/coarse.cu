// Coarse propagator (moment ODEs) and the sequential Parareal correction.
//
// Replaces, on the device and without host round-trips:
//   moments.unimodal_rhs / perturbed_ou_rhs / multimodal_rhs / integrate_macro
//     (/root/reference/pkg/src/mcparareal/moments.py:52-68, 111-125, 145-203)
//   rk54.integrate (/root/reference/pkg/src/mcparareal/rk54.py:57-129)
//   the serial loop of engine.run_micro_macro: iteration-0 cascade
//     (engine.py:170-195) and the correction
//     corrected = R(F_n) + (C(rho_n^{k+1}) - C(rho_n^k)), negative-variance
//     clamp, fraction policy (engine.py:210-236).
// The row is inherently serial in n; one thread walks it with the state in
// registers (3I <= 12 doubles).  Arithmetic follows the reference's numpy
// operation order, so forward-Euler rows are bitwise equal to the CPU
// restatement; DP5(4) matches to rounding (the reference's np.dot goes
// through BLAS).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mmpr_device.cuh"
#include "capi_internal.h"
#include "coarse_device.cuh"

namespace mmpr {

#ifdef MMPR_COARSE_PROFILE
__device__ long long g_coarse_prof[4];  // dev builds: cycles in the Euler loops, calls, total
#endif

// ---- Dormand-Prince 5(4), FSAL, PI step control (rk54.py:16-129) ----------
__constant__ double c_dp_c[7] = {0.0, 1.0 / 5, 3.0 / 10, 4.0 / 5, 8.0 / 9, 1.0, 1.0};
__constant__ double c_dp_a[7][6] = {
    {0, 0, 0, 0, 0, 0},
    {1.0 / 5, 0, 0, 0, 0, 0},
    {3.0 / 40, 9.0 / 40, 0, 0, 0, 0},
    {44.0 / 45, -56.0 / 15, 32.0 / 9, 0, 0, 0},
    {19372.0 / 6561, -25360.0 / 2187, 64448.0 / 6561, -212.0 / 729, 0, 0},
    {9017.0 / 3168, -355.0 / 33, 46732.0 / 5247, 49.0 / 176, -5103.0 / 18656, 0},
    {35.0 / 384, 0.0, 500.0 / 1113, 125.0 / 192, -2187.0 / 6784, 11.0 / 84}};
__constant__ double c_dp_b5[7] = {35.0 / 384, 0.0, 500.0 / 1113, 125.0 / 192, -2187.0 / 6784, 11.0 / 84, 0.0};
__constant__ double c_dp_b4[7] = {5179.0 / 57600, 0.0, 7571.0 / 16695, 393.0 / 640, -92097.0 / 339200,
                                  187.0 / 2100, 1.0 / 40};

template <int NV>
__device__ __forceinline__ double rms_norm(const double *e, const double *scale) {
  double q[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double r = div(e[v], scale[v]);
    q[v] = mul(r, r);
  }
  return __dsqrt_rn(div(small_pairwise(q, NV), (double)NV));
}

template <int NV, int OK, int MK>
__device__ int integrate_dp54(const mmpr_moment_ode &ode, const mmpr_model &model, const mmpr_integrator &cfg,
                              double t0, double t1, double *y) {
  constexpr int nv = NV;
  const double span = sub(t1, t0);
  if (span < 0.0) return 1;
  if (span == 0.0) return MMPR_STAT_OK;
  double t = t0;
  double k[7][NV];
  if (ode_rhs<NV, OK, MK>(ode, model, t, y, k[0])) return MMPR_COARSE_SINGULAR;
  if (!all_finite<NV>(k[0])) return 1;
  double h;
  if (cfg.first_step > 0.0) {
    h = cfg.first_step;
  } else {  // _initial_step
    double sc[NV];
#pragma unroll
    for (int v = 0; v < nv; ++v) sc[v] = add(cfg.abs_tol, mul(cfg.rel_tol, fabs(y[v])));
    const double d0 = rms_norm<NV>(y, sc), d1 = rms_norm<NV>(k[0], sc);
    h = (d0 < 1e-5 || d1 < 1e-5) ? 1e-6 : div(mul(0.01, d0), d1);
  }
  h = fmin(h, span);
  double err_prev = 1.0;
  const double min_step = mul(1e-14, fmax(fmax(fabs(t0), fabs(t1)), 1.0));
  for (int it = 0; it < cfg.max_steps; ++it) {
    h = fmin(h, sub(t1, t));
    double yi[NV];
#pragma unroll
    for (int i = 1; i < 7; ++i) {
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        double acc;
        if (i == 1) {
          acc = mul(c_dp_a[1][0], k[0][v]);
        } else {
          acc = mul(c_dp_a[i][0], k[0][v]);
#pragma unroll
          for (int l = 1; l < i; ++l) acc = add(acc, mul(c_dp_a[i][l], k[l][v]));
        }
        yi[v] = add(y[v], mul(h, acc));
      }
      if (ode_rhs<NV, OK, MK>(ode, model, add(t, mul(c_dp_c[i], h)), yi, k[i])) return MMPR_COARSE_SINGULAR;
    }
    double y5[NV], err[NV], sc[NV];
#pragma unroll
    for (int v = 0; v < nv; ++v) {
      double b5 = mul(c_dp_b5[0], k[0][v]), e = mul(sub(c_dp_b5[0], c_dp_b4[0]), k[0][v]);
#pragma unroll
      for (int l = 1; l < 7; ++l) {
        b5 = add(b5, mul(c_dp_b5[l], k[l][v]));
        e = add(e, mul(sub(c_dp_b5[l], c_dp_b4[l]), k[l][v]));
      }
      y5[v] = add(y[v], mul(h, b5));
      err[v] = mul(h, e);
    }
    if (!all_finite<NV>(y5)) return 1;
#pragma unroll
    for (int v = 0; v < nv; ++v) sc[v] = add(cfg.abs_tol, mul(cfg.rel_tol, fmax(fabs(y[v]), fabs(y5[v]))));
    const double err_norm = rms_norm<NV>(err, sc);
    if (err_norm <= 1.0) {
      t = add(t, h);
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        y[v] = y5[v];
        k[0][v] = k[6][v];
      }
      if (t >= sub(t1, min_step)) return MMPR_STAT_OK;
      const double en = fmax(err_norm, 1e-10);
      const double factor = mul(mul(0.9, pow(en, -(0.7 / 5.0))), pow(err_prev, 0.4 / 5.0));
      err_prev = en;
      h = mul(h, fmin(5.0, fmax(0.2, factor)));
    } else {
      const double factor = mul(0.9, pow(err_norm, -(0.7 / 5.0)));
      h = mul(h, fmin(1.0, fmax(0.2, factor)));
    }
    if (h < min_step) return 1;
  }
  return 1;
}

template <int NV, int OK, int MK>
__device__ __forceinline__ int coarse_step(const mmpr_moment_ode &ode, const mmpr_model &model,
                                           const mmpr_integrator &integ, double t0, double t1, double *y) {
  if (integ.kind == MMPR_INTEG_EULER) {
    long long n;
    double h;
    euler_grid(integ.dt, t0, t1, &n, &h);
    return integrate_euler_n<NV, OK, MK>(ode, model, n, h, t0, y);
  }
  return integrate_dp54<NV, OK, MK>(ode, model, integ, t0, t1, y);
}

struct CoarseParams {
  mmpr_moment_ode ode;
  mmpr_model model;
  mmpr_integrator integ;
  int n;
  const double *times;
  int iteration;
  const double *rho0;
  const double *fine;
  const double *cache_in;
  double *macro_out;
  double *cache_out;
  double *raw_out;
  int32_t *status;
  int skip_until;
};

// The row is serial in n and runs on lane 0.  Before it starts, the whole
// warp computes every slice's Euler grid (step count and size: two
// divisions per slice) into shared memory, and the next slice's inputs
// (fine moments, cached prediction) are fetched one slice ahead through the
// read-only path, so the chain waits on neither.
#define CR_GRID_MAX 2048

template <int NV, int OK, int MK>
__global__ void coarse_row_kernel(const CoarseParams p) {
  __shared__ long long s_n[CR_GRID_MAX];
  __shared__ double s_h[CR_GRID_MAX];
  constexpr int I = NV / 3;
  const bool euler = p.integ.kind == MMPR_INTEG_EULER;
  const bool staged = euler && p.n <= CR_GRID_MAX;
  if (staged) {
    for (int n = threadIdx.x; n < p.n; n += blockDim.x) {
      long long cnt;
      double h;
      euler_grid(p.integ.dt, __ldg(p.times + n), __ldg(p.times + n + 1), &cnt, &h);
      s_n[n] = cnt;
      s_h[n] = h;
    }
    __syncwarp();
  }
  if (threadIdx.x != 0) return;
#ifdef MMPR_COARSE_PROFILE
  const long long ct0 = clock64();
#endif
  const double *__restrict__ times = p.times;
  const double *__restrict__ fine = p.fine;
  const double *__restrict__ cin = p.cache_in;
  const bool corr = p.iteration >= 1;
  double cur[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cur[v] = __ldg(p.rho0 + v);
    p.macro_out[v] = cur[v];
  }
  double t0 = __ldg(times), t1 = p.n > 0 ? __ldg(times + 1) : 0.0;
  double f[NV], c[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    f[v] = (corr && p.n > 0) ? __ldg(fine + v) : 0.0;
    c[v] = (corr && p.n > 0) ? __ldg(cin + v) : 0.0;
  }
  for (int n = 0; n < p.n; ++n) {
    // prefetch slice n+1
    const bool more = n + 1 < p.n;
    const double t2 = more ? __ldg(times + n + 2) : 0.0;
    double fn[NV], cn[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      fn[v] = (corr && more) ? __ldg(fine + (n + 1) * NV + v) : 0.0;
      cn[v] = (corr && more) ? __ldg(cin + (n + 1) * NV + v) : 0.0;
    }
    double pred[NV];
    int st = MMPR_STAT_OK;
    if (corr && n < p.skip_until) {
#pragma unroll
      for (int v = 0; v < NV; ++v) pred[v] = c[v];
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) pred[v] = cur[v];
#ifdef MMPR_COARSE_PROFILE
      const long long c0 = clock64();
#endif
      if (staged) st = integrate_euler_n<NV, OK, MK>(p.ode, p.model, s_n[n], s_h[n], t0, pred);
      else st = coarse_step<NV, OK, MK>(p.ode, p.model, p.integ, t0, t1, pred);
#ifdef MMPR_COARSE_PROFILE
      const long long c1 = clock64();
      g_coarse_prof[0] += c1 - c0;
      g_coarse_prof[1] += 1;
#endif
    }
    p.status[n] = st;
#pragma unroll
    for (int v = 0; v < NV; ++v) p.cache_out[n * NV + v] = pred[v];
    if (!corr) {
#pragma unroll
      for (int v = 0; v < NV; ++v) cur[v] = pred[v];
    } else {
      double raw[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) raw[v] = add(f[v], sub(pred[v], c[v]));
#pragma unroll
      for (int v = 0; v < NV; ++v) p.raw_out[n * NV + v] = raw[v];
      bool neg = false;
#pragma unroll
      for (int i = 0; i < I; ++i) neg |= raw[I + i] < 0.0;
#pragma unroll
      for (int i = 0; i < I; ++i) {
        cur[i] = raw[i];
        cur[I + i] = (neg && raw[I + i] < 0.0) ? 0.0 : raw[I + i];
        cur[2 * I + i] = f[2 * I + i];  // fractions from the fine restriction
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) p.macro_out[(n + 1) * NV + v] = cur[v];
    t0 = t1;
    t1 = t2;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      f[v] = fn[v];
      c[v] = cn[v];
    }
  }
#ifdef MMPR_COARSE_PROFILE
  g_coarse_prof[2] += clock64() - ct0;
#endif
}

template <int NV, int OK, int MK>
__global__ void integrate_macro_kernel(const mmpr_moment_ode ode, const mmpr_model model,
                                       const mmpr_integrator integ, int n_states, const double *t0,
                                       const double *t1, const double *in, double *out, int32_t *status) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_states) return;
  double y[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) y[v] = in[s * NV + v];
  const int st = coarse_step<NV, OK, MK>(ode, model, integ, t0[s], t1[s], y);
#pragma unroll
  for (int v = 0; v < NV; ++v) out[s * NV + v] = y[v];
  status[s] = st;
}

// Kernel selection: (regions, ODE kind, model kind) -> instantiation.
template <template <int, int, int> class L, int NV, int OK>
static int by_model(int mk, const typename L<NV, OK, 0>::Args &a) {
  switch (mk) {
    case MMPR_MODEL_OU: return L<NV, OK, MMPR_MODEL_OU>::run(a);
    case MMPR_MODEL_LINEAR: return L<NV, OK, MMPR_MODEL_LINEAR>::run(a);
    case MMPR_MODEL_DOUBLE_WELL: return L<NV, OK, MMPR_MODEL_DOUBLE_WELL>::run(a);
    case MMPR_MODEL_CUBIC_MF: return L<NV, OK, MMPR_MODEL_CUBIC_MF>::run(a);
    case MMPR_MODEL_DW_MULT: return L<NV, OK, MMPR_MODEL_DW_MULT>::run(a);
    case MMPR_MODEL_ROTATOR:
      if (OK == MMPR_ODE_MULTIMODAL) return MMPR_ERR_UNSUPPORTED;  // mixture closure needs MEAN_OF_F
      return L<NV, OK, MMPR_MODEL_ROTATOR>::run(a);
    default: return MMPR_ERR_UNSUPPORTED;
  }
}

template <template <int, int, int> class L>
static int dispatch_coarse(int n_regions, int ok, int mk, const typename L<3, 1, 0>::Args &a) {
  if (n_regions == 1) {
    switch (ok) {
      case MMPR_ODE_UNIMODAL: return by_model<L, 3, MMPR_ODE_UNIMODAL>(mk, a);
      case MMPR_ODE_PERTURBED_OU: return L<3, MMPR_ODE_PERTURBED_OU, 0>::run(a);
      case MMPR_ODE_GAUSSIAN_CUBIC: return L<3, MMPR_ODE_GAUSSIAN_CUBIC, 0>::run(a);
      case MMPR_ODE_TAYLOR: return by_model<L, 3, MMPR_ODE_TAYLOR>(mk, a);
      case MMPR_ODE_ROTATOR_TAYLOR: return L<3, MMPR_ODE_ROTATOR_TAYLOR, 0>::run(a);
      case MMPR_ODE_BURGERS: return L<3, MMPR_ODE_BURGERS, 0>::run(a);
      case MMPR_ODE_MULTIMODAL: return by_model<L, 3, MMPR_ODE_MULTIMODAL>(mk, a);
      default: return MMPR_ERR_UNSUPPORTED;
    }
  }
  if (ok != MMPR_ODE_MULTIMODAL) return MMPR_ERR_ARG;
  switch (n_regions) {
    case 2: return by_model<L, 6, MMPR_ODE_MULTIMODAL>(mk, a);
    case 3: return by_model<L, 9, MMPR_ODE_MULTIMODAL>(mk, a);
    default: return by_model<L, 12, MMPR_ODE_MULTIMODAL>(mk, a);
  }
}

struct RowArgs {
  CoarseParams p;
  cudaStream_t stream;
};

template <int NV, int OK, int MK>
struct RowLaunch {
  using Args = RowArgs;
  static int run(const Args &a) {
    coarse_row_kernel<NV, OK, MK><<<1, 32, 0, a.stream>>>(a.p); mmpr_launched();
    return mmpr_check_launch("coarse_row_kernel");
  }
};

struct MacroArgs {
  mmpr_moment_ode ode;
  mmpr_model model;
  mmpr_integrator integ;
  int n_states;
  const double *t0, *t1, *in;
  double *out;
  int32_t *status;
  cudaStream_t stream;
};

template <int NV, int OK, int MK>
struct MacroLaunch {
  using Args = MacroArgs;
  static int run(const Args &a) {
    const int threads = 64;
    const int blocks = (a.n_states + threads - 1) / threads;
    integrate_macro_kernel<NV, OK, MK><<<blocks, threads, 0, a.stream>>>(a.ode, a.model, a.integ, a.n_states, a.t0,
                                                                         a.t1, a.in, a.out, a.status); mmpr_launched();
    return mmpr_check_launch("integrate_macro_kernel");
  }
};

}  // namespace mmpr

using namespace mmpr;

static int check_ode(const mmpr_moment_ode *ode, const mmpr_integrator *integ) {
  if (!ode || !integ) return MMPR_ERR_ARG;
  if (ode->n_regions < 1 || ode->n_regions > MMPR_MAX_REGIONS) return MMPR_ERR_ARG;
  if (ode->kind < MMPR_ODE_UNIMODAL || ode->kind > MMPR_ODE_BURGERS) return MMPR_ERR_UNSUPPORTED;
  if (ode->kind != MMPR_ODE_MULTIMODAL && ode->n_regions != 1) return MMPR_ERR_ARG;
  if (integ->kind == MMPR_INTEG_EULER) {
    if (!(integ->dt > 0.0)) return MMPR_ERR_ARG;
  } else if (integ->kind == MMPR_INTEG_DP54) {
    if (!(integ->rel_tol > 0.0) || !(integ->abs_tol > 0.0) || integ->max_steps < 1) return MMPR_ERR_ARG;
  } else {
    return MMPR_ERR_UNSUPPORTED;
  }
  return MMPR_OK;
}

extern "C" int mmpr_coarse_row(const mmpr_moment_ode *ode, const mmpr_model *model, const mmpr_integrator *integ,
                               int32_t n_slices, const double *times, int32_t iteration, const double *rho0,
                               const double *fine_stats, const double *cache_in, double *macro_out,
                               double *cache_out, double *raw_out, int32_t *status, int32_t skip_until,
                               void *stream) {
  int st = check_ode(ode, integ);
  if (st != MMPR_OK) return st;
  if (!model || n_slices < 0 || !times || !rho0 || !macro_out || !cache_out || !status) return MMPR_ERR_ARG;
  if (iteration >= 1 && (!fine_stats || !cache_in || !raw_out)) return MMPR_ERR_ARG;
  CoarseParams p;
  p.ode = *ode;
  p.model = *model;
  p.integ = *integ;
  p.n = n_slices;
  p.times = times;
  p.iteration = iteration;
  p.rho0 = rho0;
  p.fine = fine_stats;
  p.cache_in = cache_in;
  p.macro_out = macro_out;
  p.cache_out = cache_out;
  p.raw_out = raw_out;
  p.status = status;
  p.skip_until = skip_until;
  RowArgs a;
  a.p = p;
  a.stream = (cudaStream_t)stream;
  return dispatch_coarse<RowLaunch>(ode->n_regions, ode->kind, model->kind, a);
}

extern "C" int mmpr_integrate_macro(const mmpr_moment_ode *ode, const mmpr_model *model,
                                    const mmpr_integrator *integ, int32_t n_states, const double *t0,
                                    const double *t1, const double *state_in, double *state_out, int32_t *status,
                                    void *stream) {
  int st = check_ode(ode, integ);
  if (st != MMPR_OK) return st;
  if (!model || n_states < 0 || !t0 || !t1 || !state_in || !state_out || !status) return MMPR_ERR_ARG;
  if (n_states == 0) return MMPR_OK;
  MacroArgs a;
  a.ode = *ode;
  a.model = *model;
  a.integ = *integ;
  a.n_states = n_states;
  a.t0 = t0;
  a.t1 = t1;
  a.in = state_in;
  a.out = state_out;
  a.status = status;
  a.stream = (cudaStream_t)stream;
  return dispatch_coarse<MacroLaunch>(ode->n_regions, ode->kind, model->kind, a);
}

#ifdef MMPR_COARSE_PROFILE
extern "C" int mmpr_dev_coarse_prof(long long *host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, mmpr::g_coarse_prof, sizeof(mmpr::g_coarse_prof));
  static long long zeros[4];
  cudaMemcpyToSymbol(mmpr::g_coarse_prof, zeros, sizeof(zeros));
  return (int)cudaGetLastError();
}
#endif
