/*
 * mmpr.h -- C-ABI of libmmpr.so, the sm_100a implementation of the
 * micro-macro (mM) Parareal hot path of arXiv 2310.11365.
 *
 * The reference (mcparareal, /root/reference/pkg/src/mcparareal) is pure
 * Python/numpy with no FFI; each entry point below replaces one of its
 * callables and is bound from the host mirror paper_2310_11365_b200/_lib.py
 * through ctypes (INTEGRATION.md shows the binding).  Conventions:
 *   - every function returns an mmpr_status (0 = launched/ok);
 *   - all double/int buffers are DEVICE pointers owned by the caller, laid out
 *     as documented per argument; descriptor structs are HOST pointers passed
 *     by value into the kernels;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); every call is
 *     stream-ordered and never synchronises the host, except the explicitly
 *     named query functions;
 *   - numerical outcomes the reference reports by exception are returned in
 *     device status arrays (see each function) so one read at the end of a run
 *     reproduces the reference's first error.
 */
#ifndef MMPR_H
#define MMPR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMPR_MAX_REGIONS 4
#define MMPR_MAX_PARAMS 8
#define MMPR_MAX_ODE_PARAMS 16

typedef enum {
  MMPR_OK = 0,
  MMPR_ERR_ARG = 1,         /* invalid argument (shape, pointer, size) */
  MMPR_ERR_CUDA = 2,        /* a CUDA runtime call failed */
  MMPR_ERR_UNSUPPORTED = 3  /* descriptor/geometry not implemented on device */
} mmpr_status;

/* Drift/diffusion families (MEAN_OF_F statistic, f = identity).  Parameter
 * layouts follow the reference factories' closures:
 *  OU          make_perturbed_ou (models.py:265-279): p = {a, a_E, B}
 *  LINEAR      make_linear, constant coefficients (models.py:360-372):
 *              p = {A, A_E, A_0, B, B_E, B_0}
 *  DOUBLE_WELL make_double_well (models.py:339-357):
 *              p = {4*alpha, 2*gamma, beta, tilt, sigma, 12*alpha}
 *  CUBIC_MF    builder model for BASELINE config 2, a = cE*s - c1*x - c3*x^3:
 *              p = {c1, c3, cE, sigma}
 *  DW_MULT     double-well drift with b = s0*sqrt(1+x^2) (BASELINE config 5):
 *              p = {4*alpha, 2*gamma, beta, tilt, s0, 12*alpha}
 *  ROTATOR     make_plane_rotator (models.py:286-314), ROTATOR_SUM statistic:
 *              p = {K, sqrt(2 kBT), wrap (0/1), 2 kBT}
 *  BURGERS     make_burgers (models.py:317-334), EMPIRICAL_CDF statistic:
 *              p = {0, sigma} */
enum {
  MMPR_MODEL_OU = 1,
  MMPR_MODEL_LINEAR = 2,
  MMPR_MODEL_DOUBLE_WELL = 3,
  MMPR_MODEL_CUBIC_MF = 4,
  MMPR_MODEL_DW_MULT = 5,
  MMPR_MODEL_ROTATOR = 6,
  MMPR_MODEL_BURGERS = 7
};

/* Interaction statistics (models.py:30-33, ensemble_statistic :61-83). */
enum {
  MMPR_STAT_MEAN_OF_F = 0,     /* np.mean(x) (f = identity) */
  MMPR_STAT_EMPIRICAL_CDF = 1, /* per-particle mid-rank CDF, stable argsort */
  MMPR_STAT_ROTATOR_SUM = 2    /* (np.mean(sin x), np.mean(cos x)) */
};

typedef struct {
  int32_t kind;
  int32_t stat_kind; /* MMPR_STAT_*; mmpr_fine_sweep takes MEAN_OF_F, the
                        other two go through mmpr_fine_sweep_stepwise */
  double p[MMPR_MAX_PARAMS];
} mmpr_model;

/* Half-open regions [s_{i-1}, s_i) (state.py:13-78); a particle on a
 * separatrix belongs to the right region (searchsorted side="right"). */
typedef struct {
  int32_t n_regions;                   /* 1..MMPR_MAX_REGIONS */
  int32_t pad;
  double seps[MMPR_MAX_REGIONS - 1];   /* strictly increasing */
  double centers[MMPR_MAX_REGIONS];    /* RegionPartition.center(i) */
} mmpr_partition;

/* Moment ODE (coarse propagator) on the packed state [M_1..M_I, S_1..S_I,
 * a_1..a_I] (moments.py:29-49):
 *  UNIMODAL        unimodal_rhs(model) (moments.py:52-68), I = 1
 *  PERTURBED_OU    perturbed_ou_rhs(spec) (moments.py:111-125):
 *                  p = {mean_rate, var_rate, var_source}, I = 1
 *  MULTIMODAL      multimodal_rhs(model, ...) (moments.py:145-192):
 *                  p = {targets[I], rates[I]}
 *  GAUSSIAN_CUBIC  builder Gaussian closure for CUBIC_MF (BASELINE config 2):
 *                  p = {c1, c3, cE, sigma}, I = 1
 *  TAYLOR          taylor_enriched_rhs(model) for a MEAN_OF_F model without
 *                  its own closure (moments.py:71-108), I = 1
 *  ROTATOR_TAYLOR  the plane rotator's enriched closure (models.py:299-306):
 *                  p = {K, sigma_sq}, I = 1; status MMPR_STAT_SINGULAR at
 *                  |sin M| or |cos M| < 1e-8 (SingularityError)
 *  BURGERS         burgers_rhs(sigma) (moments.py:128-142):
 *                  p = {sigma^2, -(2/sqrt(2 pi))}, I = 1 */
enum {
  MMPR_ODE_UNIMODAL = 1,
  MMPR_ODE_PERTURBED_OU = 2,
  MMPR_ODE_MULTIMODAL = 3,
  MMPR_ODE_GAUSSIAN_CUBIC = 4,
  MMPR_ODE_TAYLOR = 5,
  MMPR_ODE_ROTATOR_TAYLOR = 6,
  MMPR_ODE_BURGERS = 7
};

typedef struct {
  int32_t kind;
  int32_t n_regions;
  double p[MMPR_MAX_ODE_PARAMS];
} mmpr_moment_ode;

/* Coarse integrators: EULER is the fixed-step forward Euler the BASELINE
 * configs ask for (n = round((t1-t0)/dt) steps); DP54 restates
 * rk54.integrate (rk54.py:69-129). */
enum { MMPR_INTEG_EULER = 1, MMPR_INTEG_DP54 = 2 };

typedef struct {
  int32_t kind;
  int32_t max_steps;   /* DP54 budget */
  double dt;           /* EULER step */
  double rel_tol;      /* DP54 */
  double abs_tol;      /* DP54 */
  double first_step;   /* DP54; <= 0 selects the initial-step heuristic */
} mmpr_integrator;

/* Status codes written to device status arrays: MMPR_STAT_OK, else the
 * failing step / region (fine sweep, match) or, for the coarse propagator,
 * MMPR_STAT_INTEG_FAILED (IntegrationFailure) / MMPR_STAT_SINGULAR
 * (SingularityError). */
#define MMPR_STAT_OK (-1)
/* the iteration pipeline's watchdog expired (a dependency never arrived):
 * written to every bad/match status of the units that ran after it */
#define MMPR_STAT_WATCHDOG (-2)

/* Counter-based Philox noise (NoiseMode.PHILOX / PHILOX_FRESH): the
 * increment of particle p at step j of global slice n is numpy's ziggurat
 * transform over Philox2x32-10 words (counter = (p, j | draw << 24),
 * key = key[0] ^ (n | kfield << 20)), generated in registers by the fine
 * kernels -- no increment buffer (paper_2310_11365_b200/csrc/
 * counter_noise.cuh).  Replaces the materialised NoisePlan.normals rows
 * (particles.py:49-61) where the north star's in-register noise is wanted;
 * statistically, not bitwise, equivalent to the reference's numpy streams.
 * Limits: n < 2^20, j < 2^24, particles < 2^32. */
typedef struct mmpr_counter_noise {
  uint32_t key[2];       /* key[0] = SeedSequence((seed, 4)).generate_state(1, uint32); key[1] unused */
  uint32_t kfield;       /* 0 = frozen, iteration + 1 = fresh (< 2^12) */
  int32_t slice_offset;  /* global index of local slice 0 */
} mmpr_counter_noise;
#define MMPR_STAT_INTEG_FAILED 1
#define MMPR_STAT_SINGULAR 2

/* ------------------------------------------------------------------ */
/* Library / device queries (host-synchronous)                         */
/* ------------------------------------------------------------------ */

/* Version string of the build ("mmpr <git-describe> sm_100a"). */
const char *mmpr_version(void);

/* Last CUDA error string recorded by a failing call on this thread. */
const char *mmpr_last_error(void);

/* Kernels this library has launched in this process so far (every launch
 * site counts; a call may launch several).  Host-side bookkeeping for the
 * benchmark's launch claim; nothing in the reference corresponds to it. */
uint64_t mmpr_kernel_launches(void);

/* mmpr_fine_sweep / mmpr_fine_sweep_restrict with counter-based Philox
 * increments generated in registers (no xi buffer).  stats/counts may be
 * NULL (no fused restriction). */
int mmpr_fine_sweep_counter(const mmpr_model *model, int32_t n_slices, int64_t particles, int32_t steps,
                            double dt, double sqrt_dt, const double *t0, const double *x_in,
                            int64_t in_pitch, double *x_out, int64_t out_pitch,
                            const mmpr_counter_noise *noise, int32_t *bad_step, double *stats,
                            int64_t *counts, void *stream);

/* Counter-mode increments written out (parity tests): out[r*pitch + i] =
 * increment of particle p0 + i at step j0 + r of global slice n. */
int mmpr_counter_normals_fill(const mmpr_counter_noise *noise, int32_t n, int32_t j0, int32_t rows,
                              int64_t p0, int64_t count, double *out, int64_t pitch, void *stream);

/* The interaction statistic of the ROTATOR_SUM / EMPIRICAL_CDF kinds
 * (models.ensemble_statistic, models.py:61-83): stat[2n], stat[2n+1] =
 * (np.mean(sin x_n), np.mean(cos x_n)) in numpy's pairwise order, or
 * stat[n*P + i] = (rank_i + 0.5) / P with ranks from a stable argsort.
 * workspace = NULL queries *workspace_bytes. */
int mmpr_ensemble_statistic(const mmpr_model *model, int32_t n_slices, int64_t particles, const double *x,
                            int64_t pitch, double *stat, void *workspace, uint64_t *workspace_bytes, void *stream);

/* Max concurrently resident clusters of the fine-sweep kernel for P
 * particles per slice (cudaOccupancyMaxActiveClusters). */
int mmpr_fine_sweep_occupancy(int64_t particles, int32_t *clusters_out, int32_t *ctas_per_slice_out);

/* ------------------------------------------------------------------ */
/* Noise: numpy-exact Philox4x64 + SeedSequence + ziggurat streams     */
/* replaces NoisePlan._generator/normals/init_rng (particles.py:49-65) */
/* ------------------------------------------------------------------ */

/* Philox keys of SeedSequence(entropy).generate_state(2, uint64) for the
 * step-noise addresses: FROZEN (seed, 1, n, j) / FRESH (seed, 2, n, j, k),
 * n in [n_offset, n_offset+n_slices), j in [0, steps).  keys: device
 * uint64[n_slices][steps][2]. (particles.py:52-61) */
int mmpr_noise_keys(uint64_t master_seed, int32_t fresh, int32_t iteration,
                    int32_t n_offset, int32_t n_slices, int32_t steps,
                    uint64_t *keys, void *stream);

/* Philox key of an arbitrary entropy tuple given as its assembled uint32
 * words (host array), written to device uint64[2]. */
int mmpr_entropy_key(const uint32_t *words, int32_t n_words, uint64_t *key_dev, void *stream);

/* Fill n_streams rows of `count` numbers: out[r*pitch + i] = loc + scale*z_i
 * where z is Generator(Philox(key_r)).standard_normal(count) bit-for-bit
 * (affine = 0 writes z itself).  keys: device uint64[n_streams][2].
 * Replaces Generator.standard_normal / Generator.normal
 * (particles.py:61, models.py:257). */
int mmpr_normals_fill(const uint64_t *keys, int32_t n_streams, int64_t count,
                      double *out, int64_t pitch, int32_t affine, double loc,
                      double scale, void *stream);

/* Wedge tests of the ziggurat (numpy's `... < exp(-x*x/2)`) whose outcome
 * lay inside the band where CUDA's exp and the host libm's exp could
 * disagree (relative 2^-50 around the value); 0 means every accept/reject
 * decision equals numpy's.  reset != 0 zeroes the device counter. */
int mmpr_noise_exp_ambiguous(uint64_t *count, int32_t reset);

/* out[i] = log1p(x[i]) as the host C library computes it (glibc 2.39 FMA
 * build, restated bit for bit; numpy's tail draws call it through
 * npy_log1p).  Exposed for the parity tests of the tail path. */
int mmpr_log1p_libm(const double *x, double *out, int64_t n, void *stream);


/* ------------------------------------------------------------------ */
/* Fine propagator (particles.py:119-159, engine.py:110-124)           */
/* ------------------------------------------------------------------ */

/* Euler-Maruyama over `steps` steps for n_slices independent ensembles of
 * `particles` each, one thread-block cluster per slice, particles resident
 * in registers, per-step ensemble mean reduced in numpy's pairwise order.
 *  x_in  : device double, slice s at x_in + s*in_pitch (P values)
 *  x_out : device double, slice s at x_out + s*out_pitch
 *  xi    : device double increments, slice s step j at
 *          xi + s*xi_slice_pitch + j*xi_row_pitch (P values; row pitch even)
 *  t0    : device double[n_slices] slice start times
 *  bad_step : device int32[n_slices]; MMPR_STAT_OK or the first step whose
 *          positions were not all finite (NumericalBlowup(slice, step))
 *  final_mean : device double[n_slices] (may be NULL): mean of the output.
 * Ensembles larger than one 16-CTA cluster (P = 2^20) run the grid variant:
 * co-resident teams of CTAs exchanging per-step partials through a
 * library-owned device buffer, so two such launches must not run
 * concurrently on one device (stream order them). */
int mmpr_fine_sweep(const mmpr_model *model, int32_t n_slices, int64_t particles,
                    int32_t steps, double dt, double sqrt_dt, const double *t0,
                    const double *x_in, int64_t in_pitch, double *x_out,
                    int64_t out_pitch, const double *xi, int64_t xi_slice_pitch,
                    int64_t xi_row_pitch, int32_t *bad_step, double *final_mean,
                    void *stream);

/* mmpr_fine_sweep followed by the single-region restriction of every
 * slice-end ensemble (restrict(F_n), engine.py:205), fused into the sweep:
 * stats + 3*n = [np.mean, np.var, 1.0] of x_out row n, counts[n] = P
 * (counts may be NULL).  Written only for slices without a blow-up. */
int mmpr_fine_sweep_restrict(const mmpr_model *model, int32_t n_slices, int64_t particles,
                             int32_t steps, double dt, double sqrt_dt, const double *t0,
                             const double *x_in, int64_t in_pitch, double *x_out,
                             int64_t out_pitch, const double *xi, int64_t xi_slice_pitch,
                             int64_t xi_row_pitch, int32_t *bad_step, double *stats,
                             int64_t *counts, void *stream);

/* Fine sweep for the ROTATOR_SUM / EMPIRICAL_CDF models (plane rotator,
 * Burgers), same buffers and status convention as mmpr_fine_sweep (no
 * final_mean).  Step-synchronous: per EM step one statistic pass (pairwise
 * sin/cos means, or a stable segmented sort giving mid-rank CDF values) and
 * one update pass with the reference's post_step (np.mod(x, 2 pi)).
 * workspace == NULL: writes the required bytes to *workspace_bytes. */
int mmpr_fine_sweep_stepwise(const mmpr_model *model, int32_t n_slices, int64_t particles,
                             int32_t steps, double dt, double sqrt_dt, const double *x_in,
                             int64_t in_pitch, double *x_out, int64_t out_pitch,
                             const double *xi, int64_t xi_slice_pitch, int64_t xi_row_pitch,
                             int32_t *bad_step, void *workspace, uint64_t *workspace_bytes,
                             void *stream);

/* ------------------------------------------------------------------ */
/* Restriction / matching (particles.py:176-205, coupling.py:26-95)    */
/* ------------------------------------------------------------------ */

/* Per-region fraction, mean and two-pass population variance of n_ens
 * ensembles, numpy summation order.  stats: device double[n_ens][3I] packed
 * [means, variances, fractions]; counts: device int64[n_ens][I]; scratch:
 * device double, >= mmpr_restrict_scratch_doubles(n_ens, particles, I)
 * values when I > 1 (NULL when I = 1). */
int mmpr_restrict(const mmpr_partition *part, int32_t n_ens, int64_t particles,
                  const double *x, int64_t pitch, double *stats, int64_t *counts,
                  double *scratch, void *stream);

/* Scratch (in doubles) mmpr_restrict needs for n_regions > 1: the region
 * arrays compacted in index order plus per-chunk counts and subtree
 * partials of the multi-CTA reduction; 0 for one region. */
int64_t mmpr_restrict_scratch_doubles(int32_t n_ens, int64_t particles, int32_t n_regions);

/* Per-region affine match x -> sqrt(var_t/var_c)(x - M_c) + mu_t with the
 * reference's clamp / degenerate / identity rules.  Ensemble e reads source
 * x_src + e*src_pitch (src_pitch 0: one shared source, e.g. lift from ens0),
 * its current moments cur_stats + e*cur_stride (packed 3I) and counts
 * cur_counts + e*cnt_stride (I), the target targets + e*tgt_stride (packed
 * 3I, fractions ignored), and writes x_out + e*out_pitch.
 *  policy: 0 = raise (DegenerateMatch), 1 = collapse
 *  status: device int32[n_ens]: MMPR_STAT_OK or the first degenerate region
 *  clamped: device int32[n_ens] (may be NULL): bit i set when region i's
 *          target variance was negative and clamped to 0 */
int mmpr_match(const mmpr_partition *part, int32_t n_ens, int64_t particles,
               const double *targets, int64_t tgt_stride, const double *cur_stats,
               int64_t cur_stride, const int64_t *cur_counts, int64_t cnt_stride,
               const double *x_src, int64_t src_pitch, double *x_out, int64_t out_pitch,
               int32_t policy, int32_t *status, int32_t *clamped, void *stream);

/* Single-region match followed by the restriction of the matched ensembles,
 * fused (engine.py:232-238: match then micro_stats = restrict): arguments of
 * mmpr_match for a one-region partition, plus stats + 3*e = [np.mean, np.var,
 * 1.0] of x_out row e and counts[e] = P (counts may be NULL). */
int mmpr_match_restrict(int32_t n_ens, int64_t particles, const double *targets,
                        int64_t tgt_stride, const double *cur_stats, int64_t cur_stride,
                        const int64_t *cur_counts, int64_t cnt_stride, const double *x_src,
                        int64_t src_pitch, double *x_out, int64_t out_pitch, int32_t policy,
                        int32_t *status, int32_t *clamped, double *stats, int64_t *counts,
                        void *stream);

/* mmpr_match (any partition) and the per-region restriction of the
 * matched ensembles in one pass, one thread-block cluster per ensemble:
 * regions of the matched positions, their members compacted in index order
 * into scratch (double[n_ens][I][particles]), each region's pairwise tree
 * over its compacted members -> stats[e][3I], counts[e][I] (as
 * mmpr_restrict).  Beyond one cluster the two separate calls run.  The
 * multi-region mmpr_restrict uses the same cluster kernel when it fits. */
int mmpr_match_restrict_regions(const mmpr_partition *part, int32_t n_ens, int64_t particles,
                                const double *targets, int64_t tgt_stride,
                                const double *cur_stats, int64_t cur_stride,
                                const int64_t *cur_counts, int64_t cnt_stride,
                                const double *x_src, int64_t src_pitch, double *x_out,
                                int64_t out_pitch, int32_t policy, int32_t *status,
                                int32_t *clamped, double *stats, int64_t *counts,
                                double *scratch, void *stream);

/* ------------------------------------------------------------------ */
/* Coarse propagator and Parareal correction (moments.py:195-203,      */
/* engine.py:170-236), one warp, no host round-trip                    */
/* ------------------------------------------------------------------ */

/* One macro row of the mM iteration for n_slices slices (times: device
 * double[n_slices+1]).  iteration == 0: pure coarse cascade from rho0.
 * iteration >= 1: corrected_n = fine_n + (C(macro_n) - cache_in_n), negative
 * variances clamped, fractions replaced by fine_n's.
 *  rho0       : device double[3I]
 *  fine_stats : device double[n][3I] (iteration >= 1)
 *  cache_in   : device double[n][3I] (iteration >= 1)
 *  macro_out  : device double[n+1][3I] (row 0 = rho0)
 *  cache_out  : device double[n][3I] this row's coarse predictions
 *  raw_out    : device double[n][3I] uncorrected-clamp corrected states (>= 1)
 *  status     : device int32[n]: MMPR_STAT_OK or 1 = IntegrationFailure
 *  skip_until : predictions for n < skip_until are copied from cache_in
 *               (bitwise equal by construction; 0 disables). */
int mmpr_coarse_row(const mmpr_moment_ode *ode, const mmpr_model *model,
                    const mmpr_integrator *integ, int32_t n_slices,
                    const double *times, int32_t iteration, const double *rho0,
                    const double *fine_stats, const double *cache_in,
                    double *macro_out, double *cache_out, double *raw_out,
                    int32_t *status, int32_t skip_until, void *stream);

/* integrate_macro(ode, state, t0, t1, cfg) for n_states independent states
 * (moments.py:195-203): in/out device double[n_states][3I]. */
int mmpr_integrate_macro(const mmpr_moment_ode *ode, const mmpr_model *model,
                         const mmpr_integrator *integ, int32_t n_states,
                         const double *t0, const double *t1, const double *state_in,
                         double *state_out, int32_t *status, void *stream);

/* ------------------------------------------------------------------ */
/* Iterations 1..K of run_micro_macro in one persistent kernel         */
/* (engine.py:197-238: fine sweep, serial correction, match, micro     */
/* restriction of every iteration, dependency-driven per (k, n) unit)  */
/* ------------------------------------------------------------------ */

/* Device buffers of one run (all caller-owned; shapes in doubles/ints).
 * The prologue (iteration 0: rho0 = R(ens0), macro/cache row 0 by
 * mmpr_coarse_row, the lifted snapshot row 0 with micro row 0, the
 * increments) must already be on the stream; the pipeline writes every
 * row k >= 1 of macro/micro/micro_counts/cache/coarse_status/match_status,
 * all rows of fine_stats/fine_counts/raw/bad, and snapshot rows 1..K. */
#define MMPR_COUNTER_FRESH 0xFFFFFFFFu

typedef struct mmpr_pipeline_io {
  const double *times;        /* [N+1] slice boundaries */
  const double *x0;           /* [P] ens0 */
  const double *rho0;         /* [3I] R(ens0) */
  const int64_t *counts0;     /* [I] */
  const double *xi;           /* increments, slice n step j at xi + n*xi_slice_pitch + j*xi_row_pitch */
  int64_t xi_slice_pitch, xi_row_pitch;
  double *snap;               /* snapshot row k slice n at snap + k'*snap_iter_stride + n*snap_slice_pitch */
  int64_t snap_iter_stride, snap_slice_pitch;
  int32_t snap_rows;          /* K+1 (k' = k) or 2 (k' = k % 2, retain_snapshots=False) */
  double *fine;               /* [2][N] rows of fine_pitch: F^k_n in row (k%2)*N + n */
  int64_t fine_pitch;
  double *macro;              /* [K+1][N+1][3I] (I regions: means, variances, fractions) */
  double *micro;              /* [K+1][N+1][3I] */
  int64_t *micro_counts;      /* [K+1][N+1][I] */
  double *fine_stats;         /* [K][N][3I] */
  int64_t *fine_counts;       /* [K][N][I] */
  double *raw;                /* [K][N][3I] */
  double *cache;              /* [K+1][N][3I] (row 0 from the prologue) */
  int32_t *bad;               /* [K][N] */
  int32_t *coarse_status;     /* [K+1][N] */
  int32_t *match_status;      /* [K+1][N] */
  int32_t *flags;             /* [mmpr_pipeline_flags_size(N, K)] scratch, reset by the call */
  int32_t counter_noise;      /* 1: increments from counter-based Philox (xi unused; see
                                 mmpr_counter_noise), 0: from xi */
  uint32_t counter_key[2];
  uint32_t counter_kfield;    /* 0: frozen; MMPR_COUNTER_FRESH: fresh, iteration k's fine parts
                                 draw with kfield k + 1 (as mmpr_counter_noise of iteration k) */
  /* two-region runs (ode->n_regions == 2, one rank; particles.region_statistics
   * and the per-region coupling.match inside the units): */
  mmpr_partition partition;   /* the run's partition (n_regions == ode->n_regions) */
  double *region_scratch;     /* [region_scratch_rows][n_regions][P] compacted region members */
  int64_t region_scratch_rows; /* persistent clusters the launch may use (>= 1) */
  int64_t *fine_times;        /* optional [K][N][2]: globaltimer ns at the start and end of each
                                 unit's fine propagation (NULL: not recorded) */
} mmpr_pipeline_io;

/* int32 scratch words the pipeline needs for (n_slices, iterations). */
int64_t mmpr_pipeline_flags_size(int32_t n_slices, int32_t iterations);

/* Per-slice timestamps of the next fine sweeps (mmpr_fine_sweep,
 * mmpr_fine_sweep_restrict, mmpr_fine_sweep_counter) launched from the
 * calling host thread: globaltimer ns at the start and the end of slice s's
 * propagation go to slice_times[2s], slice_times[2s+1] (the reference's
 * per-slice fine timings, engine.py:110-124 / :204).  NULL stops recording.
 * The pointer is bound when a launch is issued (a captured graph keeps it). */
int mmpr_set_fine_times(int64_t *slice_times);

/* MMPR_OK when (model, ode, ode_model, integrator, particles) has a pipeline
 * instantiation (MEAN_OF_F, forward-Euler coarse, an ensemble of one
 * cluster: 4096 < P <= 2^17 with a balanced pairwise tree -- specialised for
 * 13, 10 or 16 accumulator elements per lane: P = 1e5 / 1e4 and their binary
 * fractions / multiples, powers of two from 2^13 to 2^17 -- and an any-size
 * form otherwise; one region, or two regions for
 * the double well with the multimodal closure on one rank); else
 * MMPR_ERR_UNSUPPORTED
 * and the caller runs the per-iteration kernels. */
int mmpr_pipeline_supported(const mmpr_model *model, const mmpr_moment_ode *ode,
                            const mmpr_model *ode_model, const mmpr_integrator *integ,
                            int64_t particles);

/* The same for a given noise supply and rank count: the two-region units and
 * every geometry but the 13-element one exist for
 * one rank with numpy-stream or injected increments only (counter_noise = 0,
 * n_ranks = 1).  Replaces nothing in the reference (engine.py:127-259 has no
 * such switch); the host uses it to choose between the pipeline and the
 * per-iteration kernels. */
int mmpr_pipeline_supported_ex(const mmpr_model *model, const mmpr_moment_ode *ode,
                               const mmpr_model *ode_model, const mmpr_integrator *integ,
                               int64_t particles, int32_t counter_noise, int32_t n_ranks);

/* Runs iterations 1..iterations (raise policy for the matches, predictions
 * of converged slices reused when reuse_converged != 0, as mmpr_coarse_row's
 * skip_until).  Bitwise identical to the per-iteration kernel sequence. */
int mmpr_parareal_pipeline(const mmpr_model *model, const mmpr_moment_ode *ode,
                           const mmpr_model *ode_model, const mmpr_integrator *integ,
                           int32_t n_slices, int32_t iterations,
                           int64_t particles, int32_t steps, double dt, double sqrt_dt,
                           int32_t reuse_converged, const mmpr_pipeline_io *io, void *stream);

/* The same pipeline over n_ranks ranks, each owning n_slices / n_ranks
 * contiguous slices (the last rank also boundary N): ios[r] are rank r's
 * buffers, every array indexed by GLOBAL slice/boundary (rank r writes only
 * the entries of its own units), except xi, which holds rank r's own slices
 * (slice n at xi + (n - r*Ng)*xi_slice_pitch).  The launch processes the
 * units of ranks [first_rank, first_rank + launch_ranks) in (k, n) order and
 * reads the first slice's inputs of each rank -- F^{k-1}_{n-1}, its
 * restriction, macro[k][n-1] -- from the previous rank's buffers, waiting on
 * that rank's flag words; the only cross-rank traffic is one ensemble and a
 * few doubles per (rank boundary, iteration).
 *  - multi-GPU: each process launches its own rank (launch_ranks = 1) with
 *    the other ranks' ios pointing into their exchange memory opened with
 *    mmpr_ipc_open (flags, macro, fine_stats, fine_counts, fine); multi_gpu=1
 *    selects system-scope release/acquire;
 *  - one GPU: one launch over all ranks (first_rank = 0, launch_ranks =
 *    n_ranks) -- the emulation the tests use.
 * Flags accumulate across runs: run `epoch` (1, 2, ...) waits for epoch
 * times the per-run count, so no rank resets a word a peer may still read;
 * reset_flags=1 (epoch 1 only) zeroes the launch's flags first.  The ticket
 * word (flags[0] of ios[first_rank]) is reset by every call. */
int mmpr_parareal_pipeline_ranks(const mmpr_model *model, const mmpr_moment_ode *ode,
                                 const mmpr_model *ode_model, const mmpr_integrator *integ,
                                 int32_t n_slices, int32_t iterations, int64_t particles,
                                 int32_t steps, double dt, double sqrt_dt, int32_t reuse_converged,
                                 int32_t n_ranks, const mmpr_pipeline_io *ios, int32_t first_rank,
                                 int32_t launch_ranks, int32_t epoch, int32_t reset_flags,
                                 int32_t multi_gpu, void *stream);

/* Exchange memory of the multi-GPU pipeline: a cudaMalloc'd block (so one
 * IPC handle covers it), its 64-byte cudaIpcMemHandle, and the peer
 * mapping of another process's block (cudaIpcMemLazyEnablePeerAccess). */
int mmpr_exchange_alloc(int64_t bytes, void **dev_ptr);
int mmpr_exchange_free(void *dev_ptr);
int mmpr_ipc_handle(void *dev_ptr, unsigned char *handle_out);
int mmpr_ipc_open(const unsigned char *handle, void **dev_ptr);
int mmpr_ipc_close(void *dev_ptr);
int mmpr_device_can_access_peer(int32_t device, int32_t peer, int32_t *out);

/* ------------------------------------------------------------------ */
/* Error metrics (metrics.py:35-47, 73-130, 133-218)                   */
/* ------------------------------------------------------------------ */

/* Sort each of n_rows rows (count doubles at in + r*pitch) ascending into
 * out + r*pitch (np.sort; ties are equal values, so the result is unique up
 * to the order of +0.0/-0.0).  temp == NULL: writes the required temporary
 * bytes to *temp_bytes and returns; else temp is a device buffer of
 * *temp_bytes bytes.  Replaces the np.sort calls of wasserstein_1d and
 * floor_from_references (metrics.py:46, 185). */
int mmpr_sort_rows(int32_t n_rows, int64_t count, const double *in, double *out,
                   int64_t pitch, void *temp, uint64_t *temp_bytes, void *stream);

/* out[r] = np.mean(np.abs(a_r - b_r)) over count doubles (numpy pairwise
 * order), a_r = a + r*pitch_a, b_r = b + r*pitch_b: the W1 distance of two
 * sorted equally sized samples (metrics.py:35-47). */
int mmpr_mean_abs_diff(int32_t n_rows, int64_t count, const double *a, int64_t pitch_a,
                       const double *b, int64_t pitch_b, double *out, void *stream);

/* Cumulative histogram of sorted rows (np.histogram with explicit edges,
 * harness.py:314-316): cum[r*n_edges + e] = #{x in row r : x < edges[e]},
 * the last edge inclusive (x <= edges[n_edges-1]); bin counts are the
 * differences.  NaNs (sorted last) are never counted. */
int mmpr_histogram_sorted(int32_t n_rows, int64_t count, const double *sorted, int64_t pitch,
                          const double *edges, int32_t n_edges, int64_t *cum, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* MMPR_H */
