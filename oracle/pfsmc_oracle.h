/* Plain-C restatement of the reference LMM PF-SMC per-step update.
 *
 * TEST INFRASTRUCTURE — the checker, never the product. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
 * load liboracle.so. Parity of this restatement is pinned against the
 * unmodified reference (oracle/_ref/libpfsmc_ref.so, built from
 * /root/reference/proj/src by oracle/Makefile) and against the reference's
 * own golden vectors (tests/golden/, see tests/test_oracle.py).
 *
 * Every function cites the reference file:line it restates. Arithmetic is
 * written in the reference's evaluation order and compiled without FP
 * contraction (the reference's build has no FMA: CMakeLists.txt:7-9).
 */
#ifndef PFSMC_ORACLE_H
#define PFSMC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_INTERNAL = 1, OR_CONFIG = 2, OR_NUMERICAL = 3 };
enum { OR_PURPOSE_INIT = 0, OR_PURPOSE_PROLIFERATE = 1, OR_PURPOSE_INNOVATE = 2,
       OR_PURPOSE_RESAMPLE = 3 };
enum { OR_AB = 0, OR_AM = 1, OR_BDF = 2 };
enum { OR_MODEL_DECAY = 0, OR_MODEL_LV = 1, OR_MODEL_ROBERTSON = 2, OR_MODEL_CHAIN = 3,
       OR_MODEL_METABOLIC = 5 /* the reference's models::MetabolicModel (models.cpp:37-119) */,
       OR_MODEL_ADVDIFF = 6   /* the reference's models::AdvDiffModel (models.cpp:158-266):
                                 d = (n-1)^2, p = 5, grid parameter n = model const 0 */ };
enum { OR_LIK_GAUSSIAN = 0, OR_LIK_LOGNORMAL = 1 };
enum { OR_ST_OK = 0, OR_ST_INVALID_RHS = 1, OR_ST_NEWTON_DIVERGENCE = 2,
       OR_ST_SINGULAR = 3, OR_ST_STIFFNESS = 4 };

#define OR_MAX_D 1024 /* advdiff: n <= 33 */
#define OR_MAX_P 8

typedef struct or_cfg {
  int model;
  int family;
  int order;
  double h;
  double a;
  uint64_t seed;
  double newton_tol;
  int newton_max_iter;
  const uint64_t* obs_idx;
  uint64_t m_y;
  double sigma;
  int likelihood; /* OR_LIK_* ; lognormal is an extension */
  int adaptive;   /* IntegratorSpec.adaptive: variable-step BDF(1,2) (lmm.cpp:894-1019) */
  double rtol;    /* IntegratorSpec.rtol (adaptive only) */
} or_cfg;

typedef struct or_ens {
  uint64_t n, d, p;
  double* states;   /* n*d row-major */
  double* params_u; /* n*p row-major, unconstrained (log for positive) */
  double* logw;     /* n, normalised */
  double* mean_u;   /* p */
  double* cov_u;    /* p*p */
} or_ens;

/* Optional per-step diagnostics (any pointer may be NULL). */
typedef struct or_step_out {
  double* trace;       /* theta_mean[p], theta_var[p], state_mean[d], ess */
  int64_t* ancestors;  /* n */
  double* loglik_bar;  /* n, predictor log-likelihood (before reshuffle) */
  double* g;           /* n, fitness weights */
  double* gamma;       /* n*d, repropagation LTE variance (slot order) */
  int* status_new;     /* n, repropagation status (slot order) */
  int* newton_iters;   /* n, predictor + repropagation Newton iterations */
} or_step_out;

const char* or_last_error(void);
void or_philox4x64(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
int or_stream_draws(uint64_t seed, uint64_t j, uint64_t n, int purpose, int kind,
                    uint64_t count, void* out);
int or_model_dims(int model, int* d, int* p);
int or_rhs(int model, const double* theta_nat, const double* x, double* f);
/* Constants of the bound model (METABOLIC: lambda, c0, A0, A, t0_input, tau;
 * ADVDIFF: grid parameter n). */
void or_set_model_consts(const double* k);
/* models::gaussian_plume_ic (models.cpp:130-156): the advdiff truth x(0), (n-1)^2 values. */
int or_gaussian_plume_ic(int n, double* out);
/* AdvDiffModel::assemble_operator (models.cpp:251-261) as a dense d x d row-major
 * matrix (test helper). */
int or_advdiff_operator(int n, const double* theta_nat, double* dense_out);
int or_propagate_interval(int model, const double* theta_nat, const double* x0,
                          double t0, double t1, double h, int family, int order,
                          double tol, int max_iter, double* state_out,
                          double* gamma_out, int* status_out, int* iters_out);
int or_fitness_weights(const double* logw, const double* loglik, uint64_t n,
                       double* g);
int or_resample_multinomial(const double* g, uint64_t n, uint64_t seed,
                            uint64_t j, int64_t* out);
int or_weighted_mean_cov(const double* params, uint64_t n, uint64_t p,
                         const double* w, double* mean, double* cov);
int or_chol_psd(const double* cov, uint64_t p, double* lower, double* jitter);
double or_log_likelihood(const or_cfg* c, const double* y, const double* x);
int or_pf_step(const or_cfg* c, or_ens* e, const double* y, uint64_t j,
               double t_prev, double t_obs, or_step_out* out);
/* Uniform-box prior in natural space (BASELINE configs 1, 2, 4): for particle
 * i one stream (seed, 0, i, init) draws p uniforms for theta then d uniforms
 * for x; theta_u = log(U) for positive params; moments with w = 1/N as in
 * filter.cpp:101-103. */
int or_init_uniform(int model, uint64_t n, uint64_t seed, const double* th_lo,
                    const double* th_hi, const double* x_lo, const double* x_hi,
                    or_ens* e);
/* Gaussian prior in unconstrained space: filter::initialize (filter.cpp:76-105). */
int or_init_gaussian(int model, uint64_t n, uint64_t seed, const double* th_mu,
                     const double* th_sigma, const double* x_mean,
                     const double* x_std, const int* x_clamp, or_ens* e);

#ifdef __cplusplus
}
#endif
#endif
