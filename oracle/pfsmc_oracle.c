/* Plain-C restatement of the reference LMM PF-SMC per-step update
 * (/root/reference/proj, C++20). TEST INFRASTRUCTURE ONLY — see
 * pfsmc_oracle.h for the rules. Parity pinned against the unmodified
 * reference (oracle/_ref) and its golden vectors (tests/test_oracle.py).
 *
 * Conventions restated from the reference:
 *   - std::max(a, b) is (a < b) ? b : a  (NaN-propagation matters:
 *     filter.cpp:18, lmm.cpp:210-211);
 *   - every sum is the reference's left-to-right sequential sum;
 *   - compiled with -ffp-contract=off (no FMA, as CMakeLists.txt:7-9).
 */
#include "pfsmc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static _Thread_local char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* or_last_error(void) { return g_err; }

static inline double dmax(double a, double b) { return (a < b) ? b : a; }

/* Per-particle loops over host threads (the reference maps particles over its
 * thread pool, filter.cpp:234-265; exec.cpp:183-212): chunks of 256 indices
 * handed out by an atomic counter. The arithmetic per particle is unchanged,
 * so results do not depend on the thread count. ORACLE_THREADS=1 runs it
 * inline. */
typedef void (*par_body)(void* ctx, uint64_t i);
typedef struct {
  par_body f;
  void* ctx;
  uint64_t n;
  atomic_ullong next;
} par_job;
static void* par_worker(void* arg) {
  par_job* jb = (par_job*)arg;
  for (;;) {
    const uint64_t i0 = atomic_fetch_add(&jb->next, 256);
    if (i0 >= jb->n) break;
    const uint64_t i1 = i0 + 256 < jb->n ? i0 + 256 : jb->n;
    for (uint64_t i = i0; i < i1; ++i) jb->f(jb->ctx, i);
  }
  return NULL;
}
static int par_threads(void) {
  const char* e = getenv("ORACLE_THREADS");
  long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  if (t < 1) t = 1;
  if (t > 64) t = 64;
  return (int)t;
}
static void par_for(uint64_t n, par_body f, void* ctx, int allow_threads) {
  const int T = allow_threads ? par_threads() : 1;
  if (T == 1 || n < 2048) {
    for (uint64_t i = 0; i < n; ++i) f(ctx, i);
    return;
  }
  par_job jb;
  jb.f = f;
  jb.ctx = ctx;
  jb.n = n;
  atomic_init(&jb.next, 0);
  pthread_t th[64];
  int started = 0;
  for (int t = 1; t < T; ++t)
    if (pthread_create(&th[started], NULL, par_worker, &jb) == 0) ++started;
  par_worker(&jb);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* RNG: Philox4x64-10 and keyed streams (rng.cpp:9-75)                       */
/* ------------------------------------------------------------------------ */
#define K_MULT0 0xD2E7470EE14C6C93ULL
#define K_MULT1 0xCA5A826395121157ULL
#define K_WEYL0 0x9E3779B97F4A7C15ULL
#define K_WEYL1 0xBB67AE8584CAA73BULL
#define K_KEYC 0x7066736D632D3031ULL /* "pfsmc-01", rng.cpp:16 */

/* rng.cpp:28-41 */
void or_philox4x64(const uint64_t ctr_in[4], const uint64_t key_in[2],
                   uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += K_WEYL0;
      k1 += K_WEYL1;
    }
    const unsigned __int128 p0 = (unsigned __int128)K_MULT0 * c0;
    const unsigned __int128 p1 = (unsigned __int128)K_MULT1 * c2;
    const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

typedef struct stream {
  uint64_t key[2];
  uint64_t ctr[4];
  uint64_t block[4];
  uint64_t block_index;
  int lane;
  int have_spare;
  double spare;
} stream;

/* rng.cpp:43-46 */
static void stream_init(stream* s, uint64_t seed, uint64_t j, uint64_t n,
                        int purpose) {
  s->key[0] = seed; s->key[1] = K_KEYC;
  s->ctr[0] = 0; s->ctr[1] = j; s->ctr[2] = n; s->ctr[3] = (uint64_t)purpose;
  s->block_index = 0; s->lane = 4; s->have_spare = 0; s->spare = 0.0;
}
/* rng.cpp:48-55 */
static uint64_t next_u64(stream* s) {
  if (s->lane == 4) {
    s->ctr[0] = s->block_index++;
    or_philox4x64(s->ctr, s->key, s->block);
    s->lane = 0;
  }
  return s->block[s->lane++];
}
/* rng.cpp:57-59 */
static double next_uniform(stream* s) {
  return (double)(next_u64(s) >> 11) * 0x1.0p-53;
}
/* rng.cpp:61-75 */
static double next_normal(stream* s) {
  if (s->have_spare) {
    s->have_spare = 0;
    return s->spare;
  }
  const double u1 = ((double)(next_u64(s) >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = next_uniform(s);
  const double r = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.14159265358979323846 * u2;
  s->spare = r * sin(angle);
  s->have_spare = 1;
  return r * cos(angle);
}

int or_stream_draws(uint64_t seed, uint64_t j, uint64_t n, int purpose, int kind,
                    uint64_t count, void* out) {
  stream s;
  stream_init(&s, seed, j, n, purpose);
  for (uint64_t i = 0; i < count; ++i) {
    if (kind == 0) ((uint64_t*)out)[i] = next_u64(&s);
    else if (kind == 1) ((double*)out)[i] = next_uniform(&s);
    else ((double*)out)[i] = next_normal(&s);
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Models (oracle/ref/ref_models.hpp; plugin contract models.hpp:20-55)      */
/* ------------------------------------------------------------------------ */
static double g_mk_n(void);
int or_model_dims(int model, int* d, int* p) {
  switch (model) {
    case OR_MODEL_DECAY: *d = 1; *p = 1; return OR_OK;
    case OR_MODEL_LV: *d = 2; *p = 2; return OR_OK;
    case OR_MODEL_ROBERTSON: *d = 3; *p = 3; return OR_OK;
    case OR_MODEL_CHAIN: *d = 8; *p = 4; return OR_OK;
    case OR_MODEL_METABOLIC: *d = 3; *p = 4; return OR_OK;
    case OR_MODEL_ADVDIFF: {
      /* AdvDiffModel(n): m = n - 1, dim m^2, 5 params (models.cpp:185-188, 242-249) */
      const int n = (int)g_mk_n();
      if (n < 3) return fail(OR_CONFIG, "advdiff model: grid parameter n must be >= 3");
      if ((n - 1) * (n - 1) > OR_MAX_D) return fail(OR_CONFIG, "advdiff model: grid too large for the oracle");
      *d = (n - 1) * (n - 1);
      *p = 5;
      return OR_OK;
    }
  }
  return fail(OR_CONFIG, "unknown model id");
}

static int all_finite(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* Constants of the bound model (MetabolicConstants, models.hpp:67-74:
 * lambda, c0, A0, A, t0_input, tau), set with or_set_model_consts. */
static double g_mk[8] = {1.0, 1.0, 1.0, 5.0, 2.0, 1.0, 0.0, 0.0};

void or_set_model_consts(const double* k) {
  for (int i = 0; i < 8; ++i) g_mk[i] = k[i];
}

static double g_mk_n(void) { return g_mk[0]; }

/* ------------------------------------------------------------------------ */
/* AdvDiffModel (models.cpp:158-266) over linalg's CSR (linalg.cpp:24-200)   */
/* ------------------------------------------------------------------------ */
typedef struct csr {
  int nr, nc, nnz;
  int* ro;
  int* ci;
  double* v;
} csr;

static csr csr_alloc(int nr, int nc, int cap) {
  csr m;
  m.nr = nr; m.nc = nc; m.nnz = 0;
  m.ro = calloc((size_t)nr + 1, sizeof(int));
  m.ci = malloc(sizeof(int) * (size_t)(cap ? cap : 1));
  m.v = malloc(sizeof(double) * (size_t)(cap ? cap : 1));
  return m;
}
static void csr_free(csr* m) { free(m->ro); free(m->ci); free(m->v); m->ro = NULL; m->ci = NULL; m->v = NULL; }
static void csr_push(csr* m, int c, double v) { m->ci[m->nnz] = c; m->v[m->nnz] = v; ++m->nnz; }

/* CsrMatrix::identity (linalg.cpp:50-59) */
static csr csr_identity(int n) {
  csr m = csr_alloc(n, n, n);
  for (int i = 0; i < n; ++i) { csr_push(&m, i, 1.0); m.ro[i + 1] = m.nnz; }
  return m;
}
/* periodic_diff_matrix (linalg.cpp:89-113), scale 1: row 0 (+1 @0, -1 @n-1),
 * row i > 0 (-1 @i-1, +1 @i) */
static csr periodic_diff(int n) {
  csr m = csr_alloc(n, n, 2 * n);
  csr_push(&m, 0, 1.0);
  csr_push(&m, n - 1, -1.0);
  m.ro[1] = 2;
  for (int i = 1; i < n; ++i) {
    csr_push(&m, i - 1, -1.0);
    csr_push(&m, i, 1.0);
    m.ro[i + 1] = m.nnz;
  }
  return m;
}
/* kron (linalg.cpp:115-140) */
static csr csr_kron(const csr* a, const csr* b) {
  csr m = csr_alloc(a->nr * b->nr, a->nc * b->nc, a->nnz * b->nnz);
  for (int ia = 0; ia < a->nr; ++ia)
    for (int ib = 0; ib < b->nr; ++ib) {
      for (int ka = a->ro[ia]; ka < a->ro[ia + 1]; ++ka) {
        const int col_base = a->ci[ka] * b->nc;
        const double va = a->v[ka];
        for (int kb = b->ro[ib]; kb < b->ro[ib + 1]; ++kb) csr_push(&m, col_base + b->ci[kb], va * b->v[kb]);
      }
      m.ro[ia * b->nr + ib + 1] = m.nnz;
    }
  return m;
}
/* csr_add (linalg.cpp:142-180): merge of sorted rows; shared entries
 * v = 0 + alpha a, then v += beta b; a-only v = 0 + alpha a; b-only v = beta b. */
static csr csr_add(double alpha, const csr* a, double beta, const csr* b) {
  csr m = csr_alloc(a->nr, a->nc, a->nnz + b->nnz);
  for (int i = 0; i < m.nr; ++i) {
    int ka = a->ro[i], kb = b->ro[i];
    const int ea = a->ro[i + 1], eb = b->ro[i + 1];
    while (ka < ea || kb < eb) {
      int col;
      double v = 0.0;
      if (ka < ea && (kb >= eb || a->ci[ka] <= b->ci[kb])) {
        col = a->ci[ka];
        v += alpha * a->v[ka];
        ++ka;
        if (kb < eb && b->ci[kb] == col) { v += beta * b->v[kb]; ++kb; }
      } else {
        col = b->ci[kb];
        v = beta * b->v[kb];
        ++kb;
      }
      csr_push(&m, col, v);
    }
    m.ro[i + 1] = m.nnz;
  }
  return m;
}
/* AdvDiffModel's transpose_mul (models.cpp:196-233): G = A^T B, entries
 * summed per column after sorting. The operands are +-1 difference
 * matrices, so every product and sum is an exact small integer and the sort
 * order of equal columns cannot change a value. */
static csr csr_tmul(const csr* a, const csr* b) {
  const int nc = a->nc;
  double* acc = calloc((size_t)b->nc, sizeof(double));
  char* hit = calloc((size_t)b->nc, 1);
  csr g = csr_alloc(nc, b->nc, a->nnz * 4 + nc);
  /* rows[i] collects (col_b, va*vb) over k with A_ki != 0 */
  for (int i = 0; i < nc; ++i) {
    for (int k = 0; k < a->nr; ++k)
      for (int ia = a->ro[k]; ia < a->ro[k + 1]; ++ia) {
        if (a->ci[ia] != i) continue;
        const double va = a->v[ia];
        for (int ib = b->ro[k]; ib < b->ro[k + 1]; ++ib) {
          const int c = b->ci[ib];
          acc[c] = hit[c] ? acc[c] + va * b->v[ib] : va * b->v[ib];
          hit[c] = 1;
        }
      }
    for (int c = 0; c < b->nc; ++c)
      if (hit[c]) { csr_push(&g, c, acc[c]); hit[c] = 0; }
    g.ro[i + 1] = g.nnz;
  }
  free(acc); free(hit);
  return g;
}
/* spmv (linalg.cpp:182-194) */
static void csr_spmv(const csr* a, const double* x, double* y) {
  for (int i = 0; i < a->nr; ++i) {
    double sum = 0.0;
    for (int k = a->ro[i]; k < a->ro[i + 1]; ++k) sum += a->v[k] * x[a->ci[k]];
    y[i] = sum;
  }
}

/* The model's fixed matrices for grid m = n - 1 (AdvDiffModel ctor,
 * models.cpp:185-240): B1 = I (x) D, B2 = D (x) I, G11 = B1'B1, G22 = B2'B2,
 * G12 = B1'B2 + B2'B1; cached per n. */
static int g_adv_n = 0;
static csr g_b1, g_b2, g_g11, g_g22, g_g12;
static csr g_adv_L;     /* the bound operator (AdvDiffModel::bind) */
static int g_adv_bound = 0;

static void adv_build(int n) {
  if (g_adv_n == n) return;
  if (g_adv_n) {
    csr_free(&g_b1); csr_free(&g_b2); csr_free(&g_g11); csr_free(&g_g22); csr_free(&g_g12);
  }
  const int m = n - 1;
  csr ell = periodic_diff(m), eye = csr_identity(m);
  g_b1 = csr_kron(&eye, &ell);
  g_b2 = csr_kron(&ell, &eye);
  g_g11 = csr_tmul(&g_b1, &g_b1);
  g_g22 = csr_tmul(&g_b2, &g_b2);
  csr t12 = csr_tmul(&g_b1, &g_b2), t21 = csr_tmul(&g_b2, &g_b1);
  g_g12 = csr_add(1.0, &t12, 1.0, &t21);
  csr_free(&t12); csr_free(&t21); csr_free(&ell); csr_free(&eye);
  g_adv_n = n;
}

/* assemble_operator (models.cpp:251-261):
 *   L = -(k1^2 G11 + k1 k3 G12 + (k2^2 + k3^2) G22) + c1 B1 + c2 B2 */
static csr adv_assemble(const double* th) {
  adv_build((int)g_mk[0]);
  const double k1 = th[0], k2 = th[1], k3 = th[2], c1 = th[3], c2 = th[4];
  csr diff = csr_add(-(k1 * k1), &g_g11, -(k1 * k3), &g_g12);
  csr diff2 = csr_add(1.0, &diff, -(k2 * k2 + k3 * k3), &g_g22);
  csr adv = csr_add(c1, &g_b1, c2, &g_b2);
  csr L = csr_add(1.0, &diff2, 1.0, &adv);
  csr_free(&diff); csr_free(&diff2); csr_free(&adv);
  return L;
}
/* AdvDiffModel::bind for the particle being propagated (one at a time). */
static void adv_bind(const double* th) {
  if (g_adv_bound) csr_free(&g_adv_L);
  g_adv_L = adv_assemble(th);
  g_adv_bound = 1;
}

int or_advdiff_operator(int n, const double* theta_nat, double* dense_out) {
  if (n < 3) return fail(OR_CONFIG, "advdiff model: grid parameter n must be >= 3");
  const double keep = g_mk[0];
  g_mk[0] = (double)n;
  csr L = adv_assemble(theta_nat);
  g_mk[0] = keep;
  const int d = L.nr;
  memset(dense_out, 0, sizeof(double) * (size_t)d * (size_t)d);
  for (int i = 0; i < d; ++i)
    for (int k = L.ro[i]; k < L.ro[i + 1]; ++k) dense_out[(size_t)i * d + L.ci[k]] = L.v[k];
  csr_free(&L);
  return OR_OK;
}

/* gaussian_plume_ic (models.cpp:130-156) */
int or_gaussian_plume_ic(int n, double* u) {
  static const double kGamma[6] = {0.04, 0.08, 0.07, 0.10, 0.05, 0.06};
  static const double kXc[6] = {0.20, 0.30, 0.40, 0.50, 0.50, 0.70};
  static const double kYc[6] = {0.80, 0.40, 0.40, 0.50, 0.60, 0.50};
  const double kSqrt2Pi = 2.5066282746310002;
  if (n < 3) return fail(OR_CONFIG, "gaussian_plume_ic: n must be >= 3");
  const int m = n - 1;
  for (int iy = 0; iy < m; ++iy) {
    const double y = (double)iy / (double)m;
    for (int ix = 0; ix < m; ++ix) {
      const double x = (double)ix / (double)m;
      double sum = 0.0;
      for (int i = 0; i < 6; ++i) {
        const double dx = x - kXc[i];
        const double dy = y - kYc[i];
        sum += exp(-(dx * dx + dy * dy) / (2.0 * kGamma[i] * kGamma[i])) / (kGamma[i] * kSqrt2Pi);
      }
      u[iy * m + ix] = sum;
    }
  }
  return OR_OK;
}

/* The sparse Newton path's workspace (NewtonWorkspace, lmm.hpp:88-100): the
 * factorisation of I - hb0 L is cached while hb0 is unchanged
 * (lmm.cpp:233-243). The LU is the direct solver the oracle's Eigen stand-in
 * runs (oracle/ref/eigen_stub/Eigen/SparseLU): DenseLu's pivot rule. */
typedef struct sparse_ws {
  int valid;
  double hb0;
  double* lu;
  int* piv;
} sparse_ws;
static _Thread_local sparse_ws* g_sws = NULL;

/* input_phi (models.cpp:37-42) */
static double input_phi(double t, double A0, double A, double t0_input, double tau) {
  const double dt = t - t0_input;
  if (dt <= 0.0) return A0;
  return A0 + A * dt * exp(-dt / tau);
}

/* rhs(t, x) -> f; returns 0 when undefined/non-finite (models.hpp:24-27). */
static int model_rhs(int model, double t, const double* th, const double* x, double* o) {
  switch (model) {
    case OR_MODEL_METABOLIC: { /* metabolic_rhs (models.cpp:44-57) */
      const double den1 = x[0] + th[1];
      const double den2 = x[1] + th[3];
      if (den1 <= 0.0 || den2 <= 0.0) return 0;
      const double flux1 = th[0] * x[0] / den1;
      const double flux2 = th[2] * x[1] / den2;
      o[0] = input_phi(t, g_mk[2], g_mk[3], g_mk[4], g_mk[5]) - flux1;
      o[1] = flux1 - flux2;
      o[2] = flux2 - g_mk[0] * (x[2] - g_mk[1]);
      return all_finite(o, 3);
    }
    case OR_MODEL_DECAY:
      o[0] = -th[0] * x[0];
      return 1;
    case OR_MODEL_ADVDIFF: /* AdvDiffEval::rhs (models.cpp:164-170): spmv + finiteness */
      (void)th;
      csr_spmv(&g_adv_L, x, o);
      return all_finite(o, g_adv_L.nr);
    case OR_MODEL_LV:
      o[0] = th[0] * x[0] - x[0] * x[1];
      o[1] = x[0] * x[1] - th[1] * x[1];
      return all_finite(o, 2);
    case OR_MODEL_ROBERTSON: {
      const double ra = th[0] * x[0];
      const double rb = th[1] * x[1] * x[1];
      const double rc = th[2] * x[1] * x[2];
      o[0] = rc - ra;
      o[1] = ra - rb - rc;
      o[2] = rb;
      return all_finite(o, 3);
    }
    case OR_MODEL_CHAIN: {
      double flux[7];
      for (int i = 0; i < 7; ++i) {
        const double den = 1.0 + x[i];
        if (den <= 0.0) return 0;
        flux[i] = th[0] * x[i] / den;
      }
      o[0] = 1.0 - flux[0];
      for (int i = 1; i < 7; ++i) o[i] = flux[i - 1] - th[1] * x[i] - th[2] * x[i] * x[i];
      o[7] = th[1] * x[6] - th[3] * x[7];
      return all_finite(o, 8);
    }
  }
  return 0;
}

int or_rhs(int model, const double* theta_nat, const double* x, double* f) {
  return model_rhs(model, 0.0, theta_nat, x, f);
}

/* Dense Jacobian, row-major d x d. */
static int model_jac(int model, double t, const double* th, const double* x, double* J) {
  (void)t;
  switch (model) {
    case OR_MODEL_METABOLIC: { /* metabolic_jacobian (models.cpp:59-76) */
      const double den1 = x[0] + th[1];
      const double den2 = x[1] + th[3];
      if (den1 <= 0.0 || den2 <= 0.0) return 0;
      const double d1 = th[0] * th[1] / (den1 * den1);
      const double d2 = th[2] * th[3] / (den2 * den2);
      for (int i = 0; i < 9; ++i) J[i] = 0.0;
      J[0] = -d1;
      J[3] = d1;
      J[4] = -d2;
      J[7] = d2;
      J[8] = -g_mk[0];
      return isfinite(d1) && isfinite(d2);
    }
    case OR_MODEL_DECAY:
      J[0] = -th[0];
      return 1;
    case OR_MODEL_LV:
      J[0] = th[0] - x[1]; J[1] = -x[0];
      J[2] = x[1];         J[3] = x[0] - th[1];
      return all_finite(J, 4);
    case OR_MODEL_ROBERTSON:
      J[0] = -th[0]; J[1] = th[2] * x[2]; J[2] = th[2] * x[1];
      J[3] = th[0];  J[4] = -(2.0 * th[1] * x[1]) - th[2] * x[2]; J[5] = -(th[2] * x[1]);
      J[6] = 0.0;    J[7] = 2.0 * th[1] * x[1]; J[8] = 0.0;
      return all_finite(J, 9);
    case OR_MODEL_CHAIN: {
      double dflux[7];
      for (int i = 0; i < 64; ++i) J[i] = 0.0;
      for (int i = 0; i < 7; ++i) {
        const double den = 1.0 + x[i];
        if (den <= 0.0) return 0;
        dflux[i] = th[0] / (den * den);
      }
      J[0] = -dflux[0];
      for (int i = 1; i < 7; ++i) {
        J[i * 8 + i - 1] = dflux[i - 1];
        J[i * 8 + i] = -th[1] - 2.0 * th[2] * x[i];
      }
      J[7 * 8 + 6] = th[1];
      J[7 * 8 + 7] = -th[3];
      return all_finite(J, 64);
    }
  }
  return 0;
}

/* to_natural: exp for positive params (models.cpp:18-25). Every parameter of
 * the other models is positive; AdvDiffModel's are {k1, k2} positive, {k3,
 * c1, c2} not (models.cpp:242-249). */
static int param_positive(int model, int i) { return model != OR_MODEL_ADVDIFF || i < 2; }
static void to_natural_m(int model, int p, const double* u, double* nat) {
  for (int i = 0; i < p; ++i) nat[i] = param_positive(model, i) ? exp(u[i]) : u[i];
}

/* ------------------------------------------------------------------------ */
/* LMM tables (lmm.cpp:18-60)                                                */
/* ------------------------------------------------------------------------ */
typedef struct scheme {
  int family, order, na, nb;
  double alpha[3];
  double beta[5];
  double C;
} scheme;

static scheme ab_table(int order) {
  scheme s = {OR_AB, order, 1, order + 1, {1.0}, {0}, 0};
  switch (order) {
    case 1: s.beta[0] = 0.0; s.beta[1] = 1.0; s.C = 1.0 / 2.0; break;
    case 2: s.beta[0] = 0.0; s.beta[1] = 3.0 / 2.0; s.beta[2] = -1.0 / 2.0; s.C = 5.0 / 12.0; break;
    case 3:
      s.beta[0] = 0.0; s.beta[1] = 23.0 / 12.0; s.beta[2] = -16.0 / 12.0; s.beta[3] = 5.0 / 12.0;
      s.C = 3.0 / 8.0; break;
    default:
      s.beta[0] = 0.0; s.beta[1] = 55.0 / 24.0; s.beta[2] = -59.0 / 24.0;
      s.beta[3] = 37.0 / 24.0; s.beta[4] = -9.0 / 24.0; s.C = 251.0 / 720.0; break;
  }
  return s;
}
static scheme am_table(int order) {
  scheme s = {OR_AM, order, 1, order, {1.0}, {0}, 0};
  switch (order) {
    case 1: s.beta[0] = 1.0; s.C = -1.0 / 2.0; break;
    case 2: s.beta[0] = 1.0 / 2.0; s.beta[1] = 1.0 / 2.0; s.C = -1.0 / 12.0; break;
    default: s.beta[0] = 5.0 / 12.0; s.beta[1] = 8.0 / 12.0; s.beta[2] = -1.0 / 12.0; s.C = -1.0 / 24.0; break;
  }
  return s;
}
static scheme bdf_table(int order) {
  scheme s = {OR_BDF, order, order, 1, {0}, {0}, 0};
  switch (order) {
    case 1: s.alpha[0] = 1.0; s.beta[0] = 1.0; s.C = -1.0 / 2.0; break;
    case 2: s.alpha[0] = 4.0 / 3.0; s.alpha[1] = -1.0 / 3.0; s.beta[0] = 2.0 / 3.0; s.C = -2.0 / 9.0; break;
    default:
      s.alpha[0] = 18.0 / 11.0; s.alpha[1] = -9.0 / 11.0; s.alpha[2] = 2.0 / 11.0;
      s.beta[0] = 6.0 / 11.0; s.C = -3.0 / 22.0; break;
  }
  return s;
}
static scheme table_of(int family, int order) {
  return family == OR_AB ? ab_table(order) : family == OR_AM ? am_table(order) : bdf_table(order);
}

/* StepHistory ring of depth 4, newest first (lmm.cpp:79-106). */
typedef struct hist {
  int d, filled, head;
  double x[4][OR_MAX_D], f[4][OR_MAX_D];
} hist;
static void hist_push(hist* h, const double* x, const double* f) {
  h->head = (h->head + 1) % 4;
  memcpy(h->x[h->head], x, sizeof(double) * h->d);
  memcpy(h->f[h->head], f, sizeof(double) * h->d);
  if (h->filled < 4) ++h->filled;
}
static const double* hx(const hist* h, int age) { return h->x[(h->head + 4 - age) % 4]; }
static const double* hf(const hist* h, int age) { return h->f[(h->head + 4 - age) % 4]; }

/* explicit_step / implicit_history_terms (lmm.cpp:108-144): alpha terms in
 * ascending order, then h*beta_i f_{n+1-i} with the product h*beta_i first. */
static void combine(const hist* H, double h, const scheme* s, double* out) {
  for (int j = 0; j < H->d; ++j) out[j] = 0.0;
  for (int i = 0; i < s->na; ++i) {
    const double* xs = hx(H, i);
    const double a = s->alpha[i];
    for (int j = 0; j < H->d; ++j) out[j] += a * xs[j];
  }
  for (int i = 1; i < s->nb; ++i) {
    const double* fs = hf(H, i - 1);
    const double hb = h * s->beta[i];
    for (int j = 0; j < H->d; ++j) out[j] += hb * fs[j];
  }
}

/* extrapolate_predictor (lmm.cpp:146-165) */
static void extrapolate(const hist* H, int q, double* out) {
  for (int j = 0; j < H->d; ++j) out[j] = 0.0;
  double binom = (double)q + 1.0;
  double sign = 1.0;
  for (int i = 0; i <= q; ++i) {
    const double* xs = hx(H, i);
    const double coef = sign * binom;
    for (int j = 0; j < H->d; ++j) out[j] += coef * xs[j];
    sign = -sign;
    binom = binom * (double)(q + 1 - (i + 1)) / (double)(i + 2);
  }
}

/* DenseLu::factor / solve (linalg.cpp:201-258) */
static int lu_factor(int n, double* lu, int* piv) {
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    double best = fabs(lu[col * n + col]);
    for (int r = col + 1; r < n; ++r) {
      const double v = fabs(lu[r * n + col]);
      if (v > best) { best = v; pivot = r; }
    }
    if (best == 0.0) return 0;
    piv[col] = pivot;
    if (pivot != col) {
      for (int j = 0; j < n; ++j) {
        const double t = lu[col * n + j];
        lu[col * n + j] = lu[pivot * n + j];
        lu[pivot * n + j] = t;
      }
    }
    const double inv = 1.0 / lu[col * n + col];
    for (int r = col + 1; r < n; ++r) {
      const double f = lu[r * n + col] * inv;
      lu[r * n + col] = f;
      if (f != 0.0)
        for (int j = col + 1; j < n; ++j) lu[r * n + j] -= f * lu[col * n + j];
    }
  }
  return 1;
}
static void lu_solve(int n, const double* lu, const int* piv, double* x) {
  for (int i = 0; i < n; ++i) {
    const int p = piv[i];
    if (p != i) { const double t = x[i]; x[i] = x[p]; x[p] = t; }
    for (int j = 0; j < i; ++j) x[i] -= lu[i * n + j] * x[j];
  }
  for (int ii = n; ii-- > 0;) {
    for (int j = ii + 1; j < n; ++j) x[ii] -= lu[ii * n + j] * x[j];
    x[ii] /= lu[ii * n + ii];
  }
}

/* newton_solve (lmm.cpp:219-266), dense path. Returns status, iterations. */
static int newton_solve(int model, double t_next, const double* th, int d, double hb0,
                        const double* c, const double* guess, double tol,
                        int max_iter, double* out, int* iters) {
  double f[OR_MAX_D], r[OR_MAX_D], J[64];
  int piv[8];
  memcpy(out, guess, sizeof(double) * d);
  for (int iter = 1; iter <= max_iter; ++iter) {
    *iters = iter;
    if (!model_rhs(model, t_next, th, out, f)) return OR_ST_INVALID_RHS;
    for (int j = 0; j < d; ++j) r[j] = out[j] - hb0 * f[j] - c[j];
    if (model == OR_MODEL_ADVDIFF) {
      /* sparse path (lmm.cpp:233-243): M = csr_add(1, I, -hb0, L), factored
       * once per hb0 and workspace */
      sparse_ws* ws = g_sws;
      if (!ws->valid || ws->hb0 != hb0) {
        csr I = csr_identity(d);
        csr M = csr_add(1.0, &I, -hb0, &g_adv_L);
        memset(ws->lu, 0, sizeof(double) * (size_t)d * (size_t)d);
        for (int i = 0; i < d; ++i)
          for (int k = M.ro[i]; k < M.ro[i + 1]; ++k) ws->lu[(size_t)i * d + M.ci[k]] += M.v[k];
        csr_free(&I); csr_free(&M);
        if (!lu_factor(d, ws->lu, ws->piv)) return OR_ST_SINGULAR;
        ws->hb0 = hb0;
        ws->valid = 1;
      }
      lu_solve(d, ws->lu, ws->piv, r);
    } else {
    if (!model_jac(model, t_next, th, out, J)) return OR_ST_INVALID_RHS;
    for (int i = 0; i < d * d; ++i) J[i] = -hb0 * J[i];
    for (int i = 0; i < d; ++i) J[i * d + i] += 1.0;
    if (!lu_factor(d, J, piv)) return OR_ST_SINGULAR;
    lu_solve(d, J, piv, r);
    }
    /* newton_update_and_test (lmm.cpp:204-215) */
    double dn = 0.0, xn = 0.0;
    for (int j = 0; j < d; ++j) {
      out[j] -= r[j];
      dn = dmax(dn, fabs(r[j]));
      xn = dmax(xn, fabs(out[j]));
    }
    if (!isfinite(xn) || !isfinite(dn)) return OR_ST_INVALID_RHS;
    if (dn <= tol * (1.0 + xn)) return OR_ST_OK;
  }
  *iters = max_iter;
  return OR_ST_NEWTON_DIVERGENCE;
}

/* lte_scale_factor (lmm.cpp:307-311) */
static double lte_factor(const scheme* s, double pred_C) {
  return fabs(s->C) / fabs(pred_C - s->C);
}

/* interval_step_count (lmm.cpp:350-362) */
static int step_count(double t0, double t1, double h, long* m_out) {
  if (!(t1 > t0) || !(h > 0.0)) return fail(OR_CONFIG, "propagate_interval: need t1 > t0 and h > 0");
  const double ratio = (t1 - t0) / h;
  const long m = llround(ratio);
  if (m < 1 || fabs(ratio - (double)m) > 1e-9 * dmax(1.0, ratio))
    return fail(OR_CONFIG, "propagate_interval: (t1 - t0)/h must be an integer step count");
  *m_out = m;
  return OR_OK;
}

/* propagate_interval + ParticleRun (lmm.cpp:365-503). */
static int propagate(int model, int d, const double* th, const double* x0,
                     double t0, double t1, double h, int family, int order,
                     double tol, int max_iter, double* state, double* gamma,
                     int* status, int* iters) {
  long m;
  int rc = step_count(t0, t1, h, &m);
  if (rc) return rc;
  hist H;
  memset(&H, 0, sizeof H);
  H.d = d;
  double x[OR_MAX_D], fnew[OR_MAX_D], xnew[OR_MAX_D], aux[OR_MAX_D], guess[OR_MAX_D],
      pred[OR_MAX_D], c[OR_MAX_D];
  memcpy(x, x0, sizeof(double) * d);
  for (int j = 0; j < d; ++j) gamma[j] = 0.0;
  *status = OR_ST_OK;
  *iters = 0;
  if (!model_rhs(model, t0, th, x, fnew)) {
    *status = OR_ST_INVALID_RHS;
    memcpy(state, x, sizeof(double) * d);
    return OR_OK;
  }
  H.filled = 0; H.head = 0;
  hist_push(&H, x, fnew);
  for (long k = 1; k <= m; ++k) {
    const int p = (int)(k < order ? k : order);
    const scheme act = table_of(family, p);
    const double t_next = t0 + (double)k * h;
    const int avail = H.filled;
    double factor;
    const double* ref;
    /* prepare_step (lmm.cpp:400-434) */
    if (family == OR_AB) {
      combine(&H, h, &act, xnew);
      if (avail >= p + 1) {
        const scheme s = ab_table(p + 1);
        combine(&H, h, &s, aux);
      } else if (p >= 2) {
        const scheme s = ab_table(p - 1);
        combine(&H, h, &s, aux);
      } else {
        memcpy(aux, hx(&H, 0), sizeof(double) * d);
      }
      factor = 1.0;
      ref = aux;
    } else {
      combine(&H, h, &act, c);
      const int q = p < avail ? p : avail;
      const scheme sq = ab_table(q);
      combine(&H, h, &sq, guess);
      if (family == OR_AM) {
        memcpy(pred, guess, sizeof(double) * d);
        const scheme sp = ab_table(p);
        factor = lte_factor(&act, sp.C);
      } else if (avail >= p + 1) {
        extrapolate(&H, p, pred);
        factor = lte_factor(&act, 1.0);
      } else if (k == 1 || avail < 2) {
        memcpy(pred, guess, sizeof(double) * d);
        factor = lte_factor(&act, sq.C);
      } else {
        extrapolate(&H, avail - 1, pred);
        factor = lte_factor(&act, 1.0);
      }
      ref = pred;
      int it = 0;
      const int st = newton_solve(model, t_next, th, d, h * act.beta[0], c, guess, tol,
                                  max_iter, xnew, &it);
      *iters += it;
      if (st != OR_ST_OK) {
        *status = st;
        break;
      }
    }
    /* finish_step (lmm.cpp:438-452) */
    for (int j = 0; j < d; ++j) {
      const double est = factor * fabs(xnew[j] - ref[j]);
      gamma[j] += est * est;
    }
    if (!model_rhs(model, t_next, th, xnew, fnew)) {
      *status = OR_ST_INVALID_RHS;
      break;
    }
    hist_push(&H, xnew, fnew);
    memcpy(x, xnew, sizeof(double) * d);
  }
  memcpy(state, x, sizeof(double) * d);
  return OR_OK;
}

/* adaptive_bdf_interval (lmm.cpp:894-1019): variable-step BDF(1,2) with a
 * Newton corrector, predictor-based error control, gamma = rtol * steps. */
static double clampd(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }
static double dmin(double a, double b) { return (b < a) ? b : a; }

static int adaptive_bdf(int model, int d, const double* th, const double* x0, double t0, double t1,
                        double rtol, double tol, int max_iter, double* state, double* gamma,
                        int* status, int* iters) {
  if (!(rtol > 0.0)) return fail(OR_CONFIG, "adaptive_bdf_interval: rtol must be positive");
  if (!(t1 > t0)) return fail(OR_CONFIG, "adaptive_bdf_interval: need t1 > t0");
  const double total = t1 - t0;
  const double h_min = total * 1e-10;
  double x[OR_MAX_D], fcur[OR_MAX_D], c[OR_MAX_D], pred[OR_MAX_D], xnew[OR_MAX_D], xm1[OR_MAX_D],
      xm2[OR_MAX_D];
  double tm1 = 0.0, tm2 = 0.0;
  int npoints = 1;
  long steps_taken = 0;
  memcpy(x, x0, sizeof(double) * d);
  memset(xm1, 0, sizeof xm1);
  memset(xm2, 0, sizeof xm2);
  for (int j = 0; j < d; ++j) gamma[j] = 0.0;
  *status = OR_ST_OK;
  *iters = 0;
  if (!model_rhs(model, t0, th, x, fcur)) {
    *status = OR_ST_INVALID_RHS;
    memcpy(state, x, sizeof(double) * d);
    return OR_OK;
  }
  double t = t0;
  double h = total * 1e-2;
  while (t < t1 - total * 1e-12) {
    h = dmin(h, t1 - t);
    if (h < h_min) {
      *status = OR_ST_STIFFNESS;
      memcpy(state, x, sizeof(double) * d);
      return OR_OK;
    }
    const int p = npoints >= 2 ? 2 : 1;
    const double t_next = t + h;
    double hb0, factor;
    if (p == 1) {
      for (int j = 0; j < d; ++j) {
        c[j] = x[j];
        pred[j] = x[j] + h * fcur[j];
      }
      hb0 = h;
      factor = 0.5;
    } else {
      const double h_prev = t - tm1;
      const double omega = h / h_prev;
      const double a2 = -(omega * omega) / (1.0 + 2.0 * omega);
      hb0 = h * (1.0 + omega) / (1.0 + 2.0 * omega);
      for (int j = 0; j < d; ++j) c[j] = x[j] + a2 * (xm1[j] - x[j]);
      if (npoints >= 3) {
        const double dt1 = t - tm1;
        const double dt2 = tm1 - tm2;
        for (int j = 0; j < d; ++j) {
          const double dd1 = (x[j] - xm1[j]) / dt1;
          const double dd1p = (xm1[j] - xm2[j]) / dt2;
          const double dd2 = (dd1 - dd1p) / (t - tm2);
          pred[j] = x[j] + h * dd1 + h * (h + dt1) * dd2;
        }
      } else {
        for (int j = 0; j < d; ++j) pred[j] = x[j] + omega * (x[j] - xm1[j]);
      }
      factor = 2.0 / 11.0;
    }
    int it = 0;
    const int st = newton_solve(model, t_next, th, d, hb0, c, pred, tol, max_iter, xnew, &it);
    *iters += it;
    if (st != OR_ST_OK) {
      h *= 0.25;
      continue;
    }
    double err = 0.0, xn = 0.0;
    for (int j = 0; j < d; ++j) {
      err = dmax(err, factor * fabs(xnew[j] - pred[j]));
      xn = dmax(xn, fabs(xnew[j]));
    }
    const double est_rel = err / (1.0 + xn);
    double growth;
    if (est_rel == 0.0) {
      growth = 4.0;
    } else {
      growth = 0.9 * pow(rtol / est_rel, 1.0 / ((double)p + 1.0));
      growth = clampd(growth, 0.25, 4.0);
    }
    if (est_rel <= rtol) {
      if (!model_rhs(model, t_next, th, xnew, fcur)) {
        *status = OR_ST_INVALID_RHS;
        memcpy(state, x, sizeof(double) * d);
        return OR_OK;
      }
      memcpy(xm2, xm1, sizeof(double) * d);
      tm2 = tm1;
      memcpy(xm1, x, sizeof(double) * d);
      tm1 = t;
      memcpy(x, xnew, sizeof(double) * d);
      t = t_next;
      npoints = npoints + 1 < 3 ? npoints + 1 : 3;
      ++steps_taken;
    }
    h *= growth;
  }
  const double g = rtol * (double)steps_taken;
  for (int j = 0; j < d; ++j) gamma[j] = g;
  memcpy(state, x, sizeof(double) * d);
  return OR_OK;
}

/* Per-propagation model binding (OdeModel::bind, models.hpp:29-33) and, for
 * the sparse model, a fresh NewtonWorkspace (ParticleRun::ws, lmm.cpp:365-369;
 * adaptive_bdf_interval's ws, lmm.cpp:914-915). */
static void model_begin(int model, const double* th, int d, sparse_ws* ws) {
  ws->valid = 0;
  ws->lu = NULL;
  ws->piv = NULL;
  if (model == OR_MODEL_ADVDIFF) {
    adv_bind(th);
    ws->lu = malloc(sizeof(double) * (size_t)d * (size_t)d);
    ws->piv = malloc(sizeof(int) * (size_t)d);
  }
  g_sws = ws;
}
static void model_end(sparse_ws* ws) {
  free(ws->lu);
  free(ws->piv);
  g_sws = NULL;
}

/* the integrator the config selects (filter.cpp:242-264) */
static int propagate_cfg(const or_cfg* c, int d, const double* th, const double* x0, double t0,
                         double t1, double* state, double* gamma, int* status, int* iters) {
  sparse_ws ws;
  model_begin(c->model, th, d, &ws);
  int rc;
  if (c->adaptive)
    rc = adaptive_bdf(c->model, d, th, x0, t0, t1, c->rtol, c->newton_tol, c->newton_max_iter, state,
                      gamma, status, iters);
  else
    rc = propagate(c->model, d, th, x0, t0, t1, c->h, c->family, c->order, c->newton_tol,
                   c->newton_max_iter, state, gamma, status, iters);
  model_end(&ws);
  return rc;
}

int or_propagate_interval(int model, const double* theta_nat, const double* x0,
                          double t0, double t1, double h, int family, int order,
                          double tol, int max_iter, double* state_out,
                          double* gamma_out, int* status_out, int* iters_out) {
  int d, p;
  int rc = or_model_dims(model, &d, &p);
  if (rc) return rc;
  if (order < 1 || order > 3) return fail(OR_CONFIG, "scheme_coefficients: order must be 1, 2 or 3");
  sparse_ws ws;
  model_begin(model, theta_nat, d, &ws);
  rc = propagate(model, d, theta_nat, x0, t0, t1, h, family, order, tol,
                 max_iter, state_out, gamma_out, status_out, iters_out);
  model_end(&ws);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Filter building blocks (filter.cpp)                                       */
/* ------------------------------------------------------------------------ */
static const double kNegInf = -INFINITY;

/* logsumexp (filter.cpp:16-23) */
static double logsumexp(const double* v, uint64_t n) {
  double mx = kNegInf;
  for (uint64_t i = 0; i < n; ++i) mx = dmax(mx, v[i]);
  if (!isfinite(mx)) return kNegInf;
  double sum = 0.0;
  for (uint64_t i = 0; i < n; ++i) sum += exp(v[i] - mx);
  return mx + log(sum);
}

/* log_likelihood (filter.cpp:124-141); the lognormal kind is an extension
 * for BASELINE config 3 with no reference counterpart (parity unpinned):
 *   ll = (c0 - ss/(2 s2)) - sum log y,  r_k = log y_k - log x_k, -inf if x<=0. */
double or_log_likelihood(const or_cfg* c, const double* y, const double* x) {
  const double m = (double)c->m_y;
  const double s2 = c->sigma * c->sigma;
  const double kLog2Pi = 1.8378770664093453;
  double ss = 0.0;
  if (c->likelihood == OR_LIK_LOGNORMAL) {
    double sly = 0.0;
    for (uint64_t k = 0; k < c->m_y; ++k) {
      const double xv = x[c->obs_idx[k]];
      if (!(xv > 0.0)) return kNegInf;
      const double r = log(y[k]) - log(xv);
      ss += r * r;
      sly += log(y[k]);
    }
    return (-0.5 * m * (kLog2Pi + log(s2)) - ss / (2.0 * s2)) - sly;
  }
  for (uint64_t k = 0; k < c->m_y; ++k) {
    const double r = y[k] - x[c->obs_idx[k]];
    ss += r * r;
  }
  return -0.5 * m * (kLog2Pi + log(s2)) - ss / (2.0 * s2);
}

/* fitness_weights (filter.cpp:143-156) */
int or_fitness_weights(const double* logw, const double* loglik, uint64_t n,
                       double* g) {
  double* lg = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) lg[i] = logw[i] + loglik[i];
  const double lse = logsumexp(lg, n);
  if (!isfinite(lse)) {
    free(lg);
    return fail(OR_NUMERICAL, "total degeneracy: every particle has zero predictive likelihood");
  }
  for (uint64_t i = 0; i < n; ++i) g[i] = exp(lg[i] - lse);
  free(lg);
  return OR_OK;
}

/* resample_multinomial (filter.cpp:158-178) */
int or_resample_multinomial(const double* g, uint64_t n, uint64_t seed,
                            uint64_t j, int64_t* out) {
  if (n == 0) return OR_OK;
  double* cdf = (double*)malloc(sizeof(double) * n);
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    acc += g[i];
    cdf[i] = acc;
  }
  cdf[n - 1] = dmax(cdf[n - 1], 1.0);
  for (uint64_t i = 0; i < n; ++i) {
    stream s;
    stream_init(&s, seed, j, i, OR_PURPOSE_RESAMPLE);
    const double u = next_uniform(&s);
    /* std::upper_bound: first element > u */
    uint64_t lo = 0, len = n;
    while (len > 0) {
      const uint64_t half = len / 2;
      if (!(u < cdf[lo + half])) {
        lo = lo + half + 1;
        len = len - half - 1;
      } else {
        len = half;
      }
    }
    out[i] = (int64_t)(lo >= n ? n - 1 : lo);
  }
  free(cdf);
  return OR_OK;
}

/* weighted_mean_cov (linalg.cpp:389-432) */
int or_weighted_mean_cov(const double* params, uint64_t n, uint64_t p,
                         const double* w, double* mean, double* cov) {
  double wsum = 0.0, comp = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    if (w[i] < 0.0 || !isfinite(w[i])) return fail(OR_CONFIG, "weighted_mean_cov: weights must be nonnegative");
    const double yk = w[i] - comp;
    const double tk = wsum + yk;
    comp = (tk - wsum) - yk;
    wsum = tk;
  }
  if (fabs(wsum - 1.0) > 1e-12) return fail(OR_CONFIG, "weighted_mean_cov: weights must sum to 1");
  for (uint64_t j = 0; j < p; ++j) mean[j] = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < p; ++j) mean[j] += w[i] * params[i * p + j];
  for (uint64_t k = 0; k < p * p; ++k) cov[k] = 0.0;
  double dev[OR_MAX_P];
  for (uint64_t i = 0; i < n; ++i) {
    const double wi = w[i];
    if (wi == 0.0) continue;
    for (uint64_t j = 0; j < p; ++j) dev[j] = params[i * p + j] - mean[j];
    for (uint64_t r = 0; r < p; ++r)
      for (uint64_t c = r; c < p; ++c) cov[r * p + c] += wi * dev[r] * dev[c];
  }
  for (uint64_t r = 0; r < p; ++r)
    for (uint64_t c = 0; c < r; ++c) cov[r * p + c] = cov[c * p + r];
  return OR_OK;
}

/* try_cholesky (linalg.cpp:439-466) */
static int try_cholesky(const double* c, uint64_t p, double tol, double* l) {
  for (uint64_t k = 0; k < p * p; ++k) l[k] = 0.0;
  for (uint64_t i = 0; i < p; ++i) {
    double d = c[i * p + i];
    for (uint64_t k = 0; k < i; ++k) d -= l[i * p + k] * l[i * p + k];
    if (d < -tol) return 0;
    if (d <= tol) {
      for (uint64_t j = i + 1; j < p; ++j) {
        double s = c[j * p + i];
        for (uint64_t k = 0; k < i; ++k) s -= l[j * p + k] * l[i * p + k];
        if (fabs(s) > tol) return 0;
      }
      l[i * p + i] = 0.0;
      continue;
    }
    const double root = sqrt(d);
    l[i * p + i] = root;
    for (uint64_t j = i + 1; j < p; ++j) {
      double s = c[j * p + i];
      for (uint64_t k = 0; k < i; ++k) s -= l[j * p + k] * l[i * p + k];
      l[j * p + i] = s / root;
    }
  }
  return 1;
}

/* chol_psd (linalg.cpp:470-500) */
int or_chol_psd(const double* cov, uint64_t p, double* lower, double* jitter) {
  for (uint64_t i = 0; i < p; ++i)
    for (uint64_t j = i + 1; j < p; ++j)
      if (fabs(cov[i * p + j] - cov[j * p + i]) > 1e-12) return fail(OR_INTERNAL, "chol_psd: matrix must be symmetric");
  double trace = 0.0;
  for (uint64_t i = 0; i < p; ++i) trace += cov[i * p + i];
  const double unit = trace / (double)p;
  const double pivot_tol = 1e-14 * dmax(1.0, fabs(unit));
  static const double ladder[] = {0.0, 1e-12, 1e-10, 1e-8, 1e-6, 1e-4};
  double shifted[OR_MAX_P * OR_MAX_P];
  for (int r = 0; r < 6; ++r) {
    const double eps = ladder[r] * unit;
    memcpy(shifted, cov, sizeof(double) * p * p);
    if (eps != 0.0)
      for (uint64_t i = 0; i < p; ++i) shifted[i * p + i] += eps;
    if (try_cholesky(shifted, p, pivot_tol, lower)) {
      *jitter = eps;
      return OR_OK;
    }
  }
  return fail(OR_NUMERICAL, "chol_psd: degenerate covariance");
}

/* ------------------------------------------------------------------------ */
/* pf_step (filter.cpp:292-394)                                              */
/* ------------------------------------------------------------------------ */
/* The two per-particle propagation passes of or_pf_step as loop bodies. */
typedef struct {
  const or_cfg* c;
  const or_ens* e;
  const double* y;
  double t_prev, t_obs;
  const double* th_u;  /* shrunk (predict) or proliferated (repropagate) params */
  double* ll;          /* ll_bar (predict) or ll_new (repropagate) */
  double* xs;          /* repropagate: the reshuffled states, updated in place */
  void* unused0;
  void* unused1;
  or_step_out* out;
  int d, p;
  _Atomic int rc;
  uint64_t j;
} prop_ctx;

static void predict_body(void* vctx, uint64_t i) {
  prop_ctx* pc = (prop_ctx*)vctx;
  const or_cfg* c = pc->c;
  double nat[OR_MAX_P], xb[OR_MAX_D], gam[OR_MAX_D];
  int st, it;
  to_natural_m(c->model, pc->p, pc->th_u + i * pc->p, nat);
  const int r2 = propagate_cfg(c, pc->d, nat, pc->e->states + i * pc->d, pc->t_prev, pc->t_obs, xb, gam, &st, &it);
  if (r2) {
    atomic_store(&pc->rc, r2);
    return;
  }
  if (pc->out && pc->out->newton_iters) pc->out->newton_iters[i] = it;
  pc->ll[i] = st == OR_ST_OK ? or_log_likelihood(c, pc->y, xb) : kNegInf;
}

static void repropagate_body(void* vctx, uint64_t i) {
  prop_ctx* pc = (prop_ctx*)vctx;
  const or_cfg* c = pc->c;
  const int d = pc->d;
  or_step_out* out = pc->out;
  double nat[OR_MAX_P], xr[OR_MAX_D], gam[OR_MAX_D];
  int st, it;
  to_natural_m(c->model, pc->p, pc->th_u + i * pc->p, nat);
  const int r2 = propagate_cfg(c, d, nat, pc->xs + i * d, pc->t_prev, pc->t_obs, xr, gam, &st, &it);
  if (r2) {
    atomic_store(&pc->rc, r2);
    return;
  }
  if (out && out->newton_iters) out->newton_iters[i] += it;
  if (out && out->status_new) out->status_new[i] = st;
  if (out && out->gamma) memcpy(out->gamma + i * d, gam, sizeof(double) * d);
  pc->ll[i] = kNegInf;
  if (st != OR_ST_OK) return;
  memcpy(pc->xs + i * d, xr, sizeof(double) * d);
  stream sn;
  stream_init(&sn, c->seed, pc->j, i, OR_PURPOSE_INNOVATE);
  for (int k = 0; k < d; ++k) pc->xs[i * d + k] += sqrt(gam[k]) * next_normal(&sn);
  pc->ll[i] = or_log_likelihood(c, pc->y, pc->xs + i * d);
}

int or_pf_step(const or_cfg* c, or_ens* e, const double* y, uint64_t j,
               double t_prev, double t_obs, or_step_out* out) {
  const uint64_t n = e->n, d = e->d, p = e->p;
  int dd, pp;
  int rc = or_model_dims(c->model, &dd, &pp);
  if (rc) return rc;
  if ((uint64_t)dd != d || (uint64_t)pp != p) return fail(OR_CONFIG, "ensemble dims do not match model");
  if (c->order < 1 || c->order > 3) return fail(OR_CONFIG, "scheme_coefficients: order must be 1, 2 or 3");
  double* w = malloc(sizeof(double) * n);
  double* tb = malloc(sizeof(double) * n * p);
  double* ll_bar = malloc(sizeof(double) * n);
  double* g = malloc(sizeof(double) * n);
  int64_t* anc = malloc(sizeof(int64_t) * n);
  double* xs = malloc(sizeof(double) * n * d);
  double* tnew = malloc(sizeof(double) * n * p);
  double* ll_new = malloc(sizeof(double) * n);
  double* lw = malloc(sizeof(double) * n);
  double mean[OR_MAX_P], covtmp[OR_MAX_P * OR_MAX_P], L[OR_MAX_P * OR_MAX_P];
  rc = OR_OK;

  /* shrink (filter.cpp:107-122) */
  for (uint64_t i = 0; i < n; ++i) w[i] = exp(e->logw[i]);
  if ((rc = or_weighted_mean_cov(e->params_u, n, p, w, mean, covtmp))) goto done;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t k = 0; k < p; ++k) tb[i * p + k] = c->a * e->params_u[i * p + k] + (1.0 - c->a) * mean[k];

  /* predict + log-likelihood (filter.cpp:304-324), per particle over host
     threads (par_for; the sparse model's bound operator is process-global,
     so it stays on one thread) */
  {
    prop_ctx pc = {c, e, y, t_prev, t_obs, tb, ll_bar, NULL, NULL, NULL, out, (int)d, (int)p, OR_OK};
    par_for(n, predict_body, &pc, c->model != OR_MODEL_ADVDIFF);
    if ((rc = pc.rc)) goto done;
  }
  if (out && out->loglik_bar) memcpy(out->loglik_bar, ll_bar, sizeof(double) * n);

  /* resample (filter.cpp:326-336) */
  if ((rc = or_fitness_weights(e->logw, ll_bar, n, g))) goto done;
  if (out && out->g) memcpy(out->g, g, sizeof(double) * n);
  or_resample_multinomial(g, n, c->seed, j, anc);
  if (out && out->ancestors) memcpy(out->ancestors, anc, sizeof(int64_t) * n);
  for (uint64_t i = 0; i < n; ++i) {
    memcpy(xs + i * d, e->states + anc[i] * d, sizeof(double) * d);
    memcpy(tnew + i * p, tb + anc[i] * p, sizeof(double) * p);
  }
  for (uint64_t i = 0; i < n; ++i) lw[i] = ll_bar[anc[i]];
  memcpy(ll_bar, lw, sizeof(double) * n); /* reshuffled ll_bar */

  /* proliferate (filter.cpp:180-199) */
  {
    double jit;
    const double s = sqrt(1.0 - c->a * c->a);
    if ((rc = or_chol_psd(e->cov_u, p, L, &jit))) goto done;
    for (uint64_t i = 0; i < n; ++i) {
      stream st;
      double z[OR_MAX_P];
      stream_init(&st, c->seed, j, i, OR_PURPOSE_PROLIFERATE);
      for (uint64_t k = 0; k < p; ++k) z[k] = next_normal(&st);
      for (uint64_t r = 0; r < p; ++r) {
        double dot = 0.0;
        for (uint64_t cc = 0; cc <= r; ++cc) dot += L[r * p + cc] * z[cc];
        tnew[i * p + r] += s * dot;
      }
    }
  }

  /* repropagate + innovate + log-lik (filter.cpp:346-366), per particle */
  {
    prop_ctx pc = {c, e, y, t_prev, t_obs, tnew, ll_new, xs, NULL, NULL, out, (int)d, (int)p, OR_OK};
    pc.j = j;
    par_for(n, repropagate_body, &pc, c->model != OR_MODEL_ADVDIFF);
    if ((rc = pc.rc)) goto done;
  }

  /* update_weights (filter.cpp:210-222) + moments (filter.cpp:368-392) */
  for (uint64_t i = 0; i < n; ++i) lw[i] = ll_new[i] - ll_bar[i];
  {
    const double lse = logsumexp(lw, n);
    if (!isfinite(lse)) {
      rc = fail(OR_NUMERICAL, "total degeneracy: every repropagated particle has zero likelihood");
      goto done;
    }
    for (uint64_t i = 0; i < n; ++i) lw[i] -= lse;
  }
  memcpy(e->params_u, tnew, sizeof(double) * n * p);
  memcpy(e->logw, lw, sizeof(double) * n);
  memcpy(e->states, xs, sizeof(double) * n * d);
  for (uint64_t i = 0; i < n; ++i) w[i] = exp(lw[i]);
  if ((rc = or_weighted_mean_cov(e->params_u, n, p, w, e->mean_u, e->cov_u))) goto done;
  if (out && out->trace) {
    double* t = out->trace;
    for (uint64_t k = 0; k < p; ++k)
      t[k] = param_positive(c->model, (int)k) ? exp(e->mean_u[k]) : e->mean_u[k]; /* to_natural (filter.cpp:381-382) */
    for (uint64_t k = 0; k < p; ++k) t[p + k] = e->cov_u[k * p + k];
    for (uint64_t k = 0; k < d; ++k) t[2 * p + k] = 0.0;
    for (uint64_t i = 0; i < n; ++i)
      for (uint64_t k = 0; k < d; ++k) t[2 * p + k] += w[i] * e->states[i * d + k];
    double sum = 0.0;
    for (uint64_t i = 0; i < n; ++i) sum += exp(2.0 * lw[i]);
    t[2 * p + d] = 1.0 / sum;
  }
done:
  free(w); free(tb); free(ll_bar); free(g); free(anc); free(xs); free(tnew);
  free(ll_new); free(lw);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Initialisation                                                            */
/* ------------------------------------------------------------------------ */
static int finish_init(uint64_t n, or_ens* e) {
  double* w = malloc(sizeof(double) * n);
  for (uint64_t i = 0; i < n; ++i) e->logw[i] = -log((double)n);
  for (uint64_t i = 0; i < n; ++i) w[i] = 1.0 / (double)n;
  const int rc = or_weighted_mean_cov(e->params_u, n, e->p, w, e->mean_u, e->cov_u);
  free(w);
  return rc;
}

int or_init_uniform(int model, uint64_t n, uint64_t seed, const double* th_lo,
                    const double* th_hi, const double* x_lo, const double* x_hi,
                    or_ens* e) {
  int d, p;
  int rc = or_model_dims(model, &d, &p);
  if (rc) return rc;
  e->n = n; e->d = (uint64_t)d; e->p = (uint64_t)p;
  for (uint64_t i = 0; i < n; ++i) {
    stream s;
    stream_init(&s, seed, 0, i, OR_PURPOSE_INIT);
    for (int k = 0; k < p; ++k)
      e->params_u[i * p + k] = log(th_lo[k] + (th_hi[k] - th_lo[k]) * next_uniform(&s));
    for (int k = 0; k < d; ++k)
      e->states[i * d + k] = x_lo[k] + (x_hi[k] - x_lo[k]) * next_uniform(&s);
  }
  return finish_init(n, e);
}

/* filter::initialize (filter.cpp:76-105) */
int or_init_gaussian(int model, uint64_t n, uint64_t seed, const double* th_mu,
                     const double* th_sigma, const double* x_mean,
                     const double* x_std, const int* x_clamp, or_ens* e) {
  int d, p;
  int rc = or_model_dims(model, &d, &p);
  if (rc) return rc;
  e->n = n; e->d = (uint64_t)d; e->p = (uint64_t)p;
  for (uint64_t i = 0; i < n; ++i) {
    stream s;
    stream_init(&s, seed, 0, i, OR_PURPOSE_INIT);
    for (int k = 0; k < p; ++k) e->params_u[i * p + k] = th_mu[k] + th_sigma[k] * next_normal(&s);
    for (int k = 0; k < d; ++k) {
      double v = x_mean[k] + x_std[k] * next_normal(&s);
      if (x_clamp[k] && v < 0.0) v = 0.0;
      e->states[i * d + k] = v;
    }
  }
  return finish_init(n, e);
}
