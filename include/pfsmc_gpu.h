/* pfsmc_gpu — B200-native drop-in for the reference per-observation update
 * `pfsmc::filter::pf_step` of the LMM PF-SMC sampler (arXiv 1411.1702).
 *
 * Plain C ABI: opaque handles, plain pointers and sizes, integer status
 * codes plus a thread-local last-error string — the same conventions as the
 * reference's C ABI (/root/reference/proj/include/pfsmc.h:12-25,
 * src/capi.cpp:13-37). The reference's own C ABI is experiment-level only
 * (config / generate / run / bench / report, pfsmc.h:27-59) and has no
 * per-step entry point; the calls below are what a caller of
 *   StepResult pf_step(Ensemble&, std::span<const double> y, size_t j,
 *                      double t_prev, double t_obs, const PfConfig&,
 *                      exec::Backend&, const models::OdeModel&,
 *                      const ObservationModel&, PhaseTimings*)
 * (filter.hpp:151-155, filter.cpp:292-394) binds instead. Each entry point
 * names the reference interface it replaces.
 *
 * Handles are not re-entrant; several handles may coexist (one per GPU).
 * Ensembles cross this boundary as the reference stores them: row-major AoS
 * (states N x d, params_u N x p, unconstrained = log space), normalised
 * logw, mean_u (p), cov_u (p x p) — filter.hpp:19-28.
 */
#ifndef PFSMC_GPU_H
#define PFSMC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same values as pfsmc_status (pfsmc.h:12-18). NUMERICAL is raised at the
 * same step j as the reference raises NumericalError (total degeneracy in
 * fitness_weights / update_weights, chol_psd failure); CONFIG where it
 * raises ConfigError (PfConfig::validate, interval_step_count). */
typedef enum pfsmc_gpu_status {
  PFSMC_GPU_OK = 0,
  PFSMC_GPU_ERR_INTERNAL = 1,
  PFSMC_GPU_ERR_CONFIG = 2,
  PFSMC_GPU_ERR_NUMERICAL = 3,
  PFSMC_GPU_ERR_IO = 4
} pfsmc_gpu_status;

/* Compiled-in OdeModel plugins (device functors; models.hpp:20-55 contract). */
enum {
  PFSMC_GPU_MODEL_DECAY = 0,      /* x' = -theta x (reference test model) */
  PFSMC_GPU_MODEL_LOTKA_VOLTERRA = 1,
  PFSMC_GPU_MODEL_ROBERTSON = 2,
  PFSMC_GPU_MODEL_CHAIN8 = 3,
  PFSMC_GPU_MODEL_PAYLOAD64 = 4,  /* 64-byte record, resample microbenchmark only */
  PFSMC_GPU_MODEL_METABOLIC = 5,  /* the reference's problem 1, models::MetabolicModel
                                     (models.cpp:37-119): d = 3, p = 4, time-dependent input */
  PFSMC_GPU_MODEL_ADVDIFF = 6     /* the reference's problem 2, models::AdvDiffModel(n)
                                     (models.cpp:158-266): periodic advection-diffusion on an
                                     (n-1) x (n-1) grid, d = (n-1)^2, p = 5 (k1, k2 positive;
                                     k3, c1, c2 not), n = model_consts[0], 4 <= n <= 33 */
};
/* Caller-defined models: ids >= PFSMC_GPU_MODEL_USER_BASE are served by
 * plugin libraries built against include/pfsmc_gpu_model.cuh (the device
 * form of the OdeModel::bind -> ModelEval::{rhs, jacobian} contract,
 * models.hpp:20-55); loading such a library registers its models. */
#define PFSMC_GPU_MODEL_USER_BASE 64
/* Called by a plugin's static initialiser (PFSMC_GPU_REGISTER_MODEL): make_kernels
 * is the plugin's `std::unique_ptr<KernelSet> (*)(int family, int order)`;
 * fast = 1 registers the FMA variant (the unit compiled with -DPFSMC_FAST=1). */
pfsmc_gpu_status pfsmc_gpu_register_model(int id, const char* name, int d, int p, int fast,
                                          void* make_kernels);
/* The i-th registered plugin model (i = 0, 1, ...); CONFIG past the end. */
pfsmc_gpu_status pfsmc_gpu_registered_model(int index, int* id, const char** name, int* d, int* p);

/* lmm::Family (lmm.hpp:12) */
enum { PFSMC_GPU_AB = 0, PFSMC_GPU_AM = 1, PFSMC_GPU_BDF = 2 };
/* Observation noise. GAUSSIAN is filter::log_likelihood (filter.cpp:124-141);
 * LOGNORMAL is an extension for BASELINE config 3 (no reference counterpart). */
enum { PFSMC_GPU_LIK_GAUSSIAN = 0, PFSMC_GPU_LIK_LOGNORMAL = 1 };
/* Device arithmetic. EXACT: the reference's operation order without FMA
 * contraction and IEEE divisions where the reference divides (the reference
 * build has no FMA, CMakeLists.txt:7-9), so Psi is bitwise the CPU's.
 * FAST: FMA contraction and one reciprocal per shared denominator; results
 * within the north_star tolerances (states 1e-10 relative, trace 1e-8,
 * ancestors exact except classified near-ties), not bitwise. Same RNG
 * streams, same exact resampling CDF. */
enum { PFSMC_GPU_ARITH_EXACT = 0, PFSMC_GPU_ARITH_FAST = 1 };

typedef struct pfsmc_gpu_sampler pfsmc_gpu_sampler;

/* The fields of filter::PfConfig + ObservationModel that pf_step reads
 * (filter.hpp:30-65), plus the device placement. */
typedef struct pfsmc_gpu_config {
  int model;               /* PFSMC_GPU_MODEL_* */
  int family;              /* PFSMC_GPU_AB / AM / BDF  (IntegratorSpec.family) */
  int order;               /* 1..3                      (IntegratorSpec.order)  */
  double shrink_a;         /* PfConfig.shrink_a, in (0, 1) */
  uint64_t seed;           /* PfConfig.seed */
  double newton_tol;       /* NewtonOpts.tol (reference default 1e-9) */
  int newton_max_iter;     /* NewtonOpts.max_iter (reference default 20) */
  uint64_t particles;      /* PfConfig.particles (global N) */
  const uint64_t* obs_indices; /* ObservationModel.indices */
  uint64_t n_obs;          /* m_y <= 8 (ADVDIFF: <= 32) */
  double sigma;            /* ObservationModel.sigma */
  int likelihood;          /* PFSMC_GPU_LIK_* */
  int device;              /* CUDA ordinal */
  double model_consts[8];  /* the bound model's constants; METABOLIC: (lambda, c0, A0, A,
                              t0_input, tau) = MetabolicConstants (models.hpp:67-74),
                              reference defaults (1, 1, 1, 5, 2, 1); ADVDIFF: (n); others:
                              unused */
  int adaptive;            /* IntegratorSpec.adaptive: variable-step BDF(1,2)
                              (lmm::adaptive_bdf_interval, lmm.cpp:894-1019); family,
                              order and the step h are then unused */
  double rtol;             /* IntegratorSpec.rtol (adaptive only; reference default 1e-3) */
  int arithmetic;          /* PFSMC_GPU_ARITH_EXACT (default, 0) or PFSMC_GPU_ARITH_FAST */
} pfsmc_gpu_config;

const char* pfsmc_gpu_version(void);
/* Thread-local message of the most recent failure (pfsmc_last_error). */
const char* pfsmc_gpu_last_error(void);

/* Validates like PfConfig::validate (filter.cpp:45-74) and allocates the
 * device-resident ensemble (SoA-of-records, double buffered). */
pfsmc_gpu_status pfsmc_gpu_create(const pfsmc_gpu_config* cfg, pfsmc_gpu_sampler** out);
void pfsmc_gpu_destroy(pfsmc_gpu_sampler* s);

/* Inject / read back a filter::Ensemble (host AoS arrays, sizes from cfg).
 * set: the shrink mean is recomputed from (params_u, exp(logw)) on the
 * device exactly as filter::shrink does each step (filter.cpp:107-122);
 * cov_u is used as given for the next proliferation (filter.cpp:343). */
pfsmc_gpu_status pfsmc_gpu_set_ensemble(pfsmc_gpu_sampler* s, const double* states,
                                        const double* params_u, const double* logw,
                                        const double* mean_u, const double* cov_u);
pfsmc_gpu_status pfsmc_gpu_get_ensemble(pfsmc_gpu_sampler* s, double* states,
                                        double* params_u, double* logw, double* mean_u,
                                        double* cov_u);

/* Device-side initialisation (replaces filter::initialize, filter.cpp:76-105).
 * gaussian: the reference prior (theta_u ~ N(mu, sigma), x ~ N(mean, std),
 * optional clamp at 0), stream (seed, 0, i, init), theta then x.
 * uniform: the BASELINE box prior U[lo, hi] in natural space, same stream
 * and order, theta_u = log U. Moments with equal weights. */
pfsmc_gpu_status pfsmc_gpu_init_gaussian(pfsmc_gpu_sampler* s, const double* th_mu,
                                         const double* th_sigma, const double* x_mean,
                                         const double* x_std, const int* x_clamp);
pfsmc_gpu_status pfsmc_gpu_init_uniform(pfsmc_gpu_sampler* s, const double* th_lo,
                                        const double* th_hi, const double* x_lo,
                                        const double* x_hi);

/* THE DROP-IN: one assimilation step, replacing filter::pf_step
 * (filter.cpp:292-394). y: n_obs host doubles; j: 1-based time index;
 * [t_prev, t_obs] with fixed LMM step h (PfConfig.h). trace_out (host,
 * optional) receives the TraceRow: theta_mean[p] (natural space),
 * theta_var[p], state_mean[d], ess — 2p + d + 1 doubles. Blocking. */
pfsmc_gpu_status pfsmc_gpu_step(pfsmc_gpu_sampler* s, const double* y, uint64_t j,
                                double t_prev, double t_obs, double h, double* trace_out);

/* Non-blocking variant for resident observation streams: enqueues the step
 * on the sampler's stream, observations taken from pfsmc_gpu_upload_observations
 * row (j - 1). Errors surface at the next pfsmc_gpu_synchronize. */
pfsmc_gpu_status pfsmc_gpu_upload_observations(pfsmc_gpu_sampler* s, const double* ys,
                                               const double* t_obs, uint64_t T, double t0,
                                               double h);
pfsmc_gpu_status pfsmc_gpu_step_resident(pfsmc_gpu_sampler* s, uint64_t j);
pfsmc_gpu_status pfsmc_gpu_synchronize(pfsmc_gpu_sampler* s, double* trace_out);
/* Host<->device bytes of one blocking pfsmc_gpu_step (step parameters up,
 * device state incl. the trace row down): the e2e accounting. */
pfsmc_gpu_status pfsmc_gpu_step_transfer_bytes(pfsmc_gpu_sampler* s, uint64_t* h2d, uint64_t* d2h);

/* filter::run (filter.cpp:396-443) on resident observations: rows (T+1) x
 * (2p + d + 1) of the PosteriorTrace, row 0 from the current ensemble;
 * degeneracy streak flags in warn_out (T+1 ints, optional). */
pfsmc_gpu_status pfsmc_gpu_run(pfsmc_gpu_sampler* s, double* trace_rows, int* warn_out);

/* Diagnostics of the last step (lock-step parity, FLOP counting):
 * ancestors (uint32, N), predictor log-likelihoods before reshuffle (N),
 * total Newton iterations of the step. Any pointer may be NULL. */
pfsmc_gpu_status pfsmc_gpu_get_step_diagnostics(pfsmc_gpu_sampler* s, uint32_t* ancestors,
                                                double* loglik_bar, uint64_t* newton_iters);

/* Kernel-level parity for resample_multinomial (filter.cpp:158-178): the
 * device CDF + ancestor search fed an injected fitness vector g (host, N
 * doubles, N = cfg.particles); ancestors_out (host, N). Also returns the
 * device CDF (optional). */
pfsmc_gpu_status pfsmc_gpu_resample_from_g(pfsmc_gpu_sampler* s, const double* g,
                                           uint64_t j, uint32_t* ancestors_out,
                                           double* cdf_out);

/* %globaltimer probes of the last step (ns): [0] exact-CDF kernel start,
 * [1] resolver start, [2] resolver end. Diagnostics for profiling. */
pfsmc_gpu_status pfsmc_gpu_debug_timestamps(pfsmc_gpu_sampler* s, uint64_t* out8);

/* The CUDA stream every launch of this handle goes to (cudaStream_t). */
void* pfsmc_gpu_stream(pfsmc_gpu_sampler* s);

/* Per-kernel device time accounting (CUDA events around each launch of the
 * step's kernels, on the sampler's stream). While enabled, steps launch
 * kernels directly instead of replaying the CUDA graph. names_out receives a
 * static, comma-separated kernel list of n_kernels entries ("-" marks an
 * event slot without a kernel: the fused scan mode has one scan launch). */
pfsmc_gpu_status pfsmc_gpu_set_kernel_timing(pfsmc_gpu_sampler* s, int enable);
pfsmc_gpu_status pfsmc_gpu_kernel_times(pfsmc_gpu_sampler* s, double* ms_out, int* n_kernels,
                                        const char** names_out);

/* BASELINE config 5 (resample / reduction bandwidth), PAYLOAD64 handles:
 * draw i.i.d. N(0, sigma^2) log-weights (keyed stream (seed, key, n, init)),
 * then enqueue iterations of: log-sum-exp, weighted 2x2 covariance of
 * theta, exact multinomial resampling, gather of the 64-byte records. */
pfsmc_gpu_status pfsmc_gpu_c5_set_logweights(pfsmc_gpu_sampler* s, double sigma, uint64_t key);
pfsmc_gpu_status pfsmc_gpu_c5_iteration(pfsmc_gpu_sampler* s, uint64_t j);
/* Ancestor search of the config-5 iteration (filter.cpp:169-176: every slot's
 * ancestor is upper_bound(cdf, u_n), bit-exact either way):
 *   GUIDE    slot-order search (guide table -> segment ends -> one CDF segment)
 *            and gather, one pass;
 *   BUCKETED the uniforms are first bucketed by value (a one-pass counting
 *            partition into 2^k ranges of [0, 1)), then searched and gathered
 *            in bucket order, so the CDF, the search tables and the ancestor
 *            records are read once, in narrow L2-resident windows; the
 *            records are written to their slots (64-byte stores);
 *   SPLIT    the GUIDE search writing only the ancestors, then a separate
 *            slot-order gather; that gather also accumulates the weighted
 *            moment sums of the ensemble it writes (the stats pass's tiles,
 *            thread layout and trees: the same bits), so the next iteration's
 *            stats pass reads the log-weights only, as long as the host does
 *            not change the log-weights, the ensemble or the mode in between. */
enum { PFSMC_GPU_C5_SEARCH_GUIDE = 0, PFSMC_GPU_C5_SEARCH_BUCKETED = 1, PFSMC_GPU_C5_SEARCH_SPLIT = 2 };
pfsmc_gpu_status pfsmc_gpu_c5_set_search(pfsmc_gpu_sampler* s, int mode);

/* The exact sequential-CDF scan of a single (unsharded) handle:
 *   FUSED    one kernel: tile classification, decoupled look-back for the exact
 *            sum before each tile, CDF values and search tables (the default);
 *   TWO_PASS the records pass with its one-block window resolver, then the CDF
 *            pass (the form the sharded step uses, where the tile records cross
 *            GPUs). Bitwise identical results. Takes effect at the next step
 *            (the blocking step's CUDA graph is rebuilt). */
enum { PFSMC_GPU_SCAN_FUSED = 0, PFSMC_GPU_SCAN_TWO_PASS = 1 };
pfsmc_gpu_status pfsmc_gpu_set_scan_mode(pfsmc_gpu_sampler* s, int mode);

/* Measured FP64 FMA throughput of `device` in TFLOP/s (DFMA loop; the FP64
 * roofline denominator the benchmarks report against). */
pfsmc_gpu_status pfsmc_gpu_fp64_peak(int device, double* tflops);
/* One noise-free trajectory of a compiled-in model through times[0..T) from
 * (t0, x0) with the adaptive BDF(1,2) integrator at rtol (the data
 * generator's truth path: bench.cpp:296-317 over lmm::adaptive_bdf_interval,
 * NewtonOpts defaults); states_out is T x d. NUMERICAL if the integration
 * fails, like the reference generator. */
pfsmc_gpu_status pfsmc_gpu_model_trajectory(int model, const double* model_consts, const double* theta_nat,
                                            const double* x0, const double* times, uint64_t T, double t0,
                                            double rtol, int device, double* states_out);

/* Measured random-gather roofline for the resampling gathers: GB/s of
   64-byte records read at hashed indices plus written in slot order, over
   n_rec records (use n_rec * 64 bytes > L2). Benchmark helper. */
pfsmc_gpu_status pfsmc_gpu_gather_peak(int device, long long n_rec, double* gbs);

/* L2 flush helper for benchmarks: writes a device buffer larger than L2 on
 * the sampler's stream. */
pfsmc_gpu_status pfsmc_gpu_flush_l2(pfsmc_gpu_sampler* s);

/* ------------------------------------------------------------------------
 * Multi-GPU sharding. One handle per GPU owns the global
 * slots [rank*N/world, (rank+1)*N/world) of the N = cfg.particles global
 * particles (N a multiple of world * 16384); every keyed stream uses the
 * global slot, so the sharded filter draws exactly the single-handle numbers
 * and reproduces its results bit for bit. The host orchestrator
 * (paper_1411_1702_b200/sharded.py) runs, per step:
 *   shard_predict -> allgather buf 0 into 1 -> shard_finish_lse
 *   allgather buf 2 into 3 -> shard_scan_records
 *   allgather the own slices of bufs 4, 5 -> shard_resolve
 *   shard_serve (counts) -> exchange payloads buf 8 -> buf 9 -> shard_update
 *   allgather buf 6 into 7 -> shard_finish_moments(7)
 * i.e. the only cross-GPU traffic is the global log-sum-exp, the tile records
 * of the exact CDF, the ancestor payloads and the moment partials. */
pfsmc_gpu_status pfsmc_gpu_create_shard(const pfsmc_gpu_config* cfg, int rank, int world,
                                        pfsmc_gpu_sampler** out);
/* Device pointer + size of exchange buffer `which` (see the sequence above;
 * 4/5 are global arrays whose own slice starts at rank * bytes / world;
 * 12/13: the config-5 stats group partials, own / all ranks). */
pfsmc_gpu_status pfsmc_gpu_shard_buffer(pfsmc_gpu_sampler* s, int which, void** ptr,
                                        uint64_t* bytes);
pfsmc_gpu_status pfsmc_gpu_shard_predict(pfsmc_gpu_sampler* s, const double* y, uint64_t j,
                                         double t_prev, double t_obs, double h);
pfsmc_gpu_status pfsmc_gpu_shard_finish_lse(pfsmc_gpu_sampler* s);
pfsmc_gpu_status pfsmc_gpu_shard_scan_records(pfsmc_gpu_sampler* s);
pfsmc_gpu_status pfsmc_gpu_shard_resolve(pfsmc_gpu_sampler* s);
/* counts_out: world send counts then world receive counts (payloads of
 * (record, ll_bar, ancestor, slot) doubles); blocking. Every rank derives the
 * whole migration count matrix locally (same keyed uniforms, same exact shard
 * ranges), so no count exchange is needed: */
pfsmc_gpu_status pfsmc_gpu_shard_serve(pfsmc_gpu_sampler* s, uint32_t* counts_out);
/* ... the world x world matrix of the last serve (row r = rank r's sends). */
pfsmc_gpu_status pfsmc_gpu_shard_count_matrix(pfsmc_gpu_sampler* s, uint32_t* out);

/* Native sharded step: the whole filter::pf_step of the global filter in one
 * call, the five exchanges as NCCL collectives on the handle's stream (NCCL is
 * bound at run time to the process's libnccl.so.2). Rank 0 makes the 128-byte
 * id, every rank attaches with it (one communicator per handle). */
pfsmc_gpu_status pfsmc_gpu_nccl_unique_id(uint8_t* out128);
pfsmc_gpu_status pfsmc_gpu_shard_attach_nccl(pfsmc_gpu_sampler* s, const uint8_t* id128);
pfsmc_gpu_status pfsmc_gpu_shard_step(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev,
                                      double t_obs, double h, double* trace_out);
/* Migration over NVLink peer memory (replaces the counted send/recv and its
 * host sync inside pfsmc_gpu_shard_step): each rank exports PFSMC_GPU_IPC_BYTES
 * of CUDA IPC handles (7 x 64 bytes: its record buffers, ll_bar, exact CDF,
 * segment ends, guide, offspring prefix), the caller allgathers them (world x
 * PFSMC_GPU_IPC_BYTES, rank order) and every rank attaches; then each slot
 * pulls its ancestor from the serving rank's memory. */
#define PFSMC_GPU_IPC_BYTES 640
pfsmc_gpu_status pfsmc_gpu_shard_ipc_handles(pfsmc_gpu_sampler* s, uint8_t* out448);
pfsmc_gpu_status pfsmc_gpu_shard_attach_peers(pfsmc_gpu_sampler* s, const uint8_t* all_handles);
/* Back to the counted send / receive (if any rank failed to map its peers). */
pfsmc_gpu_status pfsmc_gpu_shard_detach_peers(pfsmc_gpu_sampler* s);
/* Same-process shards (R handles of one filter in one process, e.g. on one
 * GPU): the peer table from the handles themselves (rank order), no IPC. */
pfsmc_gpu_status pfsmc_gpu_shard_attach_peers_local(pfsmc_gpu_sampler* s, pfsmc_gpu_sampler* const* shards);
/* Phase D over peer memory + the update kernel, phase by phase (replaces
 * shard_serve + the payload exchange + shard_update): call after every
 * rank's tables are complete (after the resolve phase). */
pfsmc_gpu_status pfsmc_gpu_shard_pull(pfsmc_gpu_sampler* s);
/* shard_resolve reading every shard's tile windows over peer memory (peers
 * attached): with it, phase C exchanges only the tile headers (buffer 4), not
 * the window lists (buffer 5). */
pfsmc_gpu_status pfsmc_gpu_shard_resolve_peers(pfsmc_gpu_sampler* s);
pfsmc_gpu_status pfsmc_gpu_shard_update(pfsmc_gpu_sampler* s, uint64_t n_recv);

/* Migration mode of the sharded step (north_star).
 * EXACT (default): every slot's ancestor from the global multinomial, bitwise
 * the single handle (ancestors, states, trace); (G-1)/G of the slots fetch a
 * remote ancestor whatever the weights.
 * OFFSPRING: the same keyed uniforms and exact CDF give each particle its
 * offspring count o_i (bitwise the single handle's counts, i.e.
 * bincount(ancestors)); the children are laid out in ancestor order, rank by
 * rank, so each GPU builds its children from its own ancestors and only the
 * load imbalance (children beyond its N_local slots) migrates; children are
 * keyed by their new global slot (a relabelling: distributionally equivalent
 * to the single handle, not bitwise, after the first step). */
enum { PFSMC_GPU_SHARD_EXACT = 0, PFSMC_GPU_SHARD_OFFSPRING = 1 };
pfsmc_gpu_status pfsmc_gpu_shard_set_mode(pfsmc_gpu_sampler* s, int mode);
/* Offspring mode, phase by phase (after shard_resolve): the walk of every
 * global slot's uniform (no exchange) -> this rank's per-particle counts and
 * the children of every rank (totals_out: world counts, identical on all
 * ranks); blocking. */
pfsmc_gpu_status pfsmc_gpu_shard_offspring(pfsmc_gpu_sampler* s, uint64_t* totals_out);
/* ... the per-particle offspring counts of this rank's particles (N_local). */
pfsmc_gpu_status pfsmc_gpu_shard_offspring_counts(pfsmc_gpu_sampler* s, uint32_t* counts_out);
/* ... counted path: packs this rank's children per destination into buffer 8
 * (the shard_serve layout: destination d's items at d * N_local) and returns
 * the world x world item matrix (row q = rank q's sends); exchange as for
 * shard_serve, then shard_update(N_local). */
pfsmc_gpu_status pfsmc_gpu_shard_offspring_pack(pfsmc_gpu_sampler* s, uint32_t* matrix_out);
/* ... peer-memory path: every slot pulls its child's ancestor from the rank
 * whose children cover it, then the update kernel (replaces pack + exchange
 * + shard_update). */
pfsmc_gpu_status pfsmc_gpu_shard_offspring_pull(pfsmc_gpu_sampler* s);
/* Offspring counts over peer memory (peers attached) instead of the walk of
 * every global slot: O(N_local) work per rank. Phases with a barrier across
 * ranks between them: 0 zero the counts, 1 count this rank's slots into the
 * ancestors' owners (every rank's CDF tables complete), 2 totals + this
 * rank's prefix (returns every rank's children, blocking). Then
 * shard_offspring_pull after a barrier. The native step uses this sequence. */
pfsmc_gpu_status pfsmc_gpu_shard_offspring_peer(pfsmc_gpu_sampler* s, int phase, uint64_t* totals_out);
pfsmc_gpu_status pfsmc_gpu_shard_moments(pfsmc_gpu_sampler* s);
/* flags: 7 completed step, 2 initialisation refresh, 0 injected ensemble. */
pfsmc_gpu_status pfsmc_gpu_shard_finish_moments(pfsmc_gpu_sampler* s, int flags, double* trace_out);

/* BASELINE config 5 over several GPUs (PAYLOAD64 shard handles, particles per
 * shard a multiple of 64 exact-CDF tiles): one resample / reduction iteration
 * of the global ensemble, exact migration (every slot's ancestor is the
 * single handle's, bitwise; its 64-byte record is pulled over NVLink peer
 * memory when another GPU holds it). Phase by phase:
 *   shard_c5_stats -> allgather buf 12 into 13 -> shard_c5_finish
 *     (global log-sum-exp, weighted mean / covariance: the single handle's
 *      group partials combined in the same order)
 *   allgather buf 2 into 3 -> shard_scan_records
 *   allgather the own slices of bufs 4, 5 -> shard_resolve
 *   allgather buf 2 into 3 (every rank's CDF tables complete) -> shard_c5_pull(j)
 *   (every rank's pull done) -> shard_c5_flip
 * or natively (NCCL attached, peers attached): shard_c5_iteration(j). */
pfsmc_gpu_status pfsmc_gpu_shard_c5_stats(pfsmc_gpu_sampler* s);
pfsmc_gpu_status pfsmc_gpu_shard_c5_finish(pfsmc_gpu_sampler* s);
pfsmc_gpu_status pfsmc_gpu_shard_c5_pull(pfsmc_gpu_sampler* s, uint64_t j);
pfsmc_gpu_status pfsmc_gpu_shard_c5_flip(pfsmc_gpu_sampler* s);
pfsmc_gpu_status pfsmc_gpu_shard_c5_iteration(pfsmc_gpu_sampler* s, uint64_t j);
/* Records this rank pulled from other GPUs so far (64 bytes each over NVLink). */
pfsmc_gpu_status pfsmc_gpu_shard_c5_remote_pulls(pfsmc_gpu_sampler* s, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
