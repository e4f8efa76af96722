/* pfsmc_gpu experiment driver — the reference's experiment-level C ABI with
 * the filter on the GPU sampler.
 *
 * Each entry point mirrors the reference call it replaces
 * (/root/reference/proj/include/pfsmc.h:27-48, src/capi.cpp:60-108):
 *
 *   pfsmc_gpu_experiment_new / _free   <- pfsmc_config_new / pfsmc_config_free
 *   pfsmc_gpu_experiment_set           <- pfsmc_config_set (same keys, same
 *                                         ConfigError messages; extra key
 *                                         "device" = CUDA ordinal)
 *   pfsmc_gpu_run_experiment           <- pfsmc_run_experiment (same data CSV +
 *                                         .json sidecar input, same trace CSV
 *                                         and report JSON outputs, run tag
 *                                         "<problem>_<integrator>_gpu")
 *   pfsmc_gpu_generate_data            <- pfsmc_generate_data (truth path on the GPU)
 *   pfsmc_gpu_string_free              <- pfsmc_string_free
 *
 * pfsmc_gpu_experiment_canonical exposes ExperimentConfig::canonical_json /
 * hash (bench.cpp:155-178) for checking. Status codes are pfsmc_gpu_status
 * (= pfsmc_status values); the message is pfsmc_gpu_experiment_last_error().
 *
 * Scope: problem "metabolic" (models::MetabolicModel on the device) with the
 * fixed-step integrators ab1-3 / am1-3 / bdf1-3 and "adaptive-bdf2" (the
 * variable-step BDF(1,2), rtol from the config). "advdiff" returns
 * PFSMC_GPU_ERR_CONFIG (the sparse model is not implemented on the GPU).
 */
#ifndef PFSMC_GPU_EXPERIMENT_H
#define PFSMC_GPU_EXPERIMENT_H

#include "pfsmc_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pfsmc_gpu_experiment pfsmc_gpu_experiment;

pfsmc_gpu_experiment* pfsmc_gpu_experiment_new(void);
void pfsmc_gpu_experiment_free(pfsmc_gpu_experiment* cfg);
const char* pfsmc_gpu_experiment_last_error(void);
pfsmc_gpu_status pfsmc_gpu_experiment_set(pfsmc_gpu_experiment* cfg, const char* key, const char* value);
pfsmc_gpu_status pfsmc_gpu_experiment_canonical(const pfsmc_gpu_experiment* cfg, char** json_out,
                                                char** hash_out);
pfsmc_gpu_status pfsmc_gpu_run_experiment(const pfsmc_gpu_experiment* cfg, const char* data_csv,
                                          const char* out_dir, char** report_path_out);
/* pfsmc_generate_data (pfsmc.h:35-37, bench.cpp:321-396): the truth trajectory
 * integrated on the GPU (pfsmc_gpu_model_trajectory, adaptive BDF(1,2), rtol
 * 1e-8), the noise from the same keyed streams, the CSV + .json sidecar. */
pfsmc_gpu_status pfsmc_gpu_generate_data(const pfsmc_gpu_experiment* cfg, const char* csv_path);
void pfsmc_gpu_string_free(char* s);

#ifdef __cplusplus
}
#endif

#endif /* PFSMC_GPU_EXPERIMENT_H */
