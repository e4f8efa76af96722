// Host-side internals shared by the translation units of libpfsmc_gpu.so:
// the sampler handle, the error / status plumbing, the cross-unit launchers.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>  // types only: NCCL is bound at run time (dlopen), see NcclApi

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace pfsmc_gpu {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " + \
                               #x);                                                      \
  } while (0)

inline constexpr const char* kKernelNames = "k_predict,k_scan_pieces,k_scan_cdf,k_serve,k_update";
inline constexpr const char* kKernelNamesFused = "k_predict,k_scan_fused,-,k_serve,k_update";
constexpr int kNumKernels = 5;


constexpr int kShardPW = 4;  // extra doubles of a migration payload beyond the record

// Every rank's search tables and records, as seen from this GPU: local
// pointers for itself, CUDA IPC mappings (NVLink peer memory) for the others.
struct PeerTable {
  const double* rec0[kMaxRanks];
  const double* rec1[kMaxRanks];
  const double* llbar[kMaxRanks];
  const double* cdf[kMaxRanks];
  const double* seg_end[kMaxRanks];
  const unsigned* coarse[kMaxRanks];
  const unsigned* ooff[kMaxRanks];  // offspring mode: exclusive prefix of per-particle offspring counts
  const TileWin* win[kMaxRanks];    // the exact scan's tile windows (read by every rank's resolver)
  unsigned* ocnt[kMaxRanks];        // offspring mode: per-particle offspring counts (peer atomics)
  unsigned long long* ocount[kMaxRanks];  // ... each rank's children per serving rank (world entries)
};

// Migration modes of a sharded step (pfsmc_gpu_shard_set_mode):
//  EXACT      every slot fetches the ancestor the global multinomial gives it
//             (bitwise the single handle; (G-1)/G of all slots cross GPUs);
//  OFFSPRING  the same uniforms and exact CDF give each particle its offspring
//             count (bitwise the single handle's counts); the children are laid
//             out in ancestor order, shard by shard, so each GPU builds its
//             children from its own ancestors and only the load imbalance
//             (children beyond a GPU's N_local) migrates. Slots are relabelled:
//             the children are a permutation of the single handle's, keyed by
//             their new global slot (distributionally equivalent after step 1).

// launchers of kernels that live in another unit (scan.cu)
void launch_scan(const Ctx& c, int ntiles, cudaStream_t st, int which);
// the global resolver over every shard's tiles, windows from `ws`
void launch_resolve_global(const Ctx& c, int ntiles, cudaStream_t st, const WinSrc& ws);
void launch_serve(const Ctx& c, int grid, cudaStream_t st);
void launch_gin(const Ctx& c, int ntiles, cudaStream_t st);
void launch_search_only(const Ctx& c, int grid, cudaStream_t st);
void launch_shard_offset(const Ctx& c, const double* gathered, cudaStream_t st);  // shard.cu

}  // namespace pfsmc_gpu

using namespace pfsmc_gpu;

// NCCL bound at run time: the process's already-loaded libnccl.so.2 (torch's)
// when there is one, so one NCCL instance serves both; nothing links it.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl_api();
void NCK(ncclResult_t r);

struct pfsmc_gpu_sampler {
  pfsmc_gpu_config cfg{};
  std::vector<uint64_t> obs;
  std::unique_ptr<KernelSet> ks;
  int d = 0, p = 0;
  long long N = 0;
  int grid = 0, ntiles = 0;
  int grid_m = 0;  // CTAs of the model kernels (predict / update / moments): N / ks->kt
  int num_sms = 148;
  Ctx ctx{};
  cudaStream_t stream = nullptr;
  // device buffers
  std::vector<void*> allocs;
  DevState* st = nullptr;
  StepParams* sp_dev = nullptr;
  StepParams* sp_host = nullptr;     // pinned
  double* trace_host = nullptr;      // pinned
  DevState* st_host = nullptr;       // pinned
  double* xmean_host = nullptr;      // pinned: the trace row's state mean (block models)
  double* flush_buf = nullptr;
  long long flush_n = 0;
  // resident observations
  std::vector<StepParams> resident;
  StepParams* resident_dev = nullptr;
  double t0_resident = 0.0;
  // graph
  cudaGraphExec_t graph = nullptr;
  bool timing = false;
  cudaEvent_t ev[kNumKernels + 1] = {};
  double kernel_ms[kNumKernels] = {};
  std::vector<cudaEvent_t> pending;  // (kNumKernels+1) per timed step
  bool have_ensemble = false;
  // An injected ensemble the reference's pf_step would reject (raised by the
  // next step, as the reference raises inside pf_step): 0 none, else the
  // pfsmc_gpu_status code, with its message.
  int pending_code = 0;
  std::string pending_msg;
  // sharding (pfsmc_gpu_create_shard)
  int rank = 0, world = 1;
  bool shard_api = false;  // created by pfsmc_gpu_create_shard
  ncclComm_t nccl = nullptr;  // pfsmc_gpu_shard_attach_nccl (native sharded step)
  PeerTable peers{};          // pfsmc_gpu_shard_attach_peers (migration over peer memory)
  bool have_peers = false;
  cudaGraphExec_t shard_graph = nullptr;  // the peer-memory step (graph with NCCL nodes)
  bool shard_graph_refused = false;
  std::vector<void*> ipc_opened;
  int ngroups_pred = 0, ngroups_upd = 0;
  double* gp_pred_all = nullptr;   // allgathered K1 group partials (world * ngroups * 2)
  double* gp_mom_all = nullptr;    // allgathered K3 group partials (world * ngroups * W)
  double* sums_all = nullptr;      // allgathered shard (sum, count) pairs
  double* sendbuf = nullptr;       // world * N_local payloads
  double* recvbuf = nullptr;       // N_local payloads
  unsigned* counts_dev = nullptr;  // [world] send + [world] recv
  unsigned* counts_all = nullptr;  // the W x W migration count matrix (k_serve_sharded)
  unsigned* counts_host = nullptr; // pinned mirror
  int shard_mode = 0;              // 0 exact, 1 offspring (PFSMC_GPU_SHARD_*)
  unsigned* ocnt = nullptr;        // offspring counts per local particle (N_local + 1)
  unsigned* ooff = nullptr;        // their exclusive prefix (N_local + 1; [N_local] = this rank's children)
  unsigned* oblk = nullptr;        // scan block sums
  unsigned long long* otot = nullptr;       // children per rank (world), from the global walk
  unsigned long long* ocount = nullptr;     // peer counting: this rank's slots per serving rank (world)
  unsigned long long* otot_host = nullptr;  // pinned mirror
  // config 5, bucketed ancestor search (c5.cu; allocated on first use)
  int scan_mode = PFSMC_GPU_SCAN_FUSED;  // exact-CDF scan of the single handle (pfsmc_gpu_set_scan_mode)
  int c5_search = 0;               // PFSMC_GPU_C5_SEARCH_GUIDE / _BUCKETED
  int c5_nb_bits = 0;              // 2^bits uniform buckets
  long long c5_cap = 0;            // slots per bucket
  long long c5_cap_override = 0;   // test knob: force a small capacity (spill path)
  unsigned* c5_count = nullptr;    // [NB] bucket fill + [NB] spill counter / overflow flag
  double* c5_u = nullptr;          // bucket-major uniforms (NB * cap), then the spill list
  unsigned* c5_n = nullptr;        // their slots
  unsigned* c5_anc = nullptr;      // their ancestors (bucket-major; scattered to ctx.anc on demand)
  bool c5_anc_pending = false;     // ctx.anc not yet written for the last bucketed iteration
  double* c5_gall = nullptr;       // sharded: every rank's stats group partials (world * groups * 7)
  bool c5_fitness_is_lw = false;   // sharded scan phases of a config-5 iteration read lw as the fitness
  unsigned long long* c5_remote = nullptr;  // sharded: records pulled from other GPUs (device counter)
  // config 5, SPLIT search: the gather makes the next iteration's moment sums (c5.cu k_c5_gather_moments)
  bool c5_fuse_moments = true;
  bool c5_moments_ready = false;   // c5_mpart holds the current ensemble's sums for the current log-weights
  double* c5_mpart = nullptr;      // [ntiles][5]

  // the Ensemble& boundary's device staging (set / get_ensemble), allocated once
  double* stage_x = nullptr;   // N x d states (AoS, the caller's layout)
  double* stage_t = nullptr;   // N x p params_u
  double* stage_w = nullptr;   // N normalised logw
  double* gate_part = nullptr; // k_weight_gate block partials
  unsigned* gate_cnt = nullptr;
  double* gate_out = nullptr;

  template <typename T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  ~pfsmc_gpu_sampler() {
    if (shard_graph) cudaGraphExecDestroy(shard_graph);
    if (nccl) nccl_api().CommDestroy(nccl);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (graph) cudaGraphExecDestroy(graph);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : pending) cudaEventDestroy(e);
    for (void* a : allocs) cudaFree(a);
    if (sp_host) cudaFreeHost(sp_host);
    if (trace_host) cudaFreeHost(trace_host);
    if (st_host) cudaFreeHost(st_host);
    if (xmean_host) cudaFreeHost(xmean_host);
    if (counts_host) cudaFreeHost(counts_host);
    if (otot_host) cudaFreeHost(otot_host);
    if (stream) cudaStreamDestroy(stream);
  }
};


// ---- status plumbing (sampler.cu) ----
extern thread_local std::string g_last_error;


template <typename F>
pfsmc_gpu_status guarded(F&& f) {
  try {
    return f();
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return PFSMC_GPU_ERR_CONFIG;
  } catch (const NumericalError& e) {
    g_last_error = e.what();
    return PFSMC_GPU_ERR_NUMERICAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PFSMC_GPU_ERR_INTERNAL;
  }
}

int step_count(double t0, double t1, double h);
StepParams make_params(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev, double t_obs, double h);
void check_error(pfsmc_gpu_sampler* s);
void ensure_staging(pfsmc_gpu_sampler* s);
void raise_pending(pfsmc_gpu_sampler* s);
void clear_error(pfsmc_gpu_sampler* s);
void ensure_exchange_buffers(pfsmc_gpu_sampler* s);
void enqueue_kernels(pfsmc_gpu_sampler* s, bool timed);
// the single handle's exact scan in the handle's scan mode (one fused pass, or records + CDF passes)
inline void launch_scan_single(pfsmc_gpu_sampler* s, const Ctx& c, cudaStream_t st) {
  if (s->scan_mode == PFSMC_GPU_SCAN_FUSED) {
    launch_scan(c, s->ntiles, st, 3);
  } else {
    launch_scan(c, s->ntiles, st, 1);
    launch_scan(c, s->ntiles, st, 2);
  }
}
void enqueue_prologue(pfsmc_gpu_sampler* s);
void build_graph(pfsmc_gpu_sampler* s);
void enqueue_readback(pfsmc_gpu_sampler* s);
void fill_trace(const pfsmc_gpu_sampler* s, const DevState& h, const double* xmean, double* out);
void harvest_timing(pfsmc_gpu_sampler* s);
void enqueue_step(pfsmc_gpu_sampler* s, const StepParams* host_sp, const StepParams* dev_sp);
namespace pfsmc_gpu {
void c5_flush_ancestors(pfsmc_gpu_sampler* s);  // c5.cu
int c5_shard_groups(const pfsmc_gpu_sampler* s);
WinSrc peer_winsrc(const pfsmc_gpu_sampler* s);  // shard.cu
double* c5_group_all(pfsmc_gpu_sampler* s);
}
