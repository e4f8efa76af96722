"""Multi-GPU PF-SMC: particle sharding with the per-step collectives
(SURVEY.md §8(e)).

Each shard owns a contiguous range of GLOBAL slots and keys every Philox
stream by the global slot (filter.cpp:88, 171, 190, 204), so a sharded step
draws exactly the numbers of the single-handle step. Per step
(`ShardedFilter.pf_step`) the only exchanges are:

  A  allgather of the predict-kernel group partials  -> global log-sum-exp
     (combined in the single-handle order: bitwise the same lse)
  B  allgather of shard (approximate g total, nonzero count) -> global
     approximate prefix for the exact-CDF classification
  C  allgather of the tile records (headers + windows) -> every rank resolves
     the exact sequential CDF chain over all shards (exact_cdf.cuh)
  D  personalised exchange of ancestor payloads: rank r serves the global
     slots whose uniform falls in its exact-CDF range and ships
     {record, ll_bar, ancestor, slot} to the slot's owner (the migration)
  E  allgather of the update-kernel moment partials -> global lse_w, mean,
     covariance, trace row, chol (same combine as the single handle)

The orchestration is backend-agnostic: a shard exposes phases and exchange
buffers (torch tensors); a communicator moves the bytes. `GpuShard` drives
the sm_100a kernels through the C ABI (include/pfsmc_gpu.h); `TorchComm`
uses torch.distributed (NCCL across GPUs, or gloo), `LocalComm` moves bytes
between shards living in one process (used to check on ONE GPU that R
shards reproduce the single-handle run bit for bit; the phases run strictly
one after another, no kernel ever waits on another shard's kernel).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from .sampler import MODEL_DIMS, MODELS, ConfigError, GpuSampler, ObservationModel, PfConfig, TraceRow, _f64, _ptr

(BUF_PRED, BUF_PRED_ALL, BUF_SUM, BUF_SUM_ALL, BUF_HDR, BUF_WIN, BUF_MOM, BUF_MOM_ALL, BUF_SEND, BUF_RECV,
 BUF_CNT, BUF_CNT_ALL, BUF_C5, BUF_C5_ALL) = range(14)
STEP_FLAGS, INIT_FLAGS, INJECT_FLAGS = 7, 2, 0
IPC_BYTES = 640  # PFSMC_GPU_IPC_BYTES
SHARD_MODES = {"exact": 0, "offspring": 1}  # PFSMC_GPU_SHARD_EXACT / _OFFSPRING


def offspring_matrix(totals, world: int, n_local: int) -> np.ndarray:
    """Offspring mode: rank q's children occupy global positions
    [P_q, P_q + O_q) (P the exclusive prefix of the totals); position p lives
    on rank p // n_local. S[q, d] = children of q placed on d (only the
    off-diagonal imbalance crosses GPUs)."""
    S = np.zeros((world, world), dtype=np.int64)
    P = 0
    for q in range(world):
        a, b = P, P + int(totals[q])
        for d in range(world):
            lo, hi = max(a, d * n_local), min(b, (d + 1) * n_local)
            if hi > lo:
                S[q, d] = hi - lo
        P = b
    return S


class _CudaArray:
    """Zero-copy view of a raw device allocation for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


class GpuShard(GpuSampler):
    """One shard of the global filter on one GPU (pfsmc_gpu_create_shard)."""

    def __init__(self, model: str, cfg: PfConfig, obs: ObservationModel, rank: int, world: int,
                 device: int = 0, model_consts=None):
        from .sampler import ARITHMETIC, FAMILIES, LIKELIHOODS, _Config, load_library, model_consts_array
        self.lib = load_library()
        self.model, self.cfg, self.obs = model, cfg, obs
        self.d, self.p = MODEL_DIMS[MODELS[model]]
        self.rank, self.world, self.device = rank, world, device
        self._idx = np.ascontiguousarray(list(obs.indices), dtype=np.uint64)
        c = _Config(MODELS[model], FAMILIES[cfg.family], cfg.order, cfg.shrink_a, cfg.seed, cfg.newton_tol,
                    cfg.newton_max_iter, cfg.particles, _ptr(self._idx, C.POINTER(C.c_uint64)), len(self._idx),
                    obs.sigma, LIKELIHOODS[obs.likelihood], device, model_consts_array(model, model_consts),
                    int(cfg.adaptive), cfg.rtol, ARITHMETIC[cfg.arithmetic])
        L = self.lib
        for name in ("pfsmc_gpu_create_shard", "pfsmc_gpu_shard_buffer", "pfsmc_gpu_shard_predict",
                     "pfsmc_gpu_shard_finish_lse", "pfsmc_gpu_shard_scan_records",
                     "pfsmc_gpu_shard_resolve", "pfsmc_gpu_shard_serve", "pfsmc_gpu_shard_update",
                     "pfsmc_gpu_shard_moments", "pfsmc_gpu_shard_finish_moments"):
            getattr(L, name).restype = C.c_int
        L.pfsmc_gpu_shard_count_matrix.restype = C.c_int
        h = C.c_void_p()
        self._check(L.pfsmc_gpu_create_shard(C.byref(c), rank, world, C.byref(h)))
        self.h = h
        self.n = cfg.particles // world
        self.n0 = rank * self.n
        self.row_width = 2 * self.p + self.d + 1
        self._bufs = {}

    # -- a shard is one part of a global filter: the single-handle step ---
    # paths would run on its local partials only (no global LSE / moments)
    def pf_step(self, *a, **k):
        raise ConfigError("a shard handle steps through ShardedFilter / native_step, not pf_step")

    def run(self, *a, **k):
        raise ConfigError("a shard handle steps through ShardedFilter / native_step, not run")

    def step_resident(self, *a, **k):
        raise ConfigError("a shard handle steps through ShardedFilter / native_step, not step_resident")

    # -- exchange buffers ------------------------------------------------
    def buffer(self, which: int):
        if which not in self._bufs:
            import torch
            ptr, nb = C.c_void_p(), C.c_uint64()
            self._check(self.lib.pfsmc_gpu_shard_buffer(self.h, which, C.byref(ptr), C.byref(nb)))
            self._bufs[which] = torch.as_tensor(_CudaArray(ptr.value, nb.value), device=f"cuda:{self.device}")
        return self._bufs[which]

    def stream(self):
        import torch
        return torch.cuda.ExternalStream(self.stream_handle, device=f"cuda:{self.device}")

    # -- phases ------------------------------------------------------------
    def predict(self, y, j, t_prev, t_obs, h):
        y = _f64(y)
        self._check(self.lib.pfsmc_gpu_shard_predict(self.h, _ptr(y), C.c_uint64(j), C.c_double(t_prev),
                                                      C.c_double(t_obs), C.c_double(h)))

    def finish_lse(self):
        self._check(self.lib.pfsmc_gpu_shard_finish_lse(self.h))

    def scan_records(self):
        self._check(self.lib.pfsmc_gpu_shard_scan_records(self.h))

    def resolve(self):
        self._check(self.lib.pfsmc_gpu_shard_resolve(self.h))

    def resolve_peers(self):
        """resolve with the windows read from the other shards over peer memory."""
        self.lib.pfsmc_gpu_shard_resolve_peers.restype = C.c_int
        self._check(self.lib.pfsmc_gpu_shard_resolve_peers(self.h))

    def serve(self) -> np.ndarray:
        counts = np.zeros(2 * self.world, dtype=np.uint32)
        self._check(self.lib.pfsmc_gpu_shard_serve(self.h, counts.ctypes.data_as(C.POINTER(C.c_uint32))))
        return counts

    def count_matrix(self) -> np.ndarray:
        """The world x world migration counts of the last serve (row r = rank r's sends),
        derived locally on every rank."""
        out = np.zeros(self.world * self.world, dtype=np.uint32)
        self._check(self.lib.pfsmc_gpu_shard_count_matrix(self.h, out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out.reshape(self.world, self.world)

    def attach_nccl(self, comm_group=None):
        """Native step: one NCCL communicator for this handle (id from rank 0,
        shared through torch.distributed)."""
        import torch
        import torch.distributed as dist
        self.lib.pfsmc_gpu_nccl_unique_id.restype = C.c_int
        self.lib.pfsmc_gpu_shard_attach_nccl.restype = C.c_int
        self.lib.pfsmc_gpu_shard_step.restype = C.c_int
        uid = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            self._check(self.lib.pfsmc_gpu_nccl_unique_id(uid.ctypes.data_as(C.POINTER(C.c_uint8))))
        t = torch.from_numpy(uid).to(f"cuda:{self.device}")
        dist.broadcast(t, 0, group=comm_group)
        uid = t.cpu().numpy()
        self._check(self.lib.pfsmc_gpu_shard_attach_nccl(self.h, uid.ctypes.data_as(C.POINTER(C.c_uint8))))
        self.native = True

    def attach_peers(self, comm_group=None) -> bool:
        """Migration over NVLink peer memory: allgather every rank's CUDA IPC
        handles (7 x 64 bytes) and map the peers' search tables and records.
        Returns False (the counted send / receive stays in use) if the mapping
        fails on any rank; every rank takes part in both collectives whatever
        happens locally, and a rank that mapped detaches again."""
        import torch
        import torch.distributed as dist
        L = self.lib
        for name in ("pfsmc_gpu_shard_ipc_handles", "pfsmc_gpu_shard_attach_peers", "pfsmc_gpu_shard_detach_peers"):
            getattr(L, name).restype = C.c_int
        mine = np.zeros(IPC_BYTES, dtype=np.uint8)
        ok_local = L.pfsmc_gpu_shard_ipc_handles(self.h, mine.ctypes.data_as(C.POINTER(C.c_uint8))) == 0
        dev = f"cuda:{self.device}"
        allh = torch.zeros(IPC_BYTES * self.world, dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(allh, torch.from_numpy(mine).to(dev), group=comm_group)
        allh = allh.cpu().numpy()
        if ok_local:
            ok_local = L.pfsmc_gpu_shard_attach_peers(self.h, allh.ctypes.data_as(C.POINTER(C.c_uint8))) == 0
        ok = torch.tensor([1 if ok_local else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=comm_group)
        self.peers = bool(ok.item())
        if not self.peers:
            self._check(L.pfsmc_gpu_shard_detach_peers(self.h))
        return self.peers

    def attach_peers_local(self, shards) -> None:
        """Peer table from same-process shards (rank order), no IPC."""
        L = self.lib
        L.pfsmc_gpu_shard_attach_peers_local.restype = C.c_int
        hs = (C.c_void_p * self.world)(*[sh.h for sh in sorted(shards, key=lambda x: x.rank)])
        self._check(L.pfsmc_gpu_shard_attach_peers_local(self.h, hs))
        self.peers = True

    # -- offspring-allocation mode ----------------------------------------
    def set_mode(self, mode: str):
        self.lib.pfsmc_gpu_shard_set_mode.restype = C.c_int
        self._check(self.lib.pfsmc_gpu_shard_set_mode(self.h, SHARD_MODES[mode]))
        self.mode = mode

    def offspring(self) -> np.ndarray:
        """Walk of every global slot's uniform: this rank's per-particle
        offspring counts (device) and the children of every rank (returned)."""
        self.lib.pfsmc_gpu_shard_offspring.restype = C.c_int
        tot = np.zeros(self.world, dtype=np.uint64)
        self._check(self.lib.pfsmc_gpu_shard_offspring(self.h, tot.ctypes.data_as(C.POINTER(C.c_uint64))))
        return tot

    def offspring_peer(self, phase: int) -> Optional[np.ndarray]:
        """Offspring counts over peer memory, phase 0 / 1 / 2 (a barrier
        across ranks between phases); phase 2 returns every rank's children."""
        self.lib.pfsmc_gpu_shard_offspring_peer.restype = C.c_int
        tot = np.zeros(self.world, dtype=np.uint64)
        self._check(self.lib.pfsmc_gpu_shard_offspring_peer(self.h, phase,
                                                            tot.ctypes.data_as(C.POINTER(C.c_uint64))))
        return tot if phase == 2 else None

    def offspring_counts(self) -> np.ndarray:
        self.lib.pfsmc_gpu_shard_offspring_counts.restype = C.c_int
        out = np.zeros(self.n, dtype=np.uint32)
        self._check(self.lib.pfsmc_gpu_shard_offspring_counts(self.h, out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out

    def offspring_pack(self) -> np.ndarray:
        self.lib.pfsmc_gpu_shard_offspring_pack.restype = C.c_int
        m = np.zeros(self.world * self.world, dtype=np.uint32)
        self._check(self.lib.pfsmc_gpu_shard_offspring_pack(self.h, m.ctypes.data_as(C.POINTER(C.c_uint32))))
        return m.reshape(self.world, self.world)

    def offspring_pull(self):
        self.lib.pfsmc_gpu_shard_offspring_pull.restype = C.c_int
        self._check(self.lib.pfsmc_gpu_shard_offspring_pull(self.h))

    def pull(self):
        """Phase D over peer memory + the update kernel."""
        self.lib.pfsmc_gpu_shard_pull.restype = C.c_int
        self._check(self.lib.pfsmc_gpu_shard_pull(self.h))

    def native_step(self, y, j, t_prev, t_obs, h) -> np.ndarray:
        out = np.zeros(self.row_width)
        y = _f64(y)
        self._check(self.lib.pfsmc_gpu_shard_step(self.h, _ptr(y), C.c_uint64(j), C.c_double(t_prev),
                                                   C.c_double(t_obs), C.c_double(h), _ptr(out)))
        return out

    def update(self, n_recv: int):
        self._check(self.lib.pfsmc_gpu_shard_update(self.h, C.c_uint64(n_recv)))

    def moments(self):
        self._check(self.lib.pfsmc_gpu_shard_moments(self.h))

    def finish_moments(self, flags: int) -> np.ndarray:
        out = np.zeros(self.row_width)
        self._check(self.lib.pfsmc_gpu_shard_finish_moments(self.h, flags, _ptr(out)))
        return out

    # -- BASELINE config 5 (payload64 shards) --------------------------------
    def _c5(self, name, *args):
        fn = getattr(self.lib, name)
        fn.restype = C.c_int
        self._check(fn(self.h, *args))

    def c5_stats(self):
        self._c5("pfsmc_gpu_shard_c5_stats")

    def c5_finish(self):
        self._c5("pfsmc_gpu_shard_c5_finish")

    def c5_pull(self, j: int):
        self._c5("pfsmc_gpu_shard_c5_pull", C.c_uint64(j))

    def c5_flip(self):
        self._c5("pfsmc_gpu_shard_c5_flip")

    def c5_native_iteration(self, j: int):
        self._c5("pfsmc_gpu_shard_c5_iteration", C.c_uint64(j))

    def c5_remote_pulls(self) -> int:
        v = C.c_uint64()
        self._c5("pfsmc_gpu_shard_c5_remote_pulls", C.byref(v))
        return int(v.value)

    def payload_doubles(self) -> int:
        return (self.d + self.p + 1) // 2 * 2 + 4

    def sync(self):
        self.synchronize()


# ------------------------------------------------------------------ comms
class LocalComm:
    """Collectives among shards that all live in this process."""

    def __init__(self, world: int):
        self.world = world

    def _fence(self, shards):
        import torch
        for s in shards:
            s.sync()
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.synchronize()

    def allgather(self, shards, src: int, dst: int):
        """dst buffer of every shard <- concat over ranks of src buffers."""
        self._fence(shards)
        parts = [s.buffer(src) for s in sorted(shards, key=lambda s: s.rank)]
        for s in shards:
            out = s.buffer(dst)
            n = parts[0].numel()
            for r, p in enumerate(parts):
                out[r * n:(r + 1) * n].copy_(p)
        self._fence(shards)

    def allgather_slices(self, shards, buf: int):
        """Each shard's global buffer carries its slice at rank * size; share them."""
        self._fence(shards)
        bufs = {s.rank: s.buffer(buf) for s in shards}
        n = bufs[0].numel() // self.world
        for r, b in bufs.items():
            for s in shards:
                if s.rank != r:
                    s.buffer(buf)[r * n:(r + 1) * n].copy_(b[r * n:(r + 1) * n])
        self._fence(shards)

    def exchange(self, shards, counts: dict, item_bytes: int):
        """Send region of rank r for dest d lives at d * cap (cap = N_local items)."""
        self._fence(shards)
        by_rank = {s.rank: s for s in shards}
        for d, sd in by_rank.items():
            off = 0
            cap = sd.n
            for r in range(self.world):
                k = int(counts[r][d])
                if k:
                    src = by_rank[r].buffer(BUF_SEND)[(d * cap) * item_bytes:(d * cap + k) * item_bytes]
                    sd.buffer(BUF_RECV)[off * item_bytes:(off + k) * item_bytes].copy_(src)
                off += k
        self._fence(shards)

    def gather_counts(self, shards, local_counts: dict) -> dict:
        return local_counts


class TorchComm:
    """One shard per process; torch.distributed (NCCL for GPUs, gloo on CPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()

    def _ctx(self, s):
        import contextlib
        import torch
        if hasattr(s, "stream_handle"):
            return torch.cuda.stream(s.stream())
        return contextlib.nullcontext()

    def allgather(self, shards, src: int, dst: int):
        (s,) = shards
        with self._ctx(s):
            self.dist.all_gather_into_tensor(s.buffer(dst), s.buffer(src))

    def allgather_slices(self, shards, buf: int):
        (s,) = shards
        b = s.buffer(buf)
        n = b.numel() // self.world
        with self._ctx(s):
            # in place: the input is this rank's slice of the output (NCCL in-place allgather)
            self.dist.all_gather_into_tensor(b, b[self.rank * n:(self.rank + 1) * n])

    def gather_counts(self, shards, local_counts: dict) -> dict:
        import torch
        (s,) = shards
        # every copy and the collective on the shard's stream: NCCL orders itself
        # after the current stream, and the host reads wait for it
        with self._ctx(s):
            t = torch.as_tensor(local_counts[s.rank].astype(np.int64))
            if hasattr(s, "stream_handle"):
                t = t.to(f"cuda:{s.device}")
            out = [torch.zeros_like(t) for _ in range(self.world)]
            self.dist.all_gather(out, t)
            return {r: out[r].cpu().numpy() for r in range(self.world)}

    def exchange(self, shards, counts: dict, item_bytes: int):
        (s,) = shards
        me, W = self.rank, self.world
        send, recv = s.buffer(BUF_SEND), s.buffer(BUF_RECV)
        cap = s.n
        ops = []
        off = 0
        for r in range(W):
            k_in = int(counts[r][me])          # rank r sends k_in payloads to me
            k_out = int(counts[me][r])         # I send k_out payloads to rank r
            rbuf = recv[off * item_bytes:(off + k_in) * item_bytes]
            sbuf = send[(r * cap) * item_bytes:(r * cap + k_out) * item_bytes]
            if r == me:
                with self._ctx(s):
                    rbuf.copy_(sbuf)
            else:
                if k_out:
                    ops.append(self.dist.P2POp(self.dist.isend, sbuf, r))
                if k_in:
                    ops.append(self.dist.P2POp(self.dist.irecv, rbuf, r))
            off += k_in
        if ops:
            with self._ctx(s):
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()


# ------------------------------------------------------------------ the filter
class ShardedFilter:
    """The global filter over `shards` (this process's shards) and `comm`."""

    def __init__(self, shards: List, comm, pull: bool = False, mode: str = "exact"):
        """pull: phase D as the peer-memory pull (shards attached with
        attach_peers / attach_peers_local) instead of the counted exchange.
        mode: "exact" (every slot's ancestor from the global multinomial,
        bitwise the single handle) or "offspring" (per-particle offspring
        counts from the same uniforms and exact CDF, children built on the
        ancestor's shard, only the load imbalance migrates; see
        pfsmc_gpu_shard_set_mode)."""
        if mode not in SHARD_MODES:
            raise ValueError(f"unknown migration mode {mode!r}")
        self.shards = sorted(shards, key=lambda s: s.rank)
        self.comm = comm
        self.pull = pull
        self.mode = mode
        for s in self.shards:
            if hasattr(s, "set_mode"):
                s.set_mode(mode)
        s0 = self.shards[0]
        self.d, self.p, self.world = s0.d, s0.p, s0.world

    def _each(self, fn):
        return [fn(s) for s in self.shards]

    def _refresh(self, flags):
        self._each(lambda s: s.moments())
        self.comm.allgather(self.shards, BUF_MOM, BUF_MOM_ALL)
        return self._each(lambda s: s.finish_moments(flags))[0]

    def initialize_uniform(self, **prior):
        self._each(lambda s: s.initialize_uniform(**prior))
        self._refresh(INIT_FLAGS)   # equal-weight mean
        self._refresh(INIT_FLAGS)   # covariance about it

    def initialize_gaussian(self, **prior):
        self._each(lambda s: s.initialize_gaussian(**prior))
        self._refresh(INIT_FLAGS)
        self._refresh(INIT_FLAGS)

    def set_ensemble(self, ens):
        """Global filter::Ensemble; each shard takes its slot range."""
        from .sampler import Ensemble
        for s in self.shards:
            sl = slice(s.n0, s.n0 + s.n)
            s.set_ensemble(Ensemble(ens.states[sl], ens.params_u[sl], ens.logw[sl], ens.mean_u, ens.cov_u))
        self._refresh(INJECT_FLAGS)

    def pf_step(self, y, j: int, t_prev: float, t_obs: float, h: float) -> TraceRow:
        sh, comm = self.shards, self.comm
        if len(sh) == 1 and getattr(sh[0], "native", False):
            # one native call: the same phases and exchanges over NCCL (pfsmc_gpu_shard_step)
            return self._row(sh[0].native_step(y, j, t_prev, t_obs, h), j, t_obs)
        self._each(lambda s: s.predict(y, j, t_prev, t_obs, h))
        comm.allgather(sh, BUF_PRED, BUF_PRED_ALL)                       # A
        self._each(lambda s: s.finish_lse())                             # (+ local tile prefixes)
        comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)                         # B
        self._each(lambda s: s.scan_records())
        self._phase_c()
        if self.mode == "offspring":
            if self.pull:
                # counts over peer memory: each rank draws only its own slots
                self._each(lambda s: s.offspring_peer(0))
                comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)                 # counts zeroed everywhere
                self._each(lambda s: s.offspring_peer(1))
                comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)                 # every increment done
                tot = [s.offspring_peer(2) for s in sh][0]               # identical on every rank
                self.last_totals = np.asarray(tot, dtype=np.int64)
                comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)                 # every rank's prefix complete
                self._each(lambda s: s.offspring_pull())
            else:
                tot = [s.offspring() for s in sh][0]                     # identical on every rank
                self.last_totals = np.asarray(tot, dtype=np.int64)
                mats = [s.offspring_pack() for s in sh]
                S = offspring_matrix(tot, self.world, sh[0].n)
                for m in mats:
                    if not np.array_equal(np.asarray(m, dtype=np.int64), S):
                        raise RuntimeError("offspring exchange: matrix mismatch")
                counts = {r: S[r] for r in range(self.world)}
                comm.exchange(sh, counts, 8 * sh[0].payload_doubles())   # D: only the imbalance
                for s in sh:
                    s.update(int(S[:, s.rank].sum()))
            comm.allgather(sh, BUF_MOM, BUF_MOM_ALL)                     # E
            return self._row(self._each(lambda s: s.finish_moments(STEP_FLAGS))[0], j, t_obs)
        if self.pull:
            # D over peer memory. The 2-double allgather (as in the native
            # step) orders every shard's pull after every shard's CDF tables;
            # the peers' record buffers a pull reads are the ones no update of
            # this step writes (double buffering), and E below orders the next
            # step's overwrite of ll_bar / the tables after every pull.
            comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)
            self._each(lambda s: s.pull())
            comm.allgather(sh, BUF_MOM, BUF_MOM_ALL)                     # E
            return self._row(self._each(lambda s: s.finish_moments(STEP_FLAGS))[0], j, t_obs)
        served = {s.rank: s.serve() for s in sh}
        mat = sh[0].count_matrix()                                       # same on every rank: no exchange
        counts = {r: mat[r] for r in range(self.world)}                  # counts[r][d]: r sends to d
        for r, c in served.items():
            if [int(v) for v in c[:self.world]] != [int(v) for v in mat[r]]:
                raise RuntimeError("sharded exchange: send count mismatch")
        item = 8 * sh[0].payload_doubles()
        comm.exchange(sh, counts, item)                                  # D: migration
        for s in sh:
            s.update(int(sum(counts[r][s.rank] for r in range(self.world))))
        comm.allgather(sh, BUF_MOM, BUF_MOM_ALL)                         # E
        return self._row(self._each(lambda s: s.finish_moments(STEP_FLAGS))[0], j, t_obs)

    def c5_iteration(self, j: int):
        """One BASELINE config-5 iteration of the global 64-byte-record
        ensemble (payload64 shards, peers attached): global log-sum-exp and
        weighted 2x2 covariance, the exact multinomial resampling and the
        gather with migration over peer memory; bitwise the single handle's
        pfsmc_gpu_c5_iteration."""
        sh, comm = self.shards, self.comm
        if len(sh) == 1 and getattr(sh[0], "native", False):
            sh[0].c5_native_iteration(j)
            return
        self._each(lambda s: s.c5_stats())
        comm.allgather(sh, BUF_C5, BUF_C5_ALL)                           # A
        self._each(lambda s: s.c5_finish())
        comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)                         # B
        self._each(lambda s: s.scan_records())
        self._phase_c()
        comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)                         # every rank's tables complete
        self._each(lambda s: s.c5_pull(j))                               # D
        comm.allgather(sh, BUF_SUM, BUF_SUM_ALL)                         # every pull done
        self._each(lambda s: s.c5_flip())

    def _phase_c(self):
        """C: tile headers to every rank; the windows too, unless the shards
        read each other's window lists over peer memory (pull mode)."""
        sh, comm = self.shards, self.comm
        comm.allgather_slices(sh, BUF_HDR)
        if self.pull and all(getattr(s, "peers", False) for s in sh):
            self._each(lambda s: s.resolve_peers())
        else:
            comm.allgather_slices(sh, BUF_WIN)
            self._each(lambda s: s.resolve())

    def _row(self, out, j, t_obs) -> TraceRow:
        p, d = self.p, self.d
        return TraceRow(j, t_obs, out[:p].copy(), out[p:2 * p].copy(), out[2 * p:2 * p + d].copy(),
                        float(out[2 * p + d]))

    def get_ensemble(self):
        """Local shards' slices concatenated (rank order)."""
        from .sampler import Ensemble
        parts = [s.get_ensemble() for s in self.shards]
        return Ensemble(np.concatenate([e.states for e in parts]), np.concatenate([e.params_u for e in parts]),
                        np.concatenate([e.logw for e in parts]), parts[0].mean_u, parts[0].cov_u)

    def ancestors(self) -> np.ndarray:
        return np.concatenate([s.step_diagnostics()[0] for s in self.shards])
