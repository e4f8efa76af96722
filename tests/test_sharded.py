"""Multi-shard path on CPU: the product orchestrator
`ShardedFilter` with `TorchComm` over world_size-2 `gloo` processes (and with
`LocalComm` in one process), shards backed by tests/cpu_shard.py, against the
single-process oracle pf_step. Ancestors must be identical (every rank
resolves the exact sequential CDF over all shards), states / weights within
1e-12, the trace row within 1e-10."""
import math
import os
import socket
import tempfile

import numpy as np
import pytest

from cpu_shard import CpuShard
from oracle_ctypes import Oracle, StepConfig

O = Oracle()
N_GLOB, STEPS, SEED = 2 * 384, 3, 13
PRIOR = dict(th_lo=[0.5, 0.5], th_hi=[1.5, 1.5], x_lo=[0.5, 0.5], x_hi=[1.5, 1.5])


def _sc():
    return StepConfig(model="lv", family="am", order=2, h=0.1, a=0.98, seed=SEED, obs_idx=(0, 1), sigma=0.05)


def _ys():
    rng = np.random.default_rng(5)
    return [np.array([1.2, 0.9]) + 0.05 * rng.standard_normal(2) for _ in range(STEPS)]


def _oracle_run():
    sc = _sc()
    ens = O.init_uniform("lv", N_GLOB, SEED, **PRIOR)
    traces, ancs = [], []
    tp = 0.0
    for j, y in enumerate(_ys(), 1):
        tr, dg = O.pf_step(sc, ens, y, j, tp, tp + 0.1, diag=True)
        traces.append(tr)
        ancs.append(dg["ancestors"])
        tp += 0.1
    return traces, ancs, ens


def _sharded_run(shards, comm):
    from paper_1411_1702_b200.sharded import ShardedFilter
    f = ShardedFilter(shards, comm)
    f.initialize_uniform(**PRIOR)
    traces, ancs = [], []
    tp = 0.0
    for j, y in enumerate(_ys(), 1):
        row = f.pf_step(y, j, tp, tp + 0.1, 0.1)
        traces.append(np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]]))
        ancs.append(f.ancestors())
        tp += 0.1
    return traces, ancs, f.get_ensemble()


def _check(traces, ancs, ens, ref):
    rt, ra, re = ref
    for j in range(STEPS):
        assert np.array_equal(ancs[j], ra[j]), f"step {j + 1}: ancestors differ"
        np.testing.assert_allclose(traces[j], rt[j], rtol=1e-10, atol=0)
    return re


def test_local_comm_two_shards_matches_oracle():
    from paper_1411_1702_b200.sharded import LocalComm
    shards = [CpuShard(_sc(), N_GLOB, r, 2) for r in range(2)]
    traces, ancs, ens = _sharded_run(shards, LocalComm(2))
    re = _check(traces, ancs, ens, _oracle_run())
    np.testing.assert_allclose(ens.states, re.states, rtol=1e-12)
    np.testing.assert_allclose(np.exp(ens.logw), np.exp(re.logw), rtol=1e-10)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1411_1702_b200.sharded import TorchComm
        shard = CpuShard(_sc(), N_GLOB, rank, world)
        traces, ancs, ens = _sharded_run([shard], TorchComm())
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), traces=np.array(traces), ancs=np.array(ancs),
                 states=ens.states, logw=ens.logw)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_matches_oracle():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        parts = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(2)]
    rt, ra, re = _oracle_run()
    half = N_GLOB // 2
    for r, p in enumerate(parts):  # same global trace on every rank; ancestors of its own slots
        for j in range(STEPS):
            assert np.array_equal(p["ancs"][j], ra[j][r * half:(r + 1) * half])
            np.testing.assert_allclose(p["traces"][j], rt[j], rtol=1e-10, atol=0)
    # rank r holds slots [r*N/2, (r+1)*N/2)
    states = np.concatenate([p["states"] for p in parts])
    np.testing.assert_allclose(states, re.states, rtol=1e-12)
