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
from oracle_ctypes import Ensemble as OEns
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


def _sharded_run(shards, comm, mode="exact"):
    from paper_1411_1702_b200.sharded import ShardedFilter
    f = ShardedFilter(shards, comm, mode=mode)
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


# ---------------------------------------------------------------- offspring mode
def _offspring_run(shards, comm, check_single=True):
    """Offspring-allocation mode: before every step the global ensemble is
    also stepped by the single-handle oracle, whose ancestors give the
    multinomial offspring counts the sharded filter must reproduce bitwise."""
    from paper_1411_1702_b200.sharded import ShardedFilter
    f = ShardedFilter(shards, comm, mode="offspring")
    f.initialize_uniform(**PRIOR)
    sc = _sc()
    out = []
    tp = 0.0
    for j, y in enumerate(_ys(), 1):
        want, anc_single = None, None
        if check_single:  # needs the whole ensemble in this process
            g = f.get_ensemble()
            ens = OEns(g.states.copy(), g.params_u.copy(), g.logw.copy(), g.mean_u.copy(), g.cov_u.copy())
            _tr, dg = O.pf_step(sc, ens, y, j, tp, tp + 0.1, diag=True)
            want, anc_single = np.bincount(dg["ancestors"], minlength=N_GLOB), dg["ancestors"]
        row = f.pf_step(y, j, tp, tp + 0.1, 0.1)
        got = np.concatenate([s.offspring_counts() for s in f.shards]).astype(np.int64)
        anc = f.ancestors()
        out.append((want, got, anc, anc_single, np.concatenate([row.theta_mean, row.theta_var,
                                                                 row.state_mean, [row.ess]])))
        tp += 0.1
    return out, f.get_ensemble()


def test_local_comm_offspring_counts_match_single_handle():
    """Offspring counts bitwise the single handle's multinomial counts (same
    keyed uniforms, same exact CDF); the children are laid out in ancestor
    order (rank by rank), so the slot ancestors are the sorted single-handle
    ancestors of the shards that hold them."""
    from paper_1411_1702_b200.sharded import LocalComm
    shards = [CpuShard(_sc(), N_GLOB, r, 2) for r in range(2)]
    out, ens = _offspring_run(shards, LocalComm(2))
    for j, (want, got, anc, anc_single, tr) in enumerate(out, 1):
        assert np.array_equal(got, want), f"step {j}: offspring counts differ"
        # the children in ancestor order: the slot ancestors are the sorted
        # single-handle ancestors
        assert np.array_equal(anc, np.sort(anc_single)), j
        assert np.isfinite(tr).all()
    assert np.isfinite(ens.states).all()


def test_offspring_matrix_moves_only_the_imbalance():
    from paper_1411_1702_b200.sharded import offspring_matrix
    n = 10
    # balanced: nothing crosses
    assert np.array_equal(offspring_matrix([10, 10, 10], 3, n), np.diag([10, 10, 10]))
    # rank 0 has 17 children: 7 spill onto rank 1, whose 5 children spill 2 onto rank 2
    S = offspring_matrix([17, 5, 8], 3, n)
    assert np.array_equal(S, np.array([[10, 7, 0], [0, 3, 2], [0, 0, 8]]))
    assert S.sum() == 30 and np.array_equal(S.sum(0), [10, 10, 10])
    # degenerate weights: one rank makes every child
    S = offspring_matrix([0, 30, 0], 3, n)
    assert np.array_equal(S, np.array([[0, 0, 0], [10, 10, 10], [0, 0, 0]]))


def _offspring_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1411_1702_b200.sharded import TorchComm
        shard = CpuShard(_sc(), N_GLOB, rank, world)
        out, ens = _offspring_run([shard], TorchComm(), check_single=False)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), got=np.array([o[1] for o in out]),
                 anc=np.array([o[2] for o in out]),
                 tr=np.array([o[4] for o in out]), states=ens.states)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_offspring_mode():
    """Offspring mode across two gloo processes: each rank's counts are the
    single handle's for its particles; the trace and the states equal the
    one-process (LocalComm) offspring run."""
    import torch.multiprocessing as mp
    from paper_1411_1702_b200.sharded import LocalComm
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_offspring_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        parts = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(2)]
    local, lens = _offspring_run([CpuShard(_sc(), N_GLOB, r, 2) for r in range(2)], LocalComm(2))
    half = N_GLOB // 2
    for r, p in enumerate(parts):
        for j in range(STEPS):
            assert np.array_equal(p["got"][j], local[j][0][r * half:(r + 1) * half]), (r, j)
            assert np.array_equal(p["anc"][j], local[j][2][r * half:(r + 1) * half]), (r, j)
            np.testing.assert_allclose(p["tr"][j], local[j][4], rtol=1e-12, atol=0)
    np.testing.assert_allclose(np.concatenate([p["states"] for p in parts]), lens.states, rtol=1e-13)
