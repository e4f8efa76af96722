"""GPU: the offspring-allocation sharded step (north_star).

R shard handles of one filter on this GPU (LocalComm: phases strictly in
order, no kernel waits on another shard), counted exchange and the
peer-memory pull:
* the per-particle offspring counts are bitwise the single handle's
  multinomial counts for the same ensemble (same keyed uniforms, same exact
  sequential CDF: filter.cpp:158-178), and the slot ancestors are the sorted
  single-handle ancestors (children in ancestor order, shard by shard);
* the children's states / weights / trace equal the same algorithm run on the
  C oracle's arithmetic (tests/cpu_shard.py) within the north_star bars;
* the native step (NCCL, world 1) equals the phase-by-phase orchestration
  bitwise, counted and pull.
"""
import numpy as np
import pytest

from cpu_shard import CpuShard
from oracle_ctypes import StepConfig

pytestmark = pytest.mark.gpu


def _prob(n, T=3, seed=31):
    from paper_1411_1702_b200 import problems
    return problems.lotka_volterra(particles=n, T=T, seed=seed)


def _trace(row):
    return np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]])


@pytest.mark.parametrize("world,pull", [(2, False), (4, False), (2, True), (4, True)])
def test_offspring_counts_bitwise_single_handle(world, pull):
    from paper_1411_1702_b200.sampler import GpuSampler
    from paper_1411_1702_b200.sharded import GpuShard, LocalComm, ShardedFilter
    n, T = 1 << 16, 4
    prob = _prob(n, T)
    single = GpuSampler("lv", prob.cfg, prob.obs)
    shards = [GpuShard("lv", prob.cfg, prob.obs, r, world) for r in range(world)]
    if pull:
        for s in shards:
            s.attach_peers_local(shards)
    f = ShardedFilter(shards, LocalComm(world), pull=pull, mode="offspring")
    f.initialize_uniform(**prob.prior)
    tp = 0.0
    moved = []
    for j in range(1, T + 1):
        t1 = prob.times[j - 1]
        single.set_ensemble(f.get_ensemble())  # the same ensemble on both sides
        single.pf_step(prob.ys[j - 1], j, tp, t1)
        f.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
        a1 = single.step_diagnostics()[0].astype(np.int64)
        counts = np.concatenate([s.offspring_counts() for s in shards]).astype(np.int64)
        assert np.array_equal(counts, np.bincount(a1, minlength=n)), f"step {j}: offspring counts"
        assert np.array_equal(f.ancestors().astype(np.int64), np.sort(a1)), f"step {j}: children order"
        tot = f.last_totals
        moved.append(int(np.abs(np.cumsum(tot)[:-1] - np.arange(1, world) * (n // world)).sum()))
        tp = t1
    # only the imbalance crosses shards: far less than exact mode's (G-1)/G of all slots
    assert max(moved) < n * (world - 1) // world // 4, moved
    single.close()
    for s in shards:
        s.close()


def test_offspring_children_match_oracle_arithmetic():
    """The children (proliferation, repropagation, innovation, reweighting
    keyed by their new global slot) against the same offspring-mode step run
    on the C oracle's arithmetic (CpuShard), same injected ensemble."""
    from paper_1411_1702_b200.sampler import Ensemble
    from paper_1411_1702_b200.sharded import GpuShard, LocalComm, ShardedFilter
    world, n, T = 2, 1 << 15, 2
    prob = _prob(n, T, seed=7)
    sc = StepConfig(model="lv", family=prob.cfg.family, order=prob.cfg.order, h=0.1, a=0.98, seed=7,
                    obs_idx=(0, 1), sigma=0.05)
    gs = [GpuShard("lv", prob.cfg, prob.obs, r, world) for r in range(world)]
    cs = [CpuShard(sc, n, r, world) for r in range(world)]
    fg = ShardedFilter(gs, LocalComm(world), mode="offspring")
    fc = ShardedFilter(cs, LocalComm(world), mode="offspring")
    fg.initialize_uniform(**prob.prior)
    tp = 0.0
    for j in range(1, T + 1):
        t1 = prob.times[j - 1]
        e = fg.get_ensemble()
        fc.set_ensemble(Ensemble(e.states, e.params_u, e.logw, e.mean_u, e.cov_u))
        rg = fg.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
        rc = fc.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
        assert np.array_equal(fg.ancestors().astype(np.int64), fc.ancestors().astype(np.int64)), j
        eg, ec = fg.get_ensemble(), fc.get_ensemble()
        assert np.max(np.abs(eg.states - ec.states) / np.maximum(np.abs(ec.states), 1e-300)) < 1e-10, j
        dp = np.max(np.abs(eg.params_u - ec.params_u), axis=0) / np.max(np.abs(ec.params_u), axis=0)
        assert np.max(dp) < 1e-10, j
        np.testing.assert_allclose(np.exp(eg.logw), np.exp(ec.logw), rtol=1e-10, atol=0)
        np.testing.assert_allclose(_trace(rg), _trace(rc), rtol=1e-8, atol=0)
        tp = t1
    for s in gs:
        s.close()


@pytest.mark.parametrize("pull", [False, True])
def test_offspring_native_step_world1(pull):
    """pfsmc_gpu_shard_step in offspring mode (NCCL at world 1, counted or
    peer-memory pull, graph-captured) == the phase-by-phase orchestration."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_1411_1702_b200.sharded import GpuShard, LocalComm, ShardedFilter, TorchComm
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        n, T = 1 << 15, 4
        prob = _prob(n, T, seed=9)
        a = GpuShard("lv", prob.cfg, prob.obs, 0, 1)
        b = GpuShard("lv", prob.cfg, prob.obs, 0, 1)
        fa = ShardedFilter([a], TorchComm(), mode="offspring")
        fb = ShardedFilter([b], LocalComm(1), mode="offspring")
        a.attach_nccl()
        if pull:
            assert a.attach_peers()
        fa.initialize_uniform(**prob.prior)
        fb.initialize_uniform(**prob.prior)
        tp = 0.0
        for j in range(1, T + 1):
            t1 = prob.times[j - 1]
            ra = fa.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
            rb = fb.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
            assert np.array_equal(_trace(ra), _trace(rb)), j
            assert np.array_equal(fa.ancestors(), fb.ancestors()), j
            tp = t1
        ea, eb = fa.get_ensemble(), fb.get_ensemble()
        assert np.array_equal(ea.states, eb.states) and np.array_equal(ea.logw, eb.logw)
        a.close()
        b.close()
    finally:
        dist.destroy_process_group()
