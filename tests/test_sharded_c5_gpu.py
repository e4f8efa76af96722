"""BASELINE config 5 over several GPUs' worth of shards on ONE GPU: R
payload64 shard handles in one process (LocalComm: the phases run strictly
one after another; the migration is the peer-memory pull through a peer table
of the other shards' device pointers) reproduce the single handle's
resample / reduction iterations bit for bit: ancestors (global indices),
records, weighted mean and covariance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_c5_iterations_are_the_single_handle_bitwise(world):
    from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
    from paper_1411_1702_b200.sharded import GpuShard, LocalComm, ShardedFilter
    n = world << 17  # 64 tiles of 2048 per shard
    rng = np.random.default_rng(21)
    ens = Ensemble(rng.standard_normal((n, 6)), rng.standard_normal((n, 2)), np.zeros(n), np.zeros(2), np.eye(2))
    cfg, obs = PfConfig(particles=n, seed=31), ObservationModel([0], 1.0)
    single = GpuSampler("payload64", cfg, obs)
    single.set_ensemble(ens)
    shards = [GpuShard("payload64", cfg, obs, r, world) for r in range(world)]
    for s in shards:
        s.attach_peers_local(shards)
    f = ShardedFilter(shards, LocalComm(world), pull=True)
    f.set_ensemble(ens)
    for sigma, key in ((2.0, 3), (0.5, 4)):
        single.c5_set_logweights(sigma, key)
        for s in shards:
            s.c5_set_logweights(sigma, key)
        for it in range(1, 4):
            single.c5_iteration(it)
            single.synchronize()
            f.c5_iteration(it)
            for s in shards:
                s.synchronize()
            a1, _, _ = single.step_diagnostics()
            assert np.array_equal(a1, f.ancestors()), (sigma, it)
            e1, e2 = single.get_ensemble(), f.get_ensemble()
            assert np.array_equal(e1.states, e2.states) and np.array_equal(e1.params_u, e2.params_u), (sigma, it)
            assert np.array_equal(e1.mean_u, e2.mean_u) and np.array_equal(e1.cov_u, e2.cov_u), (sigma, it)
    # every remote record counted once: the pulls that crossed shards
    a1, _, _ = single.step_diagnostics()
    owner = a1.astype(np.int64) // (n // world)
    crossed = sum(int(np.count_nonzero(owner[s.n0:s.n0 + s.n] != s.rank)) for s in shards)
    assert crossed > 0
    assert sum(s.c5_remote_pulls() for s in shards) >= crossed
    single.close()
    for s in shards:
        s.close()


def test_sharded_c5_rejects_ragged_shards():
    from paper_1411_1702_b200.sampler import ConfigError, ObservationModel, PfConfig
    from paper_1411_1702_b200.sharded import GpuShard
    s = GpuShard("payload64", PfConfig(particles=2 * 16384, seed=1), ObservationModel([0], 1.0), 0, 2)
    with pytest.raises(ConfigError, match="64 exact-CDF tiles"):
        s.c5_stats()
    s.close()
